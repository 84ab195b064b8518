"""Device generators (paper_2504_19308_b200.genmat, reference genmat.py:109-153): the value-exact
kinds reproduce the reference's matrices bit for bit (golden vectors from the reference itself);
the Haar kinds match in distribution (orthogonality, spectrum)."""
import numpy as np
import pytest
import torch

from paper_2504_19308_b200 import genmat as G

EXACT = ("toeplitz", "hankel", "block-toeplitz", "symmetric", "general", "circulant", "kappa")


@pytest.mark.parametrize("kind", EXACT)
def test_exact_kinds_cpu(golden, kind):
    g = golden("genmat")
    for n in (1, 2, 5, 12, 36):
        assert np.array_equal(G.generate(kind, n, 3, device="cpu").numpy(), g[f"{kind}_{n}"]), (kind, n)
    if kind == "block-toeplitz":
        assert np.array_equal(G.generate(kind, 12, 4, block=3, device="cpu").numpy(), g["block-toeplitz_12_b3"])


def test_validation():
    with pytest.raises(ValueError):
        G.generate("bogus", 4, device="cpu")
    with pytest.raises(ValueError):
        G.generate("block-toeplitz", 12, block=5, device="cpu")
    with pytest.raises(ValueError):
        G.generate("haar-spectrum", 4, device="cpu")
    with pytest.raises(ValueError):
        G.generate("general", 4, spectrum=np.ones(4), device="cpu")


def test_haar_spectrum_cpu():
    n = 48
    sig = 0.9 ** np.arange(n)
    A = G.generate("haar-spectrum", n, 5, spectrum=sig, device="cpu").numpy()
    assert np.allclose(np.linalg.svd(A, compute_uv=False), sig, rtol=1e-12, atol=1e-14)
    B = G.generate("haar-spectrum", n, 5, spectrum=sig, device="cpu").numpy()
    assert np.array_equal(A, B)  # deterministic per seed
    T1 = G.generate("type1", n, 2, device="cpu").numpy()
    assert np.allclose(np.linalg.svd(T1, compute_uv=False), np.exp(-np.arange(n) / n), rtol=1e-12)


def test_config_operands_cpu():
    A, J = G.cycle_operand(64, 5, 1, device="cpu")
    i = np.arange(64)
    lay = A.numpy()[i[:, None], (i[:, None] - i[None, :]) % 64]
    norms = np.linalg.norm(lay, axis=0)
    assert sorted(np.argsort(-norms)[:5].tolist()) == J
    C = G.circulant_operand(64, 3, 2, device="cpu")
    assert C.shape == (64, 64) and torch.isfinite(C).all()
    A5, J5 = G.c5_operand(256, 8, 2, seed=1, operand=0, device="cpu", dtype=torch.float64)
    r = np.arange(256)
    lay = A5.numpy()[r[:, None], (r[:, None] - r[None, :]) % 256]
    assert sorted(np.argsort(-np.linalg.norm(lay, axis=0))[:8].tolist()) == J5
