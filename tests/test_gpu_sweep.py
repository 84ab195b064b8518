"""Seeded randomized parity sweep: every product path through the drop-in API against the CPU
oracle on random shapes -- odd and prime n, n = 1 and 2, k = 0 and k = n, both orders, structured
and unstructured operands. Each case is small (the oracle finishes in milliseconds); the point is
breadth beyond the fixed cases of the per-path test files.

Bars (north_star): selected indices bit-exact (or an 8-ulp near tie, after which the
oracle is re-run with the device's selection), values rel. Frobenius <= 1e-10 in fp64."""
import numpy as np
import pytest

import oracle as O
from conftest import rel
from test_gpu_circulant import near_tie_ok
from test_gpu_fsparse import parity as sfft_parity

pytestmark = pytest.mark.gpu

N_CASES = 40


def _cases(stream, lo=1, hi=384):
    rng = np.random.default_rng([2504, 19308, stream])
    out = []
    for i in range(N_CASES):
        n = int(rng.integers(lo, hi + 1)) if i >= 4 else max(lo, [1, 2, 3, 127][i])
        k = int(rng.integers(0, min(n, 40) + 1))
        if i % 7 == 5:
            k = n if n <= 64 else k
        out.append((n, k, int(rng.integers(0, 2)), int(rng.integers(0, 2 ** 31))))
    return out


@pytest.fixture(scope="module")
def P():
    import paper_2504_19308_b200 as P
    return P


def _close(M, Mo, tol=1e-10):
    nrm = np.linalg.norm(Mo)
    if nrm > 0:
        assert rel(M, Mo) < tol
    else:
        assert np.linalg.norm(M) < 1e-12


@pytest.mark.parametrize("n,k,order,seed", _cases(0))
def test_sweep_cycle(P, n, k, order, seed):
    rng = np.random.default_rng(seed)
    kb = int(rng.integers(0, min(n, 40) + 1))
    if rng.integers(0, 2):  # planted cycles (distinct energies) or dense noise (flat energies)
        A = O.gen_cycle_operand(n, min(n, k + 2), seed % 10007)
        B = O.gen_cycle_operand(n, min(n, kb + 2), seed % 10009)
    else:
        A, B = rng.standard_normal((n, n)), rng.standard_normal((n, n))
    M, rep = P.cycle_first_order_multiply(A, B, k, order, k_b=kb)
    Mo, ro = O.cycle_first_order_multiply(A, B, k, order, kb=kb)
    assert rep.selected_a == ro["selected_a"] and rep.selected_b == ro["selected_b"]
    _close(M, Mo)


@pytest.mark.parametrize("n,k,order,seed", _cases(1))
def test_sweep_circulant(P, n, k, order, seed):
    rng = np.random.default_rng(seed)
    k = min(k, n)
    cplx = bool(rng.integers(0, 4) == 0)
    A, B = rng.standard_normal((n, n)), rng.standard_normal((n, n))
    if cplx:
        A = A + 1j * rng.standard_normal((n, n))
    M, rep = P.circulant_first_order_multiply(A, B, k, order)
    mags_a, mags_b = O.circulant_decompose(A)[1], O.circulant_decompose(B)[1]
    near_tie_ok(rep.selected_a, O.top_indices(mags_a, k), mags_a)
    near_tie_ok(rep.selected_b, O.top_indices(mags_b, k), mags_b)
    Mo, _ = O.circulant_first_order_multiply(A, B, k, order, rep.selected_a, rep.selected_b)
    _close(M, Mo)


@pytest.mark.parametrize("n,k,order,seed", _cases(2, hi=300))
def test_sweep_sfft(P, n, k, order, seed):
    from paper_2504_19308_b200 import fsparse as F
    rng = np.random.default_rng(seed)
    k = max(1, min(k, n))
    A, B = rng.standard_normal((n, n)), rng.standard_normal((n, n))
    sfft_parity(F, A, B, k, order, "rows" if seed % 2 else "cols")


@pytest.mark.parametrize("n,k,order,seed", _cases(3, lo=4, hi=320))
def test_sweep_svd(P, n, k, order, seed):
    rng = np.random.default_rng(seed)
    s = int(rng.integers(1, 6))
    q = int(rng.integers(0, 3))
    sigma = (np.arange(n) + 1.0) ** -float(rng.uniform(0.5, 2.0))
    A = O.gen_haar_spectrum(n, sigma, seed % 10007)
    B = O.gen_haar_spectrum(n, sigma[::-1].copy(), seed % 10009)
    M, rep = P.svd_first_order_multiply(A, B, s, order, seed % 1000, power_iterations=q)
    Mo, ro = O.svd_first_order_multiply(A, B, s, order, seed % 1000, power_iterations=q)
    assert rep.k == ro["k"]
    # the truncated factors are unique up to rounding in the discarded directions: 1e-9 covers
    # sketches whose trailing singular values approach eps * sigma_1
    _close(M, Mo, 1e-9)


# (the mixed product has no reference function; its C-ABI documents n >= 2, k_svd <= min(n, 128))
@pytest.mark.parametrize("n,k,order,seed", _cases(4, lo=8, hi=320))
def test_sweep_mixed(P, n, k, order, seed):
    rng = np.random.default_rng(seed)
    ks = int(rng.integers(1, min(n, 32) + 1))
    kc = min(k, n)
    q = int(rng.integers(0, 2))
    A = O.gen_haar_spectrum(n, (np.arange(n) + 1.0) ** -1.5, seed % 10007)
    B = O.gen_cycle_operand(n, min(n, kc + 2), seed % 10009)
    M, rep = P.mixed_first_order_multiply(A, B, ks, kc, order, seed=seed % 1000, power_iterations=q)
    Mo, ro = O.mixed_first_order_multiply(A, B, ks, kc, order, seed % 1000, power_iterations=q)
    assert rep.selected_b == ro["selected_b"]
    _close(M, Mo)


@pytest.mark.parametrize("n,k,order,seed", _cases(5, lo=8, hi=700)[:24])
def test_sweep_cycle_fp32_device_tensors(P, n, k, order, seed):
    """fp32 device tensors in, fp32 device tensor out (the C4 / C5 calling convention): planted
    cycles, so the selection is robust to fp32 rounding of the energies; values within 1e-4."""
    import torch
    kb = max(1, k // 2)
    A = O.gen_cycle_operand(n, min(n, k + 2), seed % 10007).astype(np.float32)
    B = O.gen_cycle_operand(n, min(n, kb + 2), seed % 10009).astype(np.float32)
    M, rep = P.cycle_first_order_multiply(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), k, order, k_b=kb)
    assert M.dtype == torch.float32 and M.is_cuda
    Mo, ro = O.cycle_first_order_multiply(A.astype(np.float64), B.astype(np.float64), k, order, kb=kb)
    if k <= min(n, k + 2) and kb <= min(n, kb + 2):  # only planted cycles are kept
        assert rep.selected_a == ro["selected_a"] and rep.selected_b == ro["selected_b"]
    _close(M.double().cpu().numpy(), Mo, 1e-4)
