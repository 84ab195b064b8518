"""Transforms longer than one CTA's shared memory: the four-step path of circulant.cu (batched
FFT through global memory, unfused circulant stages) for power-of-two n up to 2^18.

  * unitary_dft at n = 16384 / 65536 (contiguous and strided batches) against numpy's FFT;
  * with APX_FFT_BIG=1 (a child process: the switch is read once) the four-step path runs at
    small n and must reproduce the fused shared-memory path and the CPU oracle;
  * the C3-style circulant product at n = 8192 (too large for the fused kernels) against the
    CPU oracle, with the near-tie protocol of SURVEY §8(c).
Tolerance: 1e-10 relative Frobenius (fp64), as everywhere on the circulant path.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O
from conftest import rel

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("n", [16384, 65536, 10007, 12000])
def test_unitary_dft_long(n):
    from paper_2504_19308_b200 import core as K
    rng = np.random.default_rng(n)
    x = rng.standard_normal((3, n)) + 1j * rng.standard_normal((3, n))
    for direction, f in (("forward", np.fft.fft), ("inverse", np.fft.ifft)):
        y = K.unitary_dft(x, direction, axis=-1)
        assert rel(y, f(x, axis=-1, norm="ortho")) < 1e-12
    xt = np.ascontiguousarray(x.T)  # strided: transform along axis 0
    assert rel(K.unitary_dft(xt, "forward", axis=0), np.fft.fft(xt, axis=0, norm="ortho")) < 1e-12


def _oracle_with_protocol(A, B, k, order, sel_a, sel_b):
    """SURVEY §8(c) near-tie protocol: real operands have conjugate-symmetric spectra, so the
    magnitudes of t and n - t tie up to rounding; every differing pick must be such a near tie,
    and the oracle is then re-run with the GPU's selections (as test_circulant.py:108-110 does)."""
    from test_gpu_circulant import near_tie_ok
    _, ma = O.circulant_decompose(A)
    _, mb = O.circulant_decompose(B)
    Mo, ro = O.circulant_first_order_multiply(A, B, k, order)
    subs = near_tie_ok(sel_a, list(ro["selected_a"]), ma) + near_tie_ok(sel_b, list(ro["selected_b"]), mb)
    if subs:
        Mo, ro = O.circulant_first_order_multiply(A, B, k, order, force_sel_a=sel_a, force_sel_b=sel_b)
    return Mo, subs


_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import oracle as O
import paper_2504_19308_b200 as P
from paper_2504_19308_b200 import circulant as C
out = {}
for n, k in ((256, 5), (1024, 5), (300, 5), (997, 4)):
    A = O.gen_circulant_operand(n, 6, 11 + n)
    B = O.gen_circulant_operand(n, 6, 12 + n)
    for order in (0, 1):
        M, rep = C.circulant_first_order_multiply(A, B, k, order)
        out[f"M{n}_{order}"] = M
        out[f"sel{n}_{order}"] = np.array(rep.selected_a + rep.selected_b)
    spec = C.circulant_decompose(A)
    out[f"cols{n}"] = spec.columns
    out[f"mags{n}"] = spec.magnitudes
    x = np.random.default_rng(n).standard_normal((4, n)) + 0j
    out[f"dft{n}"] = P.unitary_dft(x, "forward", axis=-1)
np.savez(sys.argv[2], **out)
"""


def _run_child(tmp_path, big):
    path = str(tmp_path / f"child_{int(big)}.npz")
    env = dict(os.environ)
    env["APX_FFT_BIG"] = "1" if big else "0"
    r = subprocess.run([sys.executable, "-c", _CHILD, ROOT, path], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    with np.load(path) as z:
        return {k: z[k] for k in z.files}


def test_four_step_path_matches_fused_and_oracle(tmp_path):
    big = _run_child(tmp_path, True)
    fused = _run_child(tmp_path, False)
    from test_gpu_circulant import near_tie_ok
    tied = set()
    for n, k in ((256, 5), (1024, 5), (300, 5), (997, 4)):
        A = O.gen_circulant_operand(n, 6, 11 + n)
        B = O.gen_circulant_operand(n, 6, 12 + n)
        _, ma = O.circulant_decompose(A)
        _, mb = O.circulant_decompose(B)
        for order in (0, 1):
            key = f"sel{n}_{order}"
            sb, sf = [int(v) for v in big[key]], [int(v) for v in fused[key]]
            # the two transforms round differently, so an exact conjugate-pair tie (t, n - t of a
            # real operand) may break either way: allowed only as a near tie
            if sb != sf:
                near_tie_ok(sb[:k], sf[:k], ma)
                near_tie_ok(sb[k:], sf[k:], mb)
                tied.add(f"M{n}_{order}")
            for out in (big, fused):
                sel = [int(v) for v in out[key]]
                Mo, _ = _oracle_with_protocol(A, B, k, order, sel[:k], sel[k:])
                assert rel(out[f"M{n}_{order}"], Mo) < 1e-10
    for key in big:
        if not key.startswith("sel") and key not in tied:
            assert rel(big[key], fused[key]) < 1e-12, key
    for n, k in ((256, 5), (1024, 5), (300, 5), (997, 4)):
        A = O.gen_circulant_operand(n, 6, 11 + n)
        S, mags = O.circulant_decompose(A)
        assert rel(big[f"cols{n}"], S) < 1e-12
        assert rel(big[f"mags{n}"], mags) < 1e-12


def test_circulant_n8192_vs_oracle():
    from paper_2504_19308_b200 import circulant as C
    n, k = 8192, 16
    A = O.gen_circulant_operand(n, 16, 5)
    B = O.gen_circulant_operand(n, 16, 6)
    M, rep = C.circulant_first_order_multiply(A, B, k, 1)
    Mo, subs = _oracle_with_protocol(A, B, k, 1, rep.selected_a, rep.selected_b)
    err = rel(M, Mo)
    print(f"circulant n=8192 (four-step path): rel vs oracle {err:.3e}, near-tie substitutions {subs}")
    assert err < 1e-10


def test_circulant_n5000_bluestein_vs_oracle():
    """n = 5000: too long for the fused kernels' buffers and not a power of two -- Bluestein
    transforms of length 16384 through the four-step path."""
    from paper_2504_19308_b200 import circulant as C
    n, k = 5000, 6
    A = O.gen_circulant_operand(n, 8, 7)
    B = O.gen_circulant_operand(n, 8, 8)
    M, rep = C.circulant_first_order_multiply(A, B, k, 1)
    Mo, subs = _oracle_with_protocol(A, B, k, 1, rep.selected_a, rep.selected_b)
    err = rel(M, Mo)
    print(f"circulant n=5000 (Bluestein): rel vs oracle {err:.3e}, near-tie substitutions {subs}")
    assert err < 1e-10
