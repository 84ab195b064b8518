"""Config C4 at the headline size (n = 8192, fp32, rSVD rank 64 x 64 cycles, order 1) on the
bench's synthetic operands (bench.gen_c4): oracle parity over ALL 8192 rows (the oracle's
row-blocked evaluation, ~15 s of host time) and the first-order identity on a random probe.

  * selection of B's cycles: bit-exact vs the oracle;
  * every output row vs oracle.mixed_first_order_multiply: rel. Frobenius <= 1e-4 over the whole
    matrix, and the worst single row reported (and bounded);
  * (AB - M) x = dA (dB x) with the oracle's factors (fp64 matvecs), relative to ||ABx|| <= 1e-4.
"""
import numpy as np
import pytest
import torch

import oracle as O
from conftest import rel

pytestmark = pytest.mark.gpu

N, K, SEED = 8192, 64, 7


@pytest.fixture(scope="module")
def c4():
    import bench
    import paper_2504_19308_b200 as P
    A, B = bench.gen_c4(N, 1234, torch.device("cuda", 0))
    M, rep = P.mixed_first_order_multiply(A, B, K, K, 1, SEED)
    torch.cuda.synchronize()
    A64, B64 = A.double().cpu().numpy(), B.double().cpu().numpy()
    yield A, B, M, rep, A64, B64
    del A, B, M
    torch.cuda.empty_cache()


def test_c4_full_matrix_and_selection(c4):
    A, B, M, rep, A64, B64 = c4
    Mo, ro = O.mixed_first_order_multiply(A64, B64, K, K, 1, SEED)
    assert rep.selected_b == ro["selected_b"]
    Mg = M.double().cpu().numpy()
    err = rel(Mg, Mo)
    row_err = np.linalg.norm(Mg - Mo, axis=1) / np.linalg.norm(Mo, axis=1)
    print(f"C4 n={N}: all {N} rows rel vs oracle {err:.3e}; worst row {row_err.max():.3e} "
          f"(row {int(row_err.argmax())}); rel vs exact AB {rel(Mg, A64 @ B64):.3e}")
    assert err < 1e-4
    assert row_err.max() < 1e-4  # every row within the fp32 tolerance
    assert rep.norm_db == pytest.approx(ro["norm_db"], rel=1e-5)
    # ||dA||^2 is 3.6e-4 of ||A||^2 here: the TF32 range finder's subspace (the 3e-5 of M above)
    # moves it by ~10%; the truncation bias of Q^T A (which doubled it) is removed by rounding
    assert rep.norm_da == pytest.approx(ro["norm_da"], rel=0.15)
    assert rep.apriori_estimate == pytest.approx(ro["apriori_estimate"], rel=0.15)
    assert rep.posterior_estimate == pytest.approx(ro["posterior_estimate"], rel=0.15)


def test_c4_first_order_identity(c4):
    A, B, M, rep, A64, B64 = c4
    U, s, V, _ = O.rsvd(A64, K, np.random.default_rng([SEED, 0]), 0)
    Jb, lamB, _, _, _ = O.cycle_decompose(B64, K, force_sel=rep.selected_b)
    x = np.random.default_rng(11).standard_normal(N)
    i = np.arange(N)
    Bx = B64 @ x
    Bhat_x = sum(lamB[t] * x[(i - j) % N] for t, j in enumerate(Jb))
    dBx = Bx - Bhat_x
    dA_dBx = A64 @ dBx - U @ (s * (V.T @ dBx))
    lhs = A64 @ Bx - (M.double() @ torch.from_numpy(x).cuda()).cpu().numpy()
    err = float(np.linalg.norm(lhs - dA_dBx) / np.linalg.norm(A64 @ Bx))
    print(f"C4 first-order identity on a probe: {err:.3e}")
    assert err < 1e-4
