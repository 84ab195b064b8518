"""Config C5 at full size (n = 32768, fp32, k = 128, order 1): the cycle product on device-
generated operands (tests/devgen.py), checked through size-independent properties and an oracle
row sample (the full oracle cannot run at this n).

  * selection: the planted shifts (energy ~n each, every other cycle ~1e-6 n + O(1) circulant
    energy) -- bit-exact, ascending;
  * rows: oracle.cycle_product_rows on 8 rows, rel. Frobenius <= 1e-4 (fp32 tolerance);
  * first-order identity on a random probe x: (AB - M) x = dA (dB x), evaluated with fp64 matvecs,
    relative to ||A B x|| <= 1e-5.
"""
import numpy as np
import pytest
import torch

import oracle as O
from conftest import rel
from devgen import c5_operand, left_lambdas

pytestmark = pytest.mark.gpu

N, K, NCYC, NCIRC = 32768, 128, 128, 32


@pytest.fixture(scope="module")
def c5():
    import paper_2504_19308_b200 as P
    A, JA = c5_operand(N, NCYC, NCIRC, seed=5, operand=0)
    B, JB = c5_operand(N, NCYC, NCIRC, seed=5, operand=1)
    r = P.cycle.cycle_product_device(A, B, K, K, 1)
    torch.cuda.synchronize()
    yield P, A, B, JA, JB, r
    del A, B, r
    torch.cuda.empty_cache()


def test_c5_selection(c5):
    P, A, B, JA, JB, r = c5
    assert r["sel_a"].tolist() == JA
    assert r["sel_b"].tolist() == JB


def test_c5_rows_vs_oracle(c5):
    P, A, B, JA, JB, r = c5
    rows = np.array([0, 1, 777, 4096, 12345, 20000, 32766, 32767])
    Rt = torch.from_numpy(rows).cuda()
    A_rows = A[Rt].double().cpu().numpy()
    B_shift = [B[(Rt - j) % N].double().cpu().numpy() for j in JA]
    lamB = left_lambdas(B, JB).double().cpu().numpy()
    Mo = O.cycle_product_rows(rows, A_rows, JA, B_shift, JB, lamB)
    Mg = r["M"][Rt].double().cpu().numpy()
    err = rel(Mg, Mo)
    print(f"C5 n={N} k={K}: rows rel vs oracle {err:.3e}")
    assert err < 1e-4


def test_c5_first_order_identity(c5):
    P, A, B, JA, JB, r = c5
    g = torch.Generator(device="cuda")
    g.manual_seed(99)
    x = torch.randn(N, generator=g, device="cuda", dtype=torch.float64)
    i = torch.arange(N, device="cuda")

    def matvec(X, v):  # fp64, row-chunked
        return torch.cat([X[s:s + 4096].double() @ v for s in range(0, N, 4096)])

    def hat_matvec(lam, J, v):  # (sum_t Lambda_t C^J_t) v = sum_t lam_t * v[(i - J_t) % n]
        out = torch.zeros_like(v)
        for t, j in enumerate(J):
            out += lam[t].double() * v[(i - int(j)) % N]
        return out

    lamA, lamB = left_lambdas(A, JA), left_lambdas(B, JB)
    Bx = matvec(B, x)
    lhs = matvec(A, Bx) - matvec(r["M"], x)
    dBx = Bx - hat_matvec(lamB, JB, x)
    rhs = matvec(A, dBx) - hat_matvec(lamA, JA, dBx)
    err = float(torch.linalg.norm(lhs - rhs) / torch.linalg.norm(matvec(A, Bx)))
    print(f"C5 first-order identity on a probe: {err:.3e}")
    assert err < 1e-5
