"""Config C5 at full size (n = 32768, fp32, k = 128, order 1): the cycle product on device-
generated operands (tests/devgen.py), checked through size-independent properties and an oracle
row sample (the full oracle cannot run at this n).

  * selection: the planted shifts (energy ~n each, every other cycle ~1e-6 n + O(1) circulant
    energy) -- bit-exact, ascending;
  * rows: oracle.cycle_product_rows on 1024 spread rows, rel. Frobenius <= 1e-4 over the sample and
    per row (fp32 tolerance);
  * first-order identity on a random probe x: (AB - M) x = dA (dB x), evaluated with fp64 matvecs,
    relative to ||A B x|| <= 1e-5.
"""
import os

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
    """1024 spread rows of M against oracle.cycle_product_rows (B copied to the host once; the
    oracle rows run in 32-row blocks on all host cores)."""
    from concurrent.futures import ThreadPoolExecutor
    P, A, B, JA, JB, r = c5
    rows = np.unique(np.linspace(0, N - 1, 1024).astype(int))
    assert rows.size == 1024
    Rt = torch.from_numpy(rows).cuda()
    A_rows = A[Rt].double().cpu().numpy()
    Bh = B.cpu().numpy()  # fp32, 4 GiB
    lamB = left_lambdas(B, JB).double().cpu().numpy()
    Mg = r["M"][Rt].double().cpu().numpy()

    def block(b0):
        rb = rows[b0:b0 + 32]
        return O.cycle_product_rows(rb, A_rows[b0:b0 + 32], JA, [Bh[(rb - j) % N] for j in JA], JB, lamB)

    with ThreadPoolExecutor(min(16, os.cpu_count() or 1)) as ex:
        Mo = np.concatenate(list(ex.map(block, range(0, rows.size, 32))))
    err = rel(Mg, Mo)
    row_err = np.linalg.norm(Mg - Mo, axis=1) / np.linalg.norm(Mo, axis=1)
    print(f"C5 n={N} k={K}: {rows.size} rows rel vs oracle {err:.3e}, worst row {row_err.max():.3e}")
    assert err < 1e-4
    assert row_err.max() < 1e-4


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
