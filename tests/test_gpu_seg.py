"""Segmented right gather (cycle.cu K11s): the large-n path, where a whole row fits shared memory
at most twice and the CTA sweeps column segments of R rows instead (fp64 n > 5120, fp32
n > 12800 at k <= 128; both sizes below are past those limits and multiples of 512).

  * fp64 n = 6144 and fp32 n = 16384 (last row block ragged: 16384 = 6 * 2730 + 4), order 1 and
    order 0, on C5-style operands (dense noise + planted cycles + circulant terms): the full
    product against a dense torch fp64 reference built from the device selection (materialised
    cycle sums, two fp64 GEMMs), and a row sample against oracle.cycle_product_rows;
  * the selection equals the planted shifts (bit-exact, ascending);
  * ||M||_F from the kernel's fused per-block partials matches the product.
"""
import numpy as np
import pytest
import torch

import oracle as O
from conftest import rel
from devgen import c5_operand, left_lambdas

pytestmark = pytest.mark.gpu


def _hat(X, J):
    """Dense sum_t Lambda_t C^J_t of X's cycles J (left layout, core.py:123-124): entries
    X[i, (i - j) % n] kept, everything else zero."""
    n = X.shape[0]
    i = torch.arange(n, device=X.device)
    H = torch.zeros_like(X)
    for j in J:
        c = (i - int(j)) % n
        H[i, c] = X[i, c]
    return H


@pytest.mark.parametrize("n,dtype,k,order", [
    (6144, torch.float64, 32, 1),
    (6144, torch.float64, 32, 0),
    (16384, torch.float32, 64, 1),
])
def test_segmented_cycle_product(n, dtype, k, order):
    import paper_2504_19308_b200 as P
    from paper_2504_19308_b200 import _native as N
    A, JA = c5_operand(n, k, 8, seed=11, operand=0, dtype=dtype)
    B, JB = c5_operand(n, k, 8, seed=11, operand=1, dtype=dtype)
    r = P.cycle.cycle_product_device(A, B, k, k, order)
    torch.cuda.synchronize()
    assert r["sel_a"].tolist() == JA
    assert r["sel_b"].tolist() == JB
    Ad, Bd = A.double(), B.double()
    Ah, Bh = _hat(Ad, JA), _hat(Bd, JB)
    ref = Ah @ Bd + (Ad - Ah) @ Bh if order == 1 else Ah @ Bh
    M = r["M"].double()
    err = float(torch.linalg.norm(M - ref) / torch.linalg.norm(ref))
    tol = 1e-10 if dtype == torch.float64 else 1e-4
    print(f"segmented gather n={n} {dtype} k={k} order={order}: rel vs torch fp64 {err:.3e}")
    assert err < tol
    # ||M||^2 from the gather's fused partials (order 1: the segmented pass writes M last)
    fro_m = float(r["scalars"][N.S_FRO2_M].item()) ** 0.5
    assert abs(fro_m - float(torch.linalg.norm(M))) <= 1e-6 * float(torch.linalg.norm(M))
    if order == 1:
        rows = np.array([0, 1, 5, n // 2 + 3, n - 5, n - 1])
        Rt = torch.from_numpy(rows).cuda()
        A_rows = A[Rt].double().cpu().numpy()
        B_shift = [B[(Rt - j) % n].double().cpu().numpy() for j in JA]
        lamB = left_lambdas(B, JB).double().cpu().numpy()
        Mo = O.cycle_product_rows(rows, A_rows, JA, B_shift, JB, lamB)
        err_o = rel(M[Rt].cpu().numpy(), Mo)
        print(f"  rows vs oracle {err_o:.3e}")
        assert err_o < tol
