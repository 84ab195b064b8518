"""GPU parity: cycle-truncated product (config C2) through the C-ABI vs the CPU oracle.

Bar: selected cycle indices bit-exact; values rel. Frobenius <= 1e-10 (fp64) / 1e-4 (fp32)
against the oracle's approximation (north_star tolerance)."""
import numpy as np
import pytest
import torch

import oracle as O
from conftest import rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2504_19308_b200 as P
    return P


@pytest.mark.parametrize("tag", ["cy16_3_3", "cy31_4_5", "cy64_8_8", "cy64_6_10"])
@pytest.mark.parametrize("order", [0, 1])
def test_cycle_golden(P, golden, tag, order):
    g = golden("cycle")
    ka, kb = int(tag.split("_")[1]), int(tag.split("_")[2])
    M, rep = P.cycle_first_order_multiply(g[tag + "_A"], g[tag + "_B"], ka, order, k_b=kb)
    assert rep.selected_a == list(g[tag + "_Ja"])
    assert rep.selected_b == list(g[tag + "_Jb"])
    assert rel(M, g[tag + f"_M{order}"]) < 1e-12
    assert M.dtype == np.float64


@pytest.mark.parametrize("n,k,kb", [(1, 1, 1), (2, 1, 2), (3, 0, 3), (7, 7, 0), (100, 5, 9),
                                    (257, 12, 3), (512, 16, 16), (1000, 24, 8)])
@pytest.mark.parametrize("order", [0, 1])
def test_cycle_vs_oracle(P, n, k, kb, order):
    A = O.gen_cycle_operand(n, min(n, 2 * k + 1), 11 * n + k)
    B = O.gen_cycle_operand(n, min(n, 2 * kb + 1), 13 * n + kb)
    M, rep = P.cycle_first_order_multiply(A, B, k, order, k_b=kb)
    Mo, ro = O.cycle_first_order_multiply(A, B, k, order, kb=kb)
    assert rep.selected_a == ro["selected_a"]
    assert rep.selected_b == ro["selected_b"]
    if np.linalg.norm(Mo) > 0:
        assert rel(M, Mo) < 1e-10
    else:
        assert np.linalg.norm(M) == 0
    # energy-difference residuals carry sqrt(eps)*||A|| noise (circulant.py:130-133)
    tol_a = 1e-7 * np.linalg.norm(A)
    tol_b = 1e-7 * np.linalg.norm(B)
    assert rep.norm_da == pytest.approx(ro["norm_da"], rel=1e-6, abs=tol_a)
    assert rep.norm_db == pytest.approx(ro["norm_db"], rel=1e-6, abs=tol_b)
    if ro["posterior_estimate"] is not None and ro["norm_da"] > tol_a and ro["norm_db"] > tol_b:
        assert rep.posterior_estimate == pytest.approx(ro["posterior_estimate"], rel=1e-8)


def test_cycle_ties_lower_index(P):
    # two cycles of identical energy: the lower shift must win (circulant.py:63-70)
    n = 8
    A = np.zeros((n, n))
    i = np.arange(n)
    A[i, (i - 2) % n] = 1.0
    A[i, (i - 5) % n] = -1.0
    A[i, (i - 6) % n] = 0.5
    M, rep = P.cycle_first_order_multiply(A, np.eye(n), 1, 1)
    assert rep.selected_a == [2]


def test_c2_config_fp64(P):
    """Config C2: fp64, n=2048, 32 dominant cycles per operand, k=32, order 1."""
    n, k = 2048, 32
    A = O.gen_cycle_operand(n, 32, 0)
    B = O.gen_cycle_operand(n, 32, 1)
    M, rep = P.cycle_first_order_multiply(A, B, k, 1)
    Mo, ro = O.cycle_first_order_multiply(A, B, k, 1)
    assert rep.selected_a == ro["selected_a"] and rep.selected_b == ro["selected_b"]
    assert rel(M, Mo) < 1e-10
    exact = A @ B
    err_gpu, err_cpu = rel(M, exact), rel(Mo, exact)
    assert err_gpu == pytest.approx(err_cpu, rel=1e-6)
    print(f"C2 rel err vs exact AB: gpu {err_gpu:.3e} oracle {err_cpu:.3e}")


def test_fp32_device_path(P):
    """fp32 device tensors in, fp32 out; oracle in fp64 on the same fp32-representable inputs."""
    n, k = 1024, 16
    A = O.gen_cycle_operand(n, 16, 5).astype(np.float32)
    B = O.gen_cycle_operand(n, 16, 6).astype(np.float32)
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    M, rep = P.cycle_first_order_multiply(Ad, Bd, k, 1)
    assert M.is_cuda and M.dtype == torch.float32
    Mo, ro = O.cycle_first_order_multiply(A.astype(np.float64), B.astype(np.float64), k, 1)
    assert rep.selected_a == ro["selected_a"]
    assert rel(M.cpu().numpy(), Mo) < 1e-4


def test_first_order_identity_large(P):
    """Size-independent property at n=4096: AB - M = dA.dB (checked on a row sample)."""
    n, k = 4096, 16
    A = O.gen_cycle_operand(n, 16, 21)
    B = O.gen_cycle_operand(n, 16, 22)
    M, rep = P.cycle_first_order_multiply(A, B, k, 1)
    dA = A.copy()
    dB = B.copy()
    i = np.arange(n)
    for j in rep.selected_a:
        dA[i, (i - j) % n] = 0.0
    for j in rep.selected_b:
        dB[i, (i - j) % n] = 0.0
    rows = np.arange(0, n, 61)
    gap = A[rows] @ B - M[rows]
    assert np.linalg.norm(gap - dA[rows] @ dB) < 1e-10 * np.linalg.norm(A[rows] @ B)


def test_validation_errors(P):
    with pytest.raises(ValueError):
        P.cycle_first_order_multiply(np.ones((3, 4)), np.ones((4, 4)), 1, 1)
    with pytest.raises(ValueError):
        P.cycle_first_order_multiply(np.ones((4, 4)), np.ones((4, 4)), 5, 1)
    with pytest.raises(ValueError):
        P.cycle_first_order_multiply(np.ones((4, 4)), np.ones((4, 4)), 1, 2)
    with pytest.raises(ValueError):
        P.cycle_first_order_multiply([[np.nan, 1.0], [1.0, 1.0]], np.ones((2, 2)), 1, 1)


@pytest.mark.parametrize("order", [0, 1])
def test_cycle_transposed_left_fp64(P, order):
    """n = 4096 fp64: Ahat . X runs as (X^T Ahat^T)^T through the row-block gather (the column
    strip of the left gather would be 2 columns wide); full oracle comparison at 1e-10."""
    n, k = 4096, 12
    A = O.gen_cycle_operand(n, 2 * k, 71)
    B = O.gen_cycle_operand(n, 2 * k, 72)
    M, rep = P.cycle_first_order_multiply(A, B, k, order)
    rows = np.array([0, 1, 100, 2047, 4095])
    Ja, la_, _, _, _ = O.cycle_decompose(A, k)
    Jb, lb_, _, _, _ = O.cycle_decompose(B, k)
    assert rep.selected_a == Ja and rep.selected_b == Jb
    if order == 1:
        Mo = O.cycle_product_rows(rows, A[rows], Ja, [B[(rows - j) % n] for j in Ja], Jb, lb_)
    else:
        Mo = O.apx_oracle._cycle_left_apply(Ja, la_, O.cycle_materialize(Jb, lb_, n), rows=rows)
    assert rel(M[rows], Mo) < 1e-10
