"""GPU parity for the Fourier-sparsified path (reference fsparse.py) against golden vectors and
the oracle. Rows of A W* for real A are conjugate-symmetric, so |At[i,j]| and |At[i,n-j]| are
exact ties in exact arithmetic that pocketfft breaks at the ulp level: when the GPU's picks
differ, each differing pick must be a near tie and the oracle is re-run with
the GPU's selections forced, as the reference tests do with `spec.selected`."""
import numpy as np
import pytest

import oracle as O
from conftest import check_report, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def F():
    from paper_2504_19308_b200 import fsparse as F
    return F


def check_near_ties(sel_gpu, sel_ref, X, ulps=8):
    subs = 0
    for i, (a, b) in enumerate(zip(sel_gpu, sel_ref)):
        a, b = set(a), set(b)
        if a == b:
            continue
        mags = np.abs(X[i])
        tol = ulps * np.spacing(np.max(mags))
        for e, m in zip(sorted(a - b), sorted(b - a)):
            assert abs(mags[e] - mags[m]) <= tol, (i, e, m)
            subs += 1
    return subs


def parity(F, A, B, k, order, mode, ref=None):
    M, rep = F.fft_sparse_first_order_multiply(A, B, k, order, mode)
    Mo, ro = O.fft_sparse_first_order_multiply(A, B, k, order, mode)
    subs = check_near_ties(rep.selected_a, ro["selected_a"], ro["At"])
    Xb = ro["Bt"] if mode == "rows" else ro["Bt"].T
    subs += check_near_ties(rep.selected_b, ro["selected_b"], Xb)
    if subs:
        Mo, ro = O.fft_sparse_first_order_multiply(A, B, k, order, mode, rep.selected_a, rep.selected_b)
    elif ref is not None:
        Mo = ref
    if np.linalg.norm(Mo) > 0:
        assert rel(M, Mo) < 1e-10, (order, mode, subs)
    else:
        assert np.linalg.norm(M) < 1e-12
    return rep, ro, subs


@pytest.mark.parametrize("tag", ["sq16", "sq32", "rect", "full", "zero"])
def test_sfft_golden(F, golden, tag):
    g = golden("fsparse")
    A, B, k = g[tag + "_A"], g[tag + "_B"], int(g[tag + "_k"])
    for order in (0, 1):
        for mode in ("rows", "cols"):
            rep, ro, subs = parity(F, A, B, k, order, mode, g[f"{tag}_M{order}{mode}"])
            if subs == 0:
                r = g[f"{tag}_rep{order}{mode}"]
                assert rep.norm_da == pytest.approx(r[0], rel=1e-9, abs=1e-12)
                assert rep.norm_db == pytest.approx(r[1], rel=1e-9, abs=1e-12)
                check_report(rep, r, rel_tol=1e-9, abs_tol=1e-12)


def test_topk_sparsify_golden(F, golden):
    g = golden("fsparse")
    for k in range(6):
        S = F.topk_sparsify(g["tk_T"], k)
        assert np.array_equal(S.to_dense(), g[f"tk_{k}"])
    S = F.topk_sparsify(g["tk_T"], [1, 3])
    assert [len(r) for r in S.entries] == [1, 3]
    with pytest.raises(ValueError):
        F.topk_sparsify(g["tk_T"], [1])


def test_sparse_dense_both_sides(F):
    rng = np.random.default_rng(3)
    M = rng.standard_normal((6, 9)) + 1j * rng.standard_normal((6, 9))
    S = F.topk_sparsify(M, 3)
    X = rng.standard_normal((9, 4))
    Y = rng.standard_normal((5, 6))
    assert np.allclose(F.sparse_dense_multiply(S, X, "left"), S.to_dense() @ X, atol=1e-12)
    assert np.allclose(F.sparse_dense_multiply(S, Y, "right"), Y @ S.to_dense(), atol=1e-12)
    with pytest.raises(ValueError):
        F.sparse_dense_multiply(S, X, "middle")


@pytest.mark.parametrize("mode", ["rows", "cols"])
def test_sfft_vs_oracle_n256(F, mode):
    rng = np.random.default_rng(11)
    A = rng.standard_normal((256, 256))
    B = rng.standard_normal((256, 256))
    for order in (0, 1):
        parity(F, A, B, 16, order, mode)


@pytest.mark.parametrize("k", [257, 700])
@pytest.mark.parametrize("mode", ["rows", "cols"])
def test_sfft_wide_k(F, k, mode):
    """k > 256 kept entries per row (the sparse row gather stages its entries in 256-wide tiles;
    the reference has no k limit, fsparse.py:168-240)."""
    rng = np.random.default_rng(100 + k)
    A = rng.standard_normal((1024, 1024))
    B = rng.standard_normal((1024, 1024))
    for order in (0, 1):
        parity(F, A, B, k, order, mode)


def test_sparse_dense_right_dense_column(F):
    """B @ S where one column of S is kept by > 256 rows: the transposed bucket has > 256 entries
    (fsparse.py:158-164 has no limit)."""
    rng = np.random.default_rng(5)
    M = rng.standard_normal((300, 40)) + 1j * rng.standard_normal((300, 40))
    M[:, 7] *= 1e3
    S = F.topk_sparsify(M, 3)
    assert sum(1 for row in S.entries for j, _ in row if j == 7) == 300
    Y = rng.standard_normal((9, 300))
    assert np.allclose(F.sparse_dense_multiply(S, Y, "right"), Y @ S.to_dense(), rtol=0, atol=1e-9)
    X = rng.standard_normal((40, 5))
    assert np.allclose(F.sparse_dense_multiply(S, X, "left"), S.to_dense() @ X, rtol=0, atol=1e-9)


@pytest.mark.parametrize("tag", ["real", "cplx", "n1", "const", "odd"])
def test_fourier_row_decompose_golden(F, golden, tag):
    """fsparse.py:92-105 on the device vs the reference's own output (weights, directions,
    zero directions where the weight vanishes)."""
    g = golden("fsparse")
    spec = F.fourier_row_decompose(g[f"frs_{tag}_A"])
    assert np.allclose(spec.weights, g[f"frs_{tag}_w"], rtol=1e-12, atol=1e-13)
    assert np.allclose(spec.directions, g[f"frs_{tag}_d"], rtol=1e-12, atol=1e-13)
    assert spec.directions.dtype == np.complex128


def test_fourier_row_decompose_vs_oracle_large(F):
    rng = np.random.default_rng(12)
    A = rng.standard_normal((300, 1024))
    spec = F.fourier_row_decompose(A)
    w, d = O.fourier_row_decompose(A)
    assert rel(spec.weights, w) < 1e-12 and rel(spec.directions, d) < 1e-12
    assert np.sum(spec.weights ** 2) == pytest.approx(np.sum(A ** 2), rel=1e-12)
