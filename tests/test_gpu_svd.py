"""GPU parity for the randomized-SVD path (reference svd.py) -- golden vectors from the
reference, the reference test suite's known-answer cases (test_svd.py), and config C1."""
import numpy as np
import pytest

import oracle as O
from conftest import check_report, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    from paper_2504_19308_b200 import svd as S
    return S


@pytest.mark.parametrize("tag", ["svd16_1_0", "svd32_2_1", "svd64_1_0", "svd64_2_2"])
def test_svd_product_golden(S, golden, tag):
    g = golden("svd")
    n, s, q, seed = (int(v) for v in g[tag + "_par"])
    for order in (0, 1):
        M, rep = S.svd_first_order_multiply(g[tag + "_A"], g[tag + "_B"], s, order, seed, power_iterations=q)
        assert rel(M, g[tag + f"_M{order}"]) < 1e-10
        r = g[tag + f"_rep{order}"]
        assert rep.norm_da == pytest.approx(r[0], rel=1e-6, abs=1e-7 * np.linalg.norm(g[tag + "_A"]))
        assert rep.k == int(r[4])
        check_report(rep, r, rel_tol=1e-6, abs_tol=1e-7)  # apriori / posterior estimates


@pytest.mark.parametrize("tag", ["svd16_1_0", "svd32_2_1", "svd64_1_0", "svd64_2_2"])
def test_rsvd_factors_golden(S, golden, tag):
    g = golden("svd")
    n, s, q, seed = (int(v) for v in g[tag + "_par"])
    d = S.randomized_partial_svd(g[tag + "_A"], s, seed, power_iterations=q)
    assert rel(d.sigma, g[tag + "_S"]) < 1e-10
    # singular vectors agree up to column signs
    assert rel(np.abs(d.U), np.abs(g[tag + "_U"])) < 1e-8
    assert rel(np.abs(d.V), np.abs(g[tag + "_V"])) < 1e-8


def test_c1_oversampled_composition(S, golden):
    """Config C1 composition (k=8, p=4, q=2 at n=64 golden; full size below)."""
    g = golden("svd")
    n, k, p, q, t = (int(v) for v in g["c1_par"])
    M, rep = S.svd_first_order_multiply(g["c1_A"], g["c1_B"], None, 0, t, power_iterations=q,
                                        components=k, oversampling=p)
    assert rel(M, g["c1_M"]) < 1e-10
    assert rep.norm_da == pytest.approx(g["c1_nd"][0], rel=1e-8)


def test_c1_config_n512(S):
    """C1: fp64 n=512, sigma_i = 0.9^i Haar operands, k=32, p=8, q=2, order 0."""
    n = 512
    sig = 0.9 ** np.arange(n)
    A = O.gen_haar_spectrum(n, sig, 2)
    B = O.gen_haar_spectrum(n, sig, 3)
    M, rep = S.svd_first_order_multiply(A, B, None, 0, 1, power_iterations=2, components=32, oversampling=8)
    Mo, ro = O.svd_first_order_multiply(A, B, None, 0, 1, power_iterations=2, components=32, oversampling=8)
    assert rel(M, Mo) < 1e-10
    print(f"C1 rel err vs exact AB: {rel(M, A @ B):.3e}")


# ---- known-answer cases of the reference suite (test_svd.py) ----
def test_qr_kats(S):
    Q, R = S.qr_decompose(np.array([[3.0], [4.0]]))
    assert abs(R[0, 0]) == pytest.approx(5.0)
    assert np.allclose(np.abs(Q[:, 0]), [0.6, 0.8], atol=1e-15)
    rng = np.random.default_rng(1)
    Y = rng.standard_normal((20, 5))
    Q, R = S.qr_decompose(Y)
    assert np.linalg.norm(Q @ R - Y) / np.linalg.norm(Y) < 1e-12
    assert np.allclose(Q.T @ Q, np.eye(5), atol=1e-12)
    assert np.array_equal(R, np.triu(R))
    Qr, Rr = np.linalg.qr(Y)
    assert np.allclose(Q, Qr, atol=1e-12) and np.allclose(R, Rr, atol=1e-12)  # LAPACK signs
    with pytest.raises(ValueError):
        S.qr_decompose(np.ones((3, 5)))


def test_rank_one_captured_exactly(S):
    rng = np.random.default_rng(2)
    u, v = rng.standard_normal(64), rng.standard_normal(64)
    d = S.randomized_partial_svd(np.outer(u, v), 1, seed=3)
    assert d.sigma[0] == pytest.approx(np.linalg.norm(u) * np.linalg.norm(v), rel=1e-8)
    assert np.all(d.sigma[1:] < 1e-8)
    assert S.svd_residual_norm(d) < 1e-8 * d.sigma[0]
    assert np.allclose(d.U.T @ d.U, np.eye(d.k), atol=1e-10)


def test_diagonal_and_zero(S):
    diag = np.maximum(5.0 - np.arange(64), 0.0)
    d = S.randomized_partial_svd(np.diag(diag), 2, seed=4)
    assert np.allclose(d.sigma[:5], [5.0, 4.0, 3.0, 2.0, 1.0], atol=1e-6)
    z = S.randomized_partial_svd(np.zeros((16, 16)), 1, seed=0)
    assert np.all(z.sigma == 0.0)
    assert S.svd_residual_norm(z) == 0.0


def test_factor_invariants_and_reproducibility(S):
    rng = np.random.default_rng(5)
    A = rng.standard_normal((40, 40))
    d = S.randomized_partial_svd(A, 2, seed=6)
    k = d.k
    assert np.allclose(d.U.T @ d.U, np.eye(k), atol=1e-10)
    assert np.allclose(d.V.T @ d.V, np.eye(k), atol=1e-10)
    assert np.all(np.diff(d.sigma) <= 0) and np.all(d.sigma >= 0)
    d2 = S.randomized_partial_svd(A, 2, seed=6)
    assert np.array_equal(d.U, d2.U) and np.array_equal(d.sigma, d2.sigma) and np.array_equal(d.V, d2.V)
    assert np.allclose(S.svd_reconstruct(d), (d.U * d.sigma) @ d.V.T, atol=1e-12)


def test_multiply_exact_cases_and_identity(S):
    rng = np.random.default_rng(8)
    A = np.outer(rng.standard_normal(64), rng.standard_normal(64))
    B = rng.standard_normal((64, 64))
    M, rep = S.svd_first_order_multiply(A, B, 1, 1, seed=9)
    assert rel(M, A @ B) < 1e-8 and rep.norm_da < 1e-7 * np.linalg.norm(A)
    A = rng.standard_normal((64, 64))
    B = rng.standard_normal((64, 3)) @ rng.standard_normal((3, 64))
    M, _ = S.svd_first_order_multiply(A, B, 1, 1, seed=11)
    assert rel(M, A @ B) < 1e-8


def test_rectangular_and_errors(S):
    rng = np.random.default_rng(3)
    A = rng.standard_normal((30, 48))
    B = rng.standard_normal((48, 20))
    for order in (0, 1):
        M, rep = S.svd_first_order_multiply(A, B, 1, order, seed=4)
        Mo, ro = O.svd_first_order_multiply(A, B, 1, order, 4)
        assert rel(M, Mo) < 1e-10 and rep.k == ro["k"]
    with pytest.raises(ValueError):
        S.svd_first_order_multiply(np.ones((4, 4)), np.ones((5, 5)), 1, 1, seed=0)
    with pytest.raises(ValueError):
        S.svd_first_order_multiply(np.ones((4, 4)), np.ones((4, 4)), 1, 2, seed=0)
    with pytest.raises(ValueError):
        S.randomized_partial_svd(np.ones((4, 4)).astype(complex), 1, seed=0)
    with pytest.raises(ValueError):
        S.randomized_partial_svd(np.ones((4, 4)), 1, seed=0, power_iterations=-1)
    with pytest.raises(ValueError):
        S.randomized_partial_svd(np.ones((4, 4)), 1, seed=0, components=0)


def test_wide_sketch_crit4c_shape(S):
    """Sketch width > 128: the reference's crit 4c input shape (n=700, s=60 -> k=541,
    pkg/tests/test_acceptance.py:187-198). Householder QR + global-memory Jacobi SVD."""
    n, s = 700, 60
    assert S.component_count(n, s) == 541
    rng = np.random.default_rng(7)
    A = rng.standard_normal((n, n)) * np.exp(-np.arange(n) / 50.0)[None, :]
    d = S.randomized_partial_svd(A, s, 3)
    do = O.rsvd(A, 541, np.random.default_rng(3))
    assert d.k == 541
    assert rel(d.sigma, do[1]) < 1e-10
    rec = (d.U * d.sigma) @ d.V.T
    reco = (do[0] * do[1]) @ do[2].T
    assert rel(rec, reco) < 1e-9
    assert np.allclose(d.U.T @ d.U, np.eye(541), atol=1e-10)
    for order in (0, 1):
        M, rep = S.svd_first_order_multiply(A, A, s, order, 2)
        Mo, ro = O.svd_first_order_multiply(A, A, s, order, 2)
        assert rel(M, Mo) < 1e-10
        assert rep.k == 541


def test_wide_sketch_qr(S):
    rng = np.random.default_rng(8)
    Y = rng.standard_normal((400, 200))
    Q, R = S.qr_decompose(Y)
    Qn, Rn = np.linalg.qr(Y)
    assert rel(Q, Qn) < 1e-10 and rel(R, Rn) < 1e-10
