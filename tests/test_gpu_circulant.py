"""GPU parity: circulant path (reference circulant.py) -- golden vectors from the reference,
the reference suite's known-answer cases, and config C3 with the near-tie protocol."""
import numpy as np
import pytest

import oracle as O
from conftest import check_report, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def C():
    from paper_2504_19308_b200 import circulant as C
    return C


def near_tie_ok(sel_gpu, sel_ref, mags, ulps=8):
    """every differing pick must be within `ulps` ulp of max(m) of a pick it
    displaced. Returns the number of substitutions (raises AssertionError if not a near tie)."""
    a, b = set(sel_gpu), set(sel_ref)
    if a == b:
        return 0
    tol = ulps * np.spacing(np.max(mags))
    extra, missing = sorted(a - b), sorted(b - a)
    assert len(extra) == len(missing)
    for e, m in zip(extra, missing):
        assert abs(mags[e] - mags[m]) <= tol, (e, m, mags[e], mags[m])
    return len(extra)


@pytest.mark.parametrize("n", [2, 8, 16, 31, 32, 64, 97])
def test_circulant_golden(C, golden, n):
    g = golden("circulant")
    A, B, k = g[f"cd{n}_A"], g[f"cd{n}_B"], int(g[f"cd{n}_k"])
    spec = C.circulant_decompose(A)
    assert rel(spec.columns, g[f"cd{n}_cols"]) < 1e-12
    assert rel(spec.magnitudes, g[f"cd{n}_mags"]) < 1e-12
    sel = C.circulant_select(spec, k).selected
    near_tie_ok(sel, list(g[f"cd{n}_sel"]), g[f"cd{n}_mags"])
    # B's selection (the golden file pins A's): the oracle's, under the same near-tie protocol
    mags_b = O.circulant_decompose(B)[1]
    sel_b = O.top_indices(mags_b, k)
    for order in (0, 1):
        M, rep = C.circulant_first_order_multiply(A, B, k, order)
        ref = g[f"cd{n}_M{order}"]
        near_tie_ok(rep.selected_b, sel_b, mags_b)
        if rep.selected_a == list(g[f"cd{n}_sel"]) and rep.selected_b == sel_b:
            assert rel(M, ref) < 1e-10
            check_report(rep, g[f"cd{n}_rep{order}"], rel_tol=1e-6, abs_tol=1e-9)
        else:  # re-run the oracle with the GPU's selections forced
            Mo, _ = O.circulant_first_order_multiply(A, B, k, order, rep.selected_a, rep.selected_b)
            assert rel(M, Mo) < 1e-10
        assert M.dtype == np.complex128
        r = g[f"cd{n}_rep{order}"]
        assert rep.norm_da == pytest.approx(r[0], rel=1e-6, abs=1e-7 * np.linalg.norm(A))


def test_complex_input_and_hand_example(C, golden):
    g = golden("circulant")
    spec = C.circulant_decompose(g["cdz_A"])
    assert rel(spec.columns, g["cdz_cols"]) < 1e-12
    A = np.array([[1.0, 2.0], [3.0, 4.0]])
    spec = C.circulant_decompose(A)
    assert np.allclose(spec.columns[0], [2.5, 2.5], atol=1e-12)
    assert np.allclose(spec.columns[1], [-1.5, 0.5], atol=1e-12)
    assert np.allclose(C.circulant_materialize(spec).real, A, atol=1e-12)
    assert 2 * np.sum(spec.magnitudes ** 2) == pytest.approx(30.0, rel=1e-12)
    kept = C.circulant_select(spec, 1)
    assert kept.selected == [0]
    assert np.allclose(C.circulant_materialize(kept).real, np.full((2, 2), 2.5), atol=1e-12)


def test_top_indices_ties(C):
    assert C.top_indices([1.0, 3.0, 3.0, 2.0], 2) == [1, 2]
    assert C.top_indices([1.0, 3.0, 3.0, 2.0], 3) == [1, 2, 3]
    assert C.top_indices([5.0, 5.0, 5.0], 1) == [0]
    assert C.top_indices([1.0], 0) == []
    assert C.top_indices([-1.0, -3.0, 0.0, -0.0, 2.0], 3) == O.top_indices([-1.0, -3.0, 0.0, -0.0, 2.0], 3)
    with pytest.raises(ValueError):
        C.top_indices([1.0, 2.0], 3)


def test_component_and_orthogonality(C):
    rng = np.random.default_rng(0)
    A = rng.standard_normal((16, 16))
    spec = C.circulant_decompose(A)
    for k in range(16):
        assert np.linalg.norm(C.circulant_component(A, k) - spec.columns[k]) < 1e-10
    assert rel(C.circulant_materialize(spec), A) < 1e-10
    with pytest.raises(ValueError):
        C.circulant_component(np.eye(4), 4)


@pytest.mark.parametrize("n", [8, 16, 31, 32, 128, 256])
def test_optimized_equals_materialized(C, n):
    rng = np.random.default_rng(4 + n)
    A = rng.standard_normal((n, n))
    B = rng.standard_normal((n, n))
    k = 6
    M1, rep = C.circulant_first_order_multiply(A, B, k, 1)
    Mo, ro = O.circulant_first_order_multiply(A, B, k, 1, rep.selected_a, rep.selected_b)
    assert rel(M1, Mo) < 1e-10
    near_tie_ok(rep.selected_a, ro["selected_a"] if False else O.top_indices(ro["magnitudes_a"], k),
                ro["magnitudes_a"])


def test_c3_config(C):
    """Config C3: fp64 n=4096, 16 diag(d)Circ(c) terms + noise, k=16, order 1 (near-tie protocol)."""
    n, k = 4096, 16
    A = O.gen_circulant_operand(n, 16, 0)
    B = O.gen_circulant_operand(n, 16, 1)
    M, rep = C.circulant_first_order_multiply(A, B, k, 1)
    Mo, ro = O.circulant_first_order_multiply(A, B, k, 1)
    subs = near_tie_ok(rep.selected_a, ro["selected_a"], ro["magnitudes_a"])
    subs += near_tie_ok(rep.selected_b, ro["selected_b"], ro["magnitudes_b"])
    if subs:
        Mo, ro = O.circulant_first_order_multiply(A, B, k, 1, rep.selected_a, rep.selected_b)
    assert rel(M, Mo) < 1e-10
    print(f"C3: near-tie substitutions {subs}; rel err vs exact {rel(M, A @ B):.3e}")


def test_validation(C):
    A = np.ones((4, 4))
    with pytest.raises(ValueError):
        C.circulant_first_order_multiply(np.ones((3, 4)), A, 1, 0)
    with pytest.raises(ValueError):
        C.circulant_first_order_multiply(A, np.ones((5, 5)), 1, 0)
    with pytest.raises(ValueError):
        C.circulant_first_order_multiply(A, A, 5, 0)
    with pytest.raises(ValueError):
        C.circulant_first_order_multiply(A, A, 1, 2)


@pytest.mark.parametrize("n", [64, 256, 97])
def test_complex_operands_product(C, n):
    """Complex A, B (accepted by the reference, circulant.py:73-91 / core.py:38-41): the row and
    column kernels take their unpacked branch (no real-pair packing) -- checked against the oracle
    under the near-tie protocol."""
    rng = np.random.default_rng(n + 5)
    A = O.gen_circulant_operand(n, 4, 21 + n) + 1j * O.gen_circulant_operand(n, 4, 22 + n)
    B = O.gen_circulant_operand(n, 4, 23 + n) + 1j * rng.standard_normal((n, n)) * 1e-3
    for order in (0, 1):
        M, rep = C.circulant_first_order_multiply(A, B, 5, order)
        Mo, ro = O.circulant_first_order_multiply(A, B, 5, order)
        subs = near_tie_ok(rep.selected_a, ro["selected_a"], ro["magnitudes_a"])
        subs += near_tie_ok(rep.selected_b, ro["selected_b"], ro["magnitudes_b"])
        if subs:
            Mo, ro = O.circulant_first_order_multiply(A, B, 5, order, force_sel_a=rep.selected_a,
                                                      force_sel_b=rep.selected_b)
        assert rel(M, Mo) < 1e-10
