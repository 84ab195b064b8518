"""Pin the CPU oracle against the reference's own outputs (tests/golden/*.npz).

Tolerances: index lists and permutations bit-exact; values 1e-12 relative (the oracle reuses the
same numpy routines, so most agree to the last bit; the cycle/mixed compositions sum in a
different order).
"""
import numpy as np
import pytest

import oracle as O
from oracle import apx_oracle as OX
from conftest import rel


def test_cycle_layout_golden(golden):
    g = golden("core")
    assert np.array_equal(O.cycle_reorder(g["cr_A4"], "right"), g["cr_right_A4"])
    assert np.array_equal(O.cycle_reorder(g["cr_A4"], "left"), g["cr_left_A4"])
    for n in (1, 5, 7, 33):
        A = g[f"cr_A{n}r"]
        for side in ("right", "left"):
            lay = O.cycle_reorder(A, side)
            assert np.array_equal(lay, g[f"cr_{side}_A{n}r"])
            assert np.array_equal(O.cycle_reorder_inverse(lay, side), A)


def test_apply_cycle_power_golden(golden):
    g = golden("core")
    for k in (0, 1, 5):
        assert np.array_equal(O.apply_cycle_power(g["acp_M"], k, "left"), g[f"acp_left_{k}"])
        assert np.array_equal(O.apply_cycle_power(g["acp_M"], k, "right"), g[f"acp_right_{k}"])
    with pytest.raises(ValueError):
        O.apply_cycle_power(g["acp_M"], 6, "left")


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 7, 8, 16, 31, 64, 97, 128, 700])
def test_dft_golden(golden, n):
    g = golden("core")
    x = g[f"dft_x{n}"]
    assert rel(O.unitary_dft(x, "forward", 0), g[f"dft_fwd{n}"]) < 1e-14
    assert rel(O.unitary_dft(x, "inverse", 0), g[f"dft_inv{n}"]) < 1e-14


def test_top_indices_golden(golden):
    g = golden("core")
    for k in range(9):
        assert O.top_indices(g["ti_w"], k) == list(g[f"ti_{k}"])
    assert O.top_indices([5.0, 5.0, 5.0], 1) == [0]
    with pytest.raises(ValueError):
        O.top_indices([1.0], 2)


@pytest.mark.parametrize("n", [2, 8, 16, 31, 32, 64, 97])
def test_circulant_golden(golden, n):
    g = golden("circulant")
    A, B, k = g[f"cd{n}_A"], g[f"cd{n}_B"], int(g[f"cd{n}_k"])
    S, m = O.circulant_decompose(A)
    assert rel(S, g[f"cd{n}_cols"]) < 1e-13
    assert rel(m, g[f"cd{n}_mags"]) < 1e-13
    sel = O.top_indices(m, k)
    assert sel == list(g[f"cd{n}_sel"])
    assert rel(O.circulant_materialize(S, sel), g[f"cd{n}_mat"]) < 1e-12
    for order in (0, 1):
        M, rep = O.circulant_first_order_multiply(A, B, k, order)
        assert rel(M, g[f"cd{n}_M{order}"]) < 1e-12
        r = g[f"cd{n}_rep{order}"]
        assert rep["norm_da"] == pytest.approx(r[0], rel=1e-9, abs=1e-12)
        assert rep["norm_db"] == pytest.approx(r[1], rel=1e-9, abs=1e-12)


def test_circulant_complex_input(golden):
    g = golden("circulant")
    S, _ = O.circulant_decompose(g["cdz_A"])
    assert rel(S, g["cdz_cols"]) < 1e-13


@pytest.mark.parametrize("tag", ["svd16_1_0", "svd32_2_1", "svd64_1_0", "svd64_2_2"])
def test_svd_golden(golden, tag):
    g = golden("svd")
    n, s, q, seed = (int(v) for v in g[tag + "_par"])
    A, B = g[tag + "_A"], g[tag + "_B"]
    for order in (0, 1):
        M, rep = O.svd_first_order_multiply(A, B, s, order, seed, power_iterations=q)
        assert rel(M, g[tag + f"_M{order}"]) < 1e-12
        r = g[tag + f"_rep{order}"]
        assert rep["norm_da"] == pytest.approx(r[0], rel=1e-9)
        assert rep["k"] == int(r[4])
    U, S, V, _ = O.rsvd(A, O.component_count(n, s), seed, q)
    assert rel(S, g[tag + "_S"]) < 1e-12
    assert rel(np.abs(U), np.abs(g[tag + "_U"])) < 1e-10


def test_c1_oversampled_composition(golden):
    g = golden("svd")
    n, k, p, q, t = (int(v) for v in g["c1_par"])
    sig = 0.9 ** np.arange(n)
    A = O.gen_haar_spectrum(n, sig, 2 * t)
    B = O.gen_haar_spectrum(n, sig, 2 * t + 1)
    assert np.array_equal(A, g["c1_A"]) and np.array_equal(B, g["c1_B"])
    M, rep = O.svd_first_order_multiply(A, B, None, 0, t, power_iterations=q,
                                        components=k, oversampling=p)
    assert rel(M, g["c1_M"]) < 1e-12
    assert rep["norm_da"] == pytest.approx(g["c1_nd"][0], rel=1e-9)


@pytest.mark.parametrize("tag", ["sq16", "sq32", "rect", "full", "zero"])
def test_sfft_golden(golden, tag):
    g = golden("fsparse")
    A, B, k = g[tag + "_A"], g[tag + "_B"], int(g[tag + "_k"])
    for order in (0, 1):
        for mode in ("rows", "cols"):
            M, rep = O.fft_sparse_first_order_multiply(A, B, k, order, mode)
            ref = g[f"{tag}_M{order}{mode}"]
            assert rel(M, ref) < 1e-12 or np.linalg.norm(ref) == 0
            assert rep["norm_da"] == pytest.approx(g[f"{tag}_rep{order}{mode}"][0], rel=1e-9,
                                                   abs=1e-12)


def test_topk_rows_golden(golden):
    g = golden("fsparse")
    for k in range(6):
        assert np.array_equal(O.topk_rows(g["tk_T"], k)[0], g[f"tk_{k}"])


@pytest.mark.parametrize("tag", ["cy16_3_3", "cy31_4_5", "cy64_8_8", "cy64_6_10"])
def test_cycle_golden(golden, tag):
    g = golden("cycle")
    _, _, ka, kb = tag.split("_")[0], None, int(tag.split("_")[1]), int(tag.split("_")[2])
    A, B = g[tag + "_A"], g[tag + "_B"]
    for order in (0, 1):
        M, rep = O.cycle_first_order_multiply(A, B, ka, order, kb=kb)
        assert rep["selected_a"] == list(g[tag + "_Ja"])
        assert rep["selected_b"] == list(g[tag + "_Jb"])
        assert rel(M, g[tag + f"_M{order}"]) < 1e-13


def test_cycle_first_order_identity(golden):
    g = golden("cycle")
    A, B = g["cy64_8_8_A"], g["cy64_8_8_B"]
    M, rep = O.cycle_first_order_multiply(A, B, 8, 1)
    dA = OX._cycle_residual(A, rep["selected_a"])
    dB = OX._cycle_residual(B, rep["selected_b"])
    assert np.linalg.norm((A @ B - M) - dA @ dB) < 1e-12 * np.linalg.norm(A @ B)
    assert rep["norm_da"] == pytest.approx(np.linalg.norm(dA), rel=1e-9)


def test_mixed_golden(golden):
    g = golden("cycle")
    n, ks, kc, seed = (int(v) for v in g["mx_par"])
    A, B = g["mx_A"], g["mx_B"]
    for order in (0, 1):
        M, rep = O.mixed_first_order_multiply(A, B, ks, kc, order, seed)
        assert rep["selected_b"] == list(g["mx_Jb"])
        assert rel(M, g[f"mx_M{order}"]) < 1e-12
    # row-subset evaluation (the bounded CPU sample) agrees with the full product
    Mfull, _ = O.mixed_first_order_multiply(A, B, ks, kc, 1, seed)
    Mrows, _ = O.mixed_first_order_multiply(A, B, ks, kc, 1, seed, rows=np.arange(5, 20))
    assert rel(Mrows, Mfull[5:20]) < 1e-13


def test_generators_deterministic():
    a = O.gen_cycle_operand(32, 4, 3)
    assert np.array_equal(a, O.gen_cycle_operand(32, 4, 3))
    c = O.gen_circulant_operand(32, 3, 1)
    assert np.isrealobj(c) and np.array_equal(c, O.gen_circulant_operand(32, 3, 1))


def test_sketch_norm_golden(golden):
    g = golden("errest")
    for name in g["sk_names"]:
        k, seed = (int(v) for v in g[f"sk_{name}_par"])
        got = O.sketch_norm_estimate(g[f"sk_{name}_A"], g[f"sk_{name}_B"], k, seed)
        ref = float(g[f"sk_{name}_out"])
        assert abs(got - ref) <= 1e-12 * max(1.0, abs(ref)), name


@pytest.mark.parametrize("tag", ["real", "cplx", "n1", "const", "odd"])
def test_fourier_row_decompose_golden(golden, tag):
    g = golden("fsparse")
    w, d = O.fourier_row_decompose(g[f"frs_{tag}_A"])
    assert np.allclose(w, g[f"frs_{tag}_w"], rtol=1e-12, atol=1e-13)
    assert np.allclose(d, g[f"frs_{tag}_d"], rtol=1e-12, atol=1e-13)
