"""GPU parity for the core.py primitives against the reference's golden outputs."""
import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K():
    from paper_2504_19308_b200 import core as K
    return K


def test_layouts_and_powers(K, golden):
    g = golden("core")
    assert np.array_equal(K.cycle_reorder(g["cr_A4"], "right"), g["cr_right_A4"])
    assert np.array_equal(K.cycle_reorder(g["cr_A4"], "left"), g["cr_left_A4"])
    for n in (1, 5, 7, 33):
        A = g[f"cr_A{n}r"]
        for side in ("right", "left"):
            lay = K.cycle_reorder(A, side)
            assert np.array_equal(lay, g[f"cr_{side}_A{n}r"])
            assert np.array_equal(K.cycle_reorder_inverse(lay, side), A)
    for k in (0, 1, 5):
        assert np.array_equal(K.apply_cycle_power(g["acp_M"], k, "left"), g[f"acp_left_{k}"])
        assert np.array_equal(K.apply_cycle_power(g["acp_M"], k, "right"), g[f"acp_right_{k}"])
    with pytest.raises(ValueError):
        K.apply_cycle_power(g["acp_M"], 6, "left")
    with pytest.raises(ValueError):
        K.cycle_reorder(np.ones((2, 3)), "right")


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 7, 8, 16, 31, 64, 97, 128, 700])
def test_unitary_dft_golden(K, golden, n):
    g = golden("core")
    x = g[f"dft_x{n}"]
    assert rel(K.unitary_dft(x, "forward", 0), g[f"dft_fwd{n}"]) < 1e-13
    assert rel(K.unitary_dft(x, "inverse", 0), g[f"dft_inv{n}"]) < 1e-13
    assert rel(K.unitary_dft(x.T, "forward", 1), g[f"dft_fwd{n}"].T) < 1e-13


def test_dft_kats_and_errors(K):
    a, b = 3.0, 5.0
    assert np.allclose(K.unitary_dft(np.array([a, b])), [(a + b) / np.sqrt(2), (a - b) / np.sqrt(2)], atol=1e-15)
    for n in (3, 4, 7):
        p, q = np.indices((n, n))
        W = np.exp(-2j * np.pi * p * q / n) / np.sqrt(n)
        assert np.allclose(K.unitary_dft(np.eye(n), "forward", axis=0), W, atol=1e-12)
    with pytest.raises(ValueError):
        K.unitary_dft(np.array([1.0, 2.0]), "sideways")
    with pytest.raises(ValueError):
        K.unitary_dft(np.array(1.0))


def test_frobenius_relative_error_matmul(K):
    A = np.array([[1.0, 2.0], [3.0, 4.0]])
    assert K.frobenius(A) ** 2 == pytest.approx(30.0, rel=1e-15)
    assert K.frobenius(A, A) == pytest.approx(30.0, rel=1e-15)
    Z = np.array([[1j]])
    assert K.frobenius(Z, Z) == pytest.approx(1.0)
    assert K.frobenius(np.array([[1.0]]), Z) == pytest.approx(1j)
    ref = np.array([[3.0, 4.0], [0.0, 0.0]])
    assert K.relative_error(ref, ref) == 0.0
    assert K.relative_error(np.zeros((2, 2)), ref) == pytest.approx(1.0)
    with pytest.raises(ValueError):
        K.relative_error(ref, np.zeros((2, 2)))
    assert np.array_equal(K.matmul_naive([[1, 2], [3, 4]], [[5, 6], [7, 8]]), [[19.0, 22.0], [43.0, 50.0]])
    rng = np.random.default_rng(0)
    X, Y = rng.standard_normal((17, 23)), rng.standard_normal((23, 5))
    assert np.allclose(K.matmul_naive(X, Y), X @ Y, rtol=1e-13, atol=1e-13)
    with pytest.raises(ValueError):
        K.as_matrix([[1.0, np.nan]])
