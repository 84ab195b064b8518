"""sketch_norm_estimate (errest.py:139-154) on the device against the reference's own outputs
(tests/golden/errest.npz) and the reference's statistical tests (test_errest.py:108-133).

Tolerance: 1e-12 relative (fp64 DMMA GEMMs; the sketch G is drawn by numpy exactly as the
reference draws it, so only summation order differs).
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E():
    from paper_2504_19308_b200 import errest as E
    return E


def test_sketch_golden(E, golden):
    g = golden("errest")
    for name in g["sk_names"]:
        k, seed = (int(v) for v in g[f"sk_{name}_par"])
        got = E.sketch_norm_estimate(g[f"sk_{name}_A"], g[f"sk_{name}_B"], k, seed)
        ref = float(g[f"sk_{name}_out"])
        assert abs(got - ref) <= 1e-12 * max(1.0, abs(ref)), name


def test_sketch_vs_oracle_larger(E):
    rng = np.random.default_rng(5)
    A = rng.standard_normal((700, 1100))
    B = rng.standard_normal((1100, 900))
    for k, seed in ((1, 0), (16, 3), (130, 9)):
        got = E.sketch_norm_estimate(A, B, k, seed)
        ref = O.sketch_norm_estimate(A, B, k, seed)
        assert abs(got - ref) <= 1e-12 * ref


def test_sketch_zero_and_identity_mean(E):
    assert E.sketch_norm_estimate(np.zeros((4, 4)), np.eye(4), 3, 0) == 0.0
    n, k = 16, 8
    vals = [E.sketch_norm_estimate(np.eye(n), np.eye(n), k, seed) for seed in range(200)]
    assert abs(np.mean(vals) - n) < 0.05 * n


def test_sketch_unbiased_on_fixed_pair(E):
    rng = np.random.default_rng(42)
    A = rng.standard_normal((32, 32))
    B = rng.standard_normal((32, 32))
    exact = float(np.linalg.norm(A @ B) ** 2)
    vals = [E.sketch_norm_estimate(A, B, 4, seed) for seed in range(1000)]
    assert abs(np.mean(vals) / exact - 1.0) < 0.03
