import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C-ABI)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
                cache[name] = {k: z[k] for k in z.files}
        return cache[name]

    return load


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    d = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (d if d > 0 else 1.0))


def check_report(rep, r, rel_tol=1e-6, abs_tol=1e-9):
    """ApproxReport fields vs a golden rep_arr (make_golden.py): [norm_da, norm_db, apriori,
    posterior, k]; NaN in the golden file means the reference left the field None."""
    import pytest

    assert rep.k == int(r[4])
    for name, want in (("apriori_estimate", r[2]), ("posterior_estimate", r[3])):
        got = getattr(rep, name)
        if np.isnan(want):
            assert got is None, (name, got)
        else:
            assert got == pytest.approx(float(want), rel=rel_tol, abs=abs_tol), name
