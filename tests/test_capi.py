"""CPU-side checks of the drop-in boundary: the C-ABI library loads and exports every symbol
include/apx.h declares, and the ctypes table matches the header (no compute without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "apx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(apx_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2504_19308_b200 import _native as N
    lib = N.lib()
    names = declared_functions()
    assert len(names) >= 5
    for name in names:
        assert hasattr(lib, name), name
        assert name in N.SIGNATURES, f"{name} missing from the ctypes table"
    assert lib.apx_abi_version() == 1


def test_workspace_queries_are_pure():
    from paper_2504_19308_b200 import _native as N
    a = N.size("apx_cycle_first_order_workspace", 1, 2048, 32, 32, 1)
    b = N.size("apx_cycle_first_order_workspace", 1, 2048, 32, 32, 1)
    assert a == b and a > 2048 * 8


def test_argument_errors_map_to_valueerror():
    from paper_2504_19308_b200 import _native as N
    rc = N.lib().apx_top_indices(None, 4, 5, None, None)
    assert rc == N.E_ARG
    with pytest.raises(ValueError):
        N.check(rc)
    assert "out of range" in N.last_error()


def test_product_path_has_no_cpu_fallback():
    import torch
    import paper_2504_19308_b200 as P
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        P.cycle_first_order_multiply([[1.0, 2.0], [3.0, 4.0]], [[1.0, 0.0], [0.0, 1.0]], 1, 1)
