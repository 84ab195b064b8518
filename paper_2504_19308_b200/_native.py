"""ctypes binding of the in-tree CUDA extension ``_apx.so`` (C-ABI declared in include/apx.h).

There is no CPU fallback: importing the product modules succeeds on a CPU-only host (so the
C-ABI can be inspected), but every compute call raises unless the extension is built AND a
CUDA device is present.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("APX_LIB") or os.path.join(HERE, "_apx.so")  # APX_LIB: A/B builds

APX_F32, APX_F64, APX_C64, APX_C128 = 0, 1, 2, 3
E_ARG, E_CUDA, E_WS, E_NUMERIC, E_UNSUPPORTED = 1, 2, 3, 4, 5
NSCALARS = 8
S_FRO2_A, S_FRO2_B, S_KEPT_A, S_KEPT_B, S_FRO2_M, S_RES2_A, S_RES2_B = range(7)

_vp, _i64, _i32, _sz = C.c_void_p, C.c_int64, C.c_int, C.c_size_t

# name -> (restype, argtypes); kept in sync with include/apx.h (tests/test_capi.py checks it)
SIGNATURES = {
    "apx_abi_version": (C.c_int, []),
    "apx_last_error": (C.c_char_p, []),
    "apx_launch_count": (C.c_longlong, []),
    "apx_set_stage_events": (C.c_int, [_vp, _i32]),
    "apx_top_indices": (C.c_int, [_vp, _i64, _i32, _vp, _vp]),
    "apx_cycle_norms_workspace": (_sz, [_i32, _i64]),
    "apx_cycle_norms": (C.c_int, [_i32, _vp, _i64, _vp, _vp, _vp, _sz, _vp]),
    "apx_cycle_first_order_workspace": (_sz, [_i32, _i64, _i32, _i32, _i32]),
    "apx_cycle_first_order": (C.c_int, [_i32, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp,
                                        _vp, _vp, _sz, _vp]),
    "apx_debug_umma_gemm": (C.c_int, [_i32, _i32, _vp, _i64, _vp, _i64, _vp, _i64, _i64, _i64, _i64, _i32, _i32,
                                      _vp, _i32, _i32, _vp]),
    "apx_circulant_first_order_workspace": (_sz, [_i32, _i64, _i32, _i32]),
    "apx_circulant_first_order": (C.c_int, [_i32, _vp, _vp, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                            _sz, _vp]),
    "apx_circulant_decompose_workspace": (_sz, [_i32, _i64]),
    "apx_circulant_decompose": (C.c_int, [_i32, _vp, _i64, _vp, _vp, _vp, _sz, _vp]),
    "apx_circulant_materialize_workspace": (_sz, [_i64]),
    "apx_circulant_materialize": (C.c_int, [_vp, _vp, _i32, _i64, _vp, _vp, _sz, _vp]),
    "apx_circulant_component": (C.c_int, [_i32, _vp, _i64, _i32, _vp, _vp, _sz, _vp]),
    "apx_unitary_dft_workspace": (_sz, [_i64, _i64]),
    "apx_unitary_dft": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _i64, _i32, _vp, _sz, _vp]),
    "apx_cycle_layout": (C.c_int, [_i32, _vp, _i64, _i32, _vp, _vp]),
    "apx_apply_cycle_power": (C.c_int, [_i32, _vp, _i64, _i64, _i64, _i32, _vp, _vp]),
    "apx_pair_reduce_workspace": (_sz, []),
    "apx_pair_reduce": (C.c_int, [_i32, _vp, _i32, _vp, _i64, _i32, _vp, _vp, _sz, _vp]),
    "apx_sfft_first_order_workspace": (_sz, [_i64, _i64, _i64, _i32]),
    "apx_sfft_first_order": (C.c_int, [_i32, _vp, _vp, _i64, _i64, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _vp,
                                       _vp, _sz, _vp]),
    "apx_topk_rows_workspace": (_sz, [_i64, _i64]),
    "apx_fourier_row_decompose_workspace": (_sz, [_i64, _i64]),
    "apx_fourier_row_decompose": (C.c_int, [_i32, _vp, _i64, _i64, _vp, _vp, _vp, _sz, _vp]),
    "apx_sparse_rows_multiply": (C.c_int, [_vp, _vp, _i32, _i64, _vp, _i64, _vp, _vp]),
    "apx_topk_rows": (C.c_int, [_vp, _i64, _i64, _i32, _vp, _vp, _vp, _vp, _sz, _vp]),
    "apx_rsvd_workspace": (_sz, [_i32, _i64, _i64, _i32]),
    "apx_rsvd": (C.c_int, [_i32, _vp, _i64, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "apx_svd_first_order_workspace": (_sz, [_i32, _i64, _i64, _i64, _i32, _i32]),
    "apx_svd_first_order": (C.c_int, [_i32, _vp, _vp, _i64, _i64, _i64, _i32, _i32, _i32, _i32, _i32, _i32, _vp,
                                      _vp, _vp, _vp, _vp, _sz, _vp]),
    "apx_qr_workspace": (_sz, [_i32, _i64, _i64]),
    "apx_qr": (C.c_int, [_i32, _vp, _i64, _i64, _vp, _vp, _vp, _sz, _vp]),
    "apx_mixed_rows_workspace": (_sz, [_i64, _i64, _i32, _i32]),
    "apx_mixed_rows_phase": (C.c_int, [_i32, _vp, _i64, _vp, _i64, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp,
                                       _vp, _vp, _sz, _vp]),
    "apx_cycle_rows_workspace": (_sz, [_i32, _i64, _i64, _i32, _i32, _i32]),
    "apx_cycle_rows_phase": (C.c_int, [_i32, _i32, _vp, _i64, _i64, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _vp,
                                       _vp, _vp, _vp, _vp, _sz, _vp]),
    "apx_circulant_rows_grid": (C.c_int, [_i64, _vp, _vp]),
    "apx_circulant_rows_workspace": (_sz, [_i32, _i64, _i32, _i64, _i64, _i64]),
    "apx_circulant_rows_phase": (C.c_int, [_i32, _i32, _vp, _vp, _i64, _i32, _i32, _i64, _i64, _i64, _i64, _i64,
                                           _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "apx_sketch_norm_workspace": (_sz, [_i64, _i64, _i64, _i32]),
    "apx_sketch_norm": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _i32, _vp, _vp, _sz, _vp]),
    "apx_gemm_workspace": (_sz, [_i32, _i64, _i64, _i64, _i32, _i32]),
    "apx_gemm": (C.c_int, [_i32, _i32, _i32, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _i32, _vp, _sz,
                           _vp]),
    "apx_mixed_first_order_workspace": (_sz, [_i32, _i64, _i32, _i32, _i32]),
    "apx_mixed_first_order": (C.c_int, [_i32, _vp, _vp, _i64, _i32, _i32, _i32, _i32, _vp, _vp, _i32, _vp,
                                        _vp, _vp, _vp, _sz, _vp]),
}

_lib = None
_lock = threading.Lock()


class ExtensionMissing(ImportError):
    pass


def lib():
    """Load ``_apx.so`` once; raise loudly when it has not been built."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise ExtensionMissing(
                        f"CUDA extension {LIB_PATH} is not built; run "
                        "`python -m paper_2504_19308_b200.build` (there is no CPU fallback)")
                h = C.CDLL(LIB_PATH)
                for name, (res, args) in SIGNATURES.items():
                    f = getattr(h, name)
                    f.restype = res
                    f.argtypes = args
                _lib = h
    return _lib


def last_error() -> str:
    return lib().apx_last_error().decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    if rc == 0:
        return
    msg = last_error()
    if rc == E_ARG:
        raise ValueError(msg)
    raise RuntimeError(f"{what}: apx error {rc}: {msg}")


def call(name: str, *args):
    rc = getattr(lib(), name)(*args)
    check(rc, name)


def size(name: str, *args) -> int:
    return int(getattr(lib(), name)(*args))
