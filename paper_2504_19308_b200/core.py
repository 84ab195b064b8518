"""Dense-matrix primitives -- GPU drop-in for the reference module ``apxmm.core``
(pkg/src/apxmm/core.py): the validation gate, the unitary DFT, cycle layouts and cycle powers,
Frobenius algebra and the exact product, all computed through the C-ABI.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as D
from . import _native as N

__all__ = [
    "as_matrix",
    "matmul_naive",
    "frobenius",
    "unitary_dft",
    "cycle_reorder",
    "cycle_reorder_inverse",
    "apply_cycle_power",
    "relative_error",
]


def as_matrix(a, allow_complex: bool = True) -> np.ndarray:
    """core.py:24-45 -- 2-D, non-empty, finite; cast to float64 / complex128 (host gate)."""
    return D.as_host_matrix(a, allow_complex=allow_complex)


def _dev(m: np.ndarray):
    dev = D.require_cuda()
    code = N.APX_C128 if np.iscomplexobj(m) else N.APX_F64
    return torch.from_numpy(np.ascontiguousarray(m)).to(dev), code


def matmul_naive(A, B) -> np.ndarray:
    """core.py:48-61 -- exact product A @ B (device DMMA GEMM in fp64; complex operands are
    expanded into four real products)."""
    A = as_matrix(A)
    B = as_matrix(B)
    if A.shape[1] != B.shape[0]:
        raise ValueError(f"dimension mismatch: {A.shape} x {B.shape}")

    def real_gemm(X, Y):
        Xd, _ = _dev(np.ascontiguousarray(X, dtype=np.float64))
        Yd, _ = _dev(np.ascontiguousarray(Y, dtype=np.float64))
        m, k = X.shape
        n = Y.shape[1]
        out = torch.empty((m, n), dtype=torch.float64, device=Xd.device)
        ws = D.workspace(N.size("apx_gemm_workspace", N.APX_F64, m, n, k, 0, 0))
        N.call("apx_gemm", N.APX_F64, 0, 0, m, n, k, Xd.data_ptr(), k, Yd.data_ptr(), n, out.data_ptr(), n, 0,
               ws.data_ptr(), ws.numel(), D.stream_ptr())
        return out.cpu().numpy()

    if not (np.iscomplexobj(A) or np.iscomplexobj(B)):
        return real_gemm(A, B)
    Ar, Ai = A.real, (A.imag if np.iscomplexobj(A) else np.zeros_like(A.real))
    Br, Bi = B.real, (B.imag if np.iscomplexobj(B) else np.zeros_like(B.real))
    return (real_gemm(Ar, Br) - real_gemm(Ai, Bi)) + 1j * (real_gemm(Ar, Bi) + real_gemm(Ai, Br))


def _pair(A, B, mode):
    Ad, ca = _dev(A)
    Bd, cb = _dev(B)
    out = torch.zeros(2, dtype=torch.float64, device=Ad.device)
    ws = D.workspace(N.size("apx_pair_reduce_workspace"))
    N.call("apx_pair_reduce", ca, Ad.data_ptr(), cb, Bd.data_ptr(), A.size, mode, out.data_ptr(), ws.data_ptr(),
           ws.numel(), D.stream_ptr())
    return out.cpu().numpy()


def frobenius(A, B=None):
    """core.py:64-79 -- ||A||_F, or the inner product <A, B> = sum(conj(A) * B)."""
    A = as_matrix(A)
    if B is None:
        return float(np.sqrt(_pair(A, A, 0)[0]))
    B = as_matrix(B)
    if A.shape != B.shape:
        raise ValueError(f"shape mismatch: {A.shape} vs {B.shape}")
    re, im = _pair(A, B, 0)
    if not (np.iscomplexobj(A) or np.iscomplexobj(B)):
        return float(re)
    return complex(re, im)


def unitary_dft(x, direction: str = "forward", axis: int = -1) -> np.ndarray:
    """core.py:82-97 -- W (forward) or W* (inverse) along ``axis`` for any length."""
    x = np.asarray(x)
    if x.ndim == 0 or x.shape[axis] < 1:
        raise ValueError("transform length must be >= 1")
    if direction not in ("forward", "inverse"):
        raise ValueError(f"unknown direction {direction!r}")
    moved = np.moveaxis(x.astype(np.complex128, copy=False), axis, -1)
    shape = moved.shape
    n = shape[-1]
    flat = np.ascontiguousarray(moved).reshape(-1, n)
    dev = D.require_cuda()
    xd = torch.from_numpy(flat).to(dev)
    yd = torch.empty_like(xd)
    ws = D.workspace(N.size("apx_unitary_dft_workspace", n, flat.shape[0]))
    N.call("apx_unitary_dft", xd.data_ptr(), yd.data_ptr(), n, flat.shape[0], 1, n,
           1 if direction == "inverse" else 0, ws.data_ptr(), ws.numel(), D.stream_ptr())
    return np.moveaxis(yd.cpu().numpy().reshape(shape), -1, axis)


def _check_square(A) -> int:
    if A.shape[0] != A.shape[1]:
        raise ValueError(f"square matrix required, got {A.shape}")
    return A.shape[0]


def _layout(A, mode):
    n = A.shape[0]
    Ad, code = _dev(A)
    out = torch.empty_like(Ad)
    N.call("apx_cycle_layout", 16 if code == N.APX_C128 else 8, Ad.data_ptr(), n, mode, out.data_ptr(),
           D.stream_ptr())
    return out.cpu().numpy()


def cycle_reorder(A, side: str) -> np.ndarray:
    """core.py:106-125 -- right: out[i,j] = A[(i+j)%n, i]; left: out[i,j] = A[i, (i-j)%n]."""
    A = as_matrix(A)
    _check_square(A)
    if side == "right":
        return _layout(A, 0)
    if side == "left":
        return _layout(A, 1)
    raise ValueError(f"unknown side {side!r}")


def cycle_reorder_inverse(At, side: str) -> np.ndarray:
    """core.py:128-137 -- scatter the cycle columns back to matrix cycles."""
    At = as_matrix(At)
    _check_square(At)
    if side == "right":
        return _layout(At, 2)
    if side == "left":
        return _layout(At, 3)
    raise ValueError(f"unknown side {side!r}")


def apply_cycle_power(M, k: int, side: str) -> np.ndarray:
    """core.py:140-154 -- left: C^k M (rows rotate down by k); right: M C^k (columns left)."""
    M = as_matrix(M)
    n = M.shape[0] if side == "left" else M.shape[1]
    if not 0 <= k < n:
        raise ValueError(f"k={k} out of range [0, {n})")
    if side not in ("left", "right"):
        raise ValueError(f"unknown side {side!r}")
    Md, code = _dev(M)
    out = torch.empty_like(Md)
    N.call("apx_apply_cycle_power", 16 if code == N.APX_C128 else 8, Md.data_ptr(), M.shape[0], M.shape[1], k,
           0 if side == "left" else 1, out.data_ptr(), D.stream_ptr())
    return out.cpu().numpy()


def relative_error(M, C_ref) -> float:
    """core.py:157-166 -- ||C_ref - M||_F / ||C_ref||_F."""
    M = as_matrix(M)
    C_ref = as_matrix(C_ref)
    if M.shape != C_ref.shape:
        raise ValueError(f"shape mismatch: {M.shape} vs {C_ref.shape}")
    diff2, ref2 = _pair(M, C_ref, 1)
    if ref2 == 0.0:
        raise ValueError("zero-norm reference")
    return float(np.sqrt(diff2) / np.sqrt(ref2))
