"""Device plumbing: torch tensors as containers, streams, workspaces, host<->device copies.

Inputs may be numpy arrays / array-likes (the reference's calling convention -> results come
back as numpy, as the reference returns them) or torch CUDA tensors (results stay on device;
used by bench.py and by callers that keep data resident in HBM).
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _native as N

_TORCH_DT = {N.APX_F32: torch.float32, N.APX_F64: torch.float64,
             N.APX_C64: torch.complex64, N.APX_C128: torch.complex128}


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2504_19308_b200 needs a CUDA device (sm_100a); there is no CPU path")
    N.lib()
    return torch.device("cuda", torch.cuda.current_device())


def is_device(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


def check_finite_host(m: np.ndarray) -> None:
    if np.iscomplexobj(m):
        ok = np.isfinite(m.real).all() and np.isfinite(m.imag).all()
    else:
        ok = np.isfinite(m).all()
    if not ok:
        raise ValueError("matrix entries must be finite (no NaN/Inf)")


# Host arrays of at least this many bytes travel through pinned staging buffers (torch's caching
# pinned allocator: allocated once, reused by later calls) and are checked for NaN/Inf on the
# device after the upload instead of by a host pass (np.isfinite over 134 MB costs ~35 ms; the
# device pass ~0.1 ms). Smaller inputs keep the host check and a plain copy (no extra sync).
_PIN_MIN_BYTES = 1 << 20


def _upload(m: np.ndarray, dev) -> torch.Tensor:
    """Host array -> device tensor; large arrays via a pinned staging buffer and an async copy,
    validated for finiteness on the device (same ValueError as the host gate)."""
    src = torch.from_numpy(np.ascontiguousarray(m))
    if m.nbytes < _PIN_MIN_BYTES:
        return src.to(dev)
    stage = torch.empty(src.shape, dtype=src.dtype, pin_memory=True)
    stage.copy_(src)
    t = stage.to(dev, non_blocking=True)  # the pinned allocator keeps `stage` until the copy is done
    if not bool(torch.isfinite(t).all()):
        raise ValueError("matrix entries must be finite (no NaN/Inf)")
    return t


def as_host_matrix(a, allow_complex: bool = True, check_finite: bool = True) -> np.ndarray:
    """core.py:24-45 -- the reference's validation gate (2-D, non-empty, finite, f64/c128)."""
    m = np.asarray(a)
    if m.ndim != 2:
        raise ValueError(f"expected a 2-D matrix, got ndim={m.ndim}")
    if m.size == 0:
        raise ValueError("empty matrix")
    if np.iscomplexobj(m):
        if not allow_complex:
            raise ValueError("complex entries not allowed here")
        m = m.astype(np.complex128, copy=False)
    else:
        m = m.astype(np.float64, copy=False)
    if check_finite:
        check_finite_host(m)
    return m


def as_device_matrix(a, real_only: bool = False):
    """Return (device tensor, dtype code, came_from_host). Device tensors are validated for
    shape/dtype only (a finiteness scan would cost a full HBM pass)."""
    dev = require_cuda()
    if isinstance(a, torch.Tensor) and not a.is_cuda:
        # host torch tensor (pinned for the e2e path): async H2D, result goes back to the host
        t, code, _ = as_device_matrix(a.to(dev, non_blocking=True), real_only)
        return t, code, "torch"
    if is_device(a):
        t = a
        if t.dim() != 2:
            raise ValueError(f"expected a 2-D matrix, got ndim={t.dim()}")
        if t.numel() == 0:
            raise ValueError("empty matrix")
        if t.dtype == torch.float32:
            code = N.APX_F32
        elif t.dtype == torch.float64:
            code = N.APX_F64
        elif t.dtype in (torch.complex64, torch.complex128) and not real_only:
            code = N.APX_C64 if t.dtype == torch.complex64 else N.APX_C128
        else:
            raise ValueError(f"unsupported dtype {t.dtype}")
        return t.contiguous(), code, False
    m = as_host_matrix(a, allow_complex=not real_only, check_finite=False)
    if m.nbytes < _PIN_MIN_BYTES:
        check_finite_host(m)  # large arrays: checked on the device by _upload
    return _upload(m, dev), (N.APX_C128 if np.iscomplexobj(m) else N.APX_F64), True


def empty(shape, code, device=None) -> torch.Tensor:
    return torch.empty(shape, dtype=_TORCH_DT[code], device=device or require_cuda())


def workspace(nbytes: int) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=require_cuda())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def to_user(t: torch.Tensor, host, out=None):
    """Return the result in the caller's container: numpy for numpy inputs (the reference
    contract), a (pinned) host tensor for host torch inputs -- written into ``out`` when given --
    and the device tensor otherwise."""
    if not host:
        return t
    if host == "torch":
        if out is None:
            out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        out.copy_(t, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return out
    if t.numel() * t.element_size() < _PIN_MIN_BYTES or os.environ.get("APX_PINNED_RESULTS", "1") == "0":
        return t.cpu().numpy()  # (APX_PINNED_RESULTS=0: callers that hoard results keep them pageable)
    # large results land in a pinned buffer (async DMA at PCIe rate instead of a pageable copy);
    # the numpy array returned is a view that keeps it alive and hands it back to torch's pinned
    # cache when the caller drops it
    host_t = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    host_t.copy_(t, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return host_t.numpy()
