"""Circulant decomposition and the truncated first-order product -- GPU drop-in for the
reference module ``apxmm.circulant`` (pkg/src/apxmm/circulant.py). Same names, arguments,
validation and return types (M is complex128, as circulant.py:171-172 returns it); the
transforms, selection and products run in the C-ABI (apx_circulant_*, apx_top_indices).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _device as D
from . import _native as N
from .errest import ErrorModel, finish_report, energy_residual

__all__ = [
    "CirculantSpectrum",
    "circulant_decompose",
    "circulant_component",
    "circulant_select",
    "circulant_materialize",
    "circulant_first_order_multiply",
    "top_indices",
]


@dataclass
class CirculantSpectrum:
    """circulant.py:39-60 -- columns[k] = first column of R_k; magnitudes; selected (ascending)."""

    n: int
    columns: np.ndarray
    magnitudes: np.ndarray
    selected: list[int]

    def __post_init__(self):
        if self.columns.shape != (self.n, self.n):
            raise ValueError("columns must be n x n (row k = first column of R_k)")
        if self.magnitudes.shape != (self.n,):
            raise ValueError("need one magnitude per component")
        if any(not 0 <= k < self.n for k in self.selected):
            raise ValueError("selected index out of range")


def _matrix(A):
    """Device copy in the reference's working precision (float64 / complex128) + dtype code."""
    if D.is_device(A):
        t = A
        if t.dtype == torch.float32:
            t = t.double()
        elif t.dtype == torch.complex64:
            t = t.to(torch.complex128)
        code = N.APX_C128 if t.is_complex() else N.APX_F64
        return t.contiguous(), code, False
    m = D.as_host_matrix(A)
    code = N.APX_C128 if np.iscomplexobj(m) else N.APX_F64
    dev = D.require_cuda()
    return torch.from_numpy(np.ascontiguousarray(m)).to(dev), code, True


def top_indices(weights, k: int) -> list[int]:
    """circulant.py:63-70 -- k largest weights, ties to the lower index, ascending (device)."""
    w = np.asarray(weights, dtype=np.float64).ravel() if not D.is_device(weights) else None
    size = w.size if w is not None else weights.numel()
    if not 0 <= k <= size:
        raise ValueError(f"k={k} out of range [0, {size}]")
    if k == 0:
        return []
    dev = D.require_cuda()
    wd = torch.from_numpy(w).to(dev) if w is not None else weights.to(torch.float64).contiguous()
    out = torch.empty(k, dtype=torch.int32, device=dev)
    N.call("apx_top_indices", wd.data_ptr(), size, k, out.data_ptr(), D.stream_ptr())
    return [int(i) for i in out.cpu().tolist()]


def circulant_decompose(A) -> CirculantSpectrum:
    """circulant.py:73-91 -- all n circulant components via one batched FFT pass."""
    Ad, code, _ = _matrix(A)
    n = Ad.shape[0]
    if Ad.shape[1] != n:
        raise ValueError(f"square matrix required, got {tuple(Ad.shape)}")
    cols = torch.empty((n, n), dtype=torch.complex128, device=Ad.device)
    mags = torch.empty(n, dtype=torch.float64, device=Ad.device)
    ws = D.workspace(N.size("apx_circulant_decompose_workspace", code, n))
    N.call("apx_circulant_decompose", code, Ad.data_ptr(), n, cols.data_ptr(), mags.data_ptr(), ws.data_ptr(),
           ws.numel(), D.stream_ptr())
    return CirculantSpectrum(n=n, columns=cols.cpu().numpy(), magnitudes=mags.cpu().numpy(),
                             selected=list(range(n)))


def circulant_component(A, k: int) -> np.ndarray:
    """circulant.py:94-108 -- first column of R_k by cycle averaging, O(n^2)."""
    Ad, code, _ = _matrix(A)
    n = Ad.shape[0]
    if Ad.shape[1] != n:
        raise ValueError(f"square matrix required, got {tuple(Ad.shape)}")
    if not 0 <= k < n:
        raise ValueError(f"component index {k} out of range [0, {n})")
    out = torch.empty(n, dtype=torch.complex128, device=Ad.device)
    ws = D.workspace(N.size("apx_circulant_materialize_workspace", n))
    N.call("apx_circulant_component", code, Ad.data_ptr(), n, k, out.data_ptr(), ws.data_ptr(), ws.numel(),
           D.stream_ptr())
    return out.cpu().numpy()


def circulant_select(spectrum: CirculantSpectrum, k: int) -> CirculantSpectrum:
    """circulant.py:111-113."""
    return replace(spectrum, selected=top_indices(spectrum.magnitudes, k))


def circulant_materialize(spectrum: CirculantSpectrum) -> np.ndarray:
    """circulant.py:116-127 -- dense sum over the selected components (device)."""
    n = spectrum.n
    sel = list(spectrum.selected)
    if not sel:
        return np.zeros((n, n), dtype=np.complex128)
    dev = D.require_cuda()
    ssel = torch.from_numpy(np.ascontiguousarray(spectrum.columns[sel], dtype=np.complex128)).to(dev)
    seld = torch.tensor(sel, dtype=torch.int32, device=dev)
    out = torch.empty((n, n), dtype=torch.complex128, device=dev)
    ws = D.workspace(N.size("apx_circulant_materialize_workspace", n))
    N.call("apx_circulant_materialize", ssel.data_ptr(), seld.data_ptr(), len(sel), n, out.data_ptr(),
           ws.data_ptr(), ws.numel(), D.stream_ptr())
    return out.cpu().numpy()


def circulant_product_device(Ad, Bd, code, k: int, order: int, force_sel_a=None, force_sel_b=None, out=None):
    n = Ad.shape[0]
    dev = Ad.device
    M = out if out is not None else torch.empty((n, n), dtype=torch.complex128, device=dev)
    sa = torch.empty(max(k, 1), dtype=torch.int32, device=dev)
    sb = torch.empty(max(k, 1), dtype=torch.int32, device=dev)
    fa = None if force_sel_a is None else torch.as_tensor(force_sel_a, dtype=torch.int32).to(dev)
    fb = None if force_sel_b is None else torch.as_tensor(force_sel_b, dtype=torch.int32).to(dev)
    scal = torch.zeros(N.NSCALARS, dtype=torch.float64, device=dev)
    ws = D.workspace(N.size("apx_circulant_first_order_workspace", code, n, k, order))
    N.call("apx_circulant_first_order", code, Ad.data_ptr(), Bd.data_ptr(), n, k, order, D.ptr(fa), D.ptr(fb),
           M.data_ptr(), sa.data_ptr(), sb.data_ptr(), scal.data_ptr(), ws.data_ptr(), ws.numel(), D.stream_ptr())
    return {"M": M, "sel_a": sa[:k], "sel_b": sb[:k], "scalars": scal, "ws": ws}


def circulant_first_order_multiply(A, B, k: int, order: int, model: ErrorModel | None = None,
                                   force_sel_a=None, force_sel_b=None):
    """circulant.py:164-218 -- approximate A @ B keeping the k largest circulant components of
    each operand; returns (M complex128, ApproxReport('cd', ...)). ``force_sel_*`` pin the
    selections (the near-tie protocol of the parity tests)."""
    Ad, ca, host = _matrix(A)
    Bd, cb, _ = _matrix(B)
    n = Ad.shape[0]
    if Ad.shape[1] != n or tuple(Bd.shape) != (n, n):
        raise ValueError(f"two square n x n matrices required, got {tuple(Ad.shape)} x {tuple(Bd.shape)}")
    if not 0 <= k <= n:
        raise ValueError(f"k={k} out of range [0, {n}]")
    if order not in (0, 1):
        raise ValueError("order must be 0 or 1")
    code = N.APX_C128 if (ca == N.APX_C128 or cb == N.APX_C128) else N.APX_F64
    if code == N.APX_C128:
        Ad, Bd = Ad.to(torch.complex128), Bd.to(torch.complex128)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = circulant_product_device(Ad, Bd, code, k, order, force_sel_a, force_sel_b)
    s = r["scalars"].tolist()
    wall = time.perf_counter() - t0
    nA, nB = math.sqrt(max(0.0, s[N.S_FRO2_A])), math.sqrt(max(0.0, s[N.S_FRO2_B]))
    ndA = energy_residual(s[N.S_FRO2_A], s[N.S_KEPT_A], n * n)  # circulant.py:130-133
    ndB = energy_residual(s[N.S_FRO2_B], s[N.S_KEPT_B], n * n)
    rep = finish_report("cd", order, k, nA, nB, ndA, ndB, math.sqrt(max(0.0, s[N.S_FRO2_M])), n, wall, model)
    rep.selected_a = r["sel_a"].tolist()
    rep.selected_b = r["sel_b"].tolist()
    return D.to_user(r["M"], host), rep
