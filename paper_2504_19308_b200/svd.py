"""Randomized truncated SVD and the SVD-based approximate product -- GPU drop-in for the
reference module ``apxmm.svd`` (pkg/src/apxmm/svd.py). Same names, arguments, validation and
return types; the arithmetic runs in the C-ABI (include/apx.h: apx_rsvd, apx_svd_first_order,
apx_qr, apx_gemm). The Gaussian sketch is drawn on the host with numpy exactly as the reference
draws it (svd.py:105-106, seeds svd.py:161-162), so a given seed sketches the same Omega.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from . import _native as N
from .errest import ErrorModel, energy_residual, finish_report

__all__ = [
    "TruncatedSVD",
    "qr_decompose",
    "component_count",
    "randomized_partial_svd",
    "svd_residual_norm",
    "svd_reconstruct",
    "svd_first_order_multiply",
]


@dataclass
class TruncatedSVD:
    """svd.py:34-60 -- rank-k factorization A ~ U diag(sigma) V^T (numpy arrays)."""

    U: np.ndarray
    sigma: np.ndarray
    V: np.ndarray
    source_frobenius_sq: float

    def __post_init__(self):
        if self.U.ndim != 2 or self.V.ndim != 2 or self.sigma.ndim != 1:
            raise ValueError("U, V must be 2-D and sigma 1-D")
        k = self.sigma.size
        if self.U.shape[1] != k or self.V.shape[1] != k:
            raise ValueError("U, sigma, V have inconsistent component counts")
        if self.source_frobenius_sq < 0:
            raise ValueError("source_frobenius_sq must be >= 0")

    @property
    def k(self) -> int:
        return self.sigma.size


def _dev64(x) -> torch.Tensor:
    t, code, _ = D.as_device_matrix(x, real_only=True)
    if code != N.APX_F64:
        t = t.to(torch.float64)
    return t


def qr_decompose(Y):
    """svd.py:63-69 -- thin QR of an m x k sketch (m >= k), returns (Q m x k, R k x k)."""
    Yh = D.as_host_matrix(Y)
    m, k = Yh.shape
    if m < k:
        raise ValueError(f"need at least as many rows as columns, got {m} x {k}")
    if np.iscomplexobj(Yh):
        raise ValueError("qr_decompose: real input required")
    Yd = _dev64(Yh)
    Q = torch.empty((m, k), dtype=torch.float64, device=Yd.device)
    R = torch.empty((k, k), dtype=torch.float64, device=Yd.device)
    ws = D.workspace(N.size("apx_qr_workspace", N.APX_F64, m, k))
    N.call("apx_qr", N.APX_F64, Yd.data_ptr(), m, k, Q.data_ptr(), R.data_ptr(), ws.data_ptr(), ws.numel(),
           D.stream_ptr())
    return Q.cpu().numpy(), R.cpu().numpy()


def component_count(n: int, s: int) -> int:
    """svd.py:72-80 -- k = min(s * floor(log2 n) + 1, n)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    if s < 1:
        raise ValueError("s must be >= 1")
    if n == 1:
        return 1
    return min(s * int(math.floor(math.log2(n))) + 1, n)


def _rsvd_device(Ad: torch.Tensor, l: int, k: int, q: int, omega: np.ndarray):
    m, n = Ad.shape
    dev = Ad.device
    om = torch.from_numpy(np.ascontiguousarray(omega, dtype=np.float64)).to(dev)
    U = torch.empty((m, k), dtype=torch.float64, device=dev)
    V = torch.empty((n, k), dtype=torch.float64, device=dev)
    S = torch.empty(k, dtype=torch.float64, device=dev)
    scal = torch.zeros(N.NSCALARS, dtype=torch.float64, device=dev)
    ws = D.workspace(N.size("apx_rsvd_workspace", N.APX_F64, m, n, l))
    N.call("apx_rsvd", N.APX_F64, Ad.data_ptr(), m, n, l, k, q, om.data_ptr(), U.data_ptr(), S.data_ptr(),
           V.data_ptr(), scal.data_ptr(), ws.data_ptr(), ws.numel(), D.stream_ptr())
    return U, S, V, scal


def randomized_partial_svd(A, s: int, seed, power_iterations: int = 0,
                           components: int | None = None) -> TruncatedSVD:
    """svd.py:83-119 -- rank-k randomized SVD with k from `s` (or `components`)."""
    Ah = D.as_host_matrix(A)
    if np.iscomplexobj(Ah):
        raise ValueError("randomized_partial_svd expects a real matrix")
    m, n = Ah.shape
    if components is not None:
        if components < 1:
            raise ValueError("components must be >= 1")
        k = min(components, m, n)
    else:
        k = min(component_count(n, s), m)
    if power_iterations < 0:
        raise ValueError("power_iterations must be >= 0")
    rng = np.random.default_rng(seed)
    phi = rng.standard_normal((n, k))
    U, S, V, scal = _rsvd_device(_dev64(Ah), k, k, power_iterations, phi)
    fro2 = float(scal[N.S_FRO2_A].item())
    return TruncatedSVD(U=U.cpu().numpy(), sigma=S.cpu().numpy(), V=V.cpu().numpy(), source_frobenius_sq=fro2)


def svd_residual_norm(decomp: TruncatedSVD) -> float:
    """svd.py:122-130 -- sqrt(max(0, ||A||^2 - sum sigma^2))."""
    retained = float(np.sum(decomp.sigma ** 2))
    return math.sqrt(max(0.0, decomp.source_frobenius_sq - retained))


def svd_reconstruct(decomp: TruncatedSVD) -> np.ndarray:
    """svd.py:133-135 -- (U diag(sigma)) V^T on the device (apx_gemm, V consumed transposed)."""
    Us = np.ascontiguousarray(decomp.U * decomp.sigma)
    m, k = Us.shape
    n = decomp.V.shape[0]
    Ud = _dev64(Us)
    Vd = _dev64(np.ascontiguousarray(decomp.V))
    out = torch.empty((m, n), dtype=torch.float64, device=Ud.device)
    ws = D.workspace(N.size("apx_gemm_workspace", N.APX_F64, m, n, k, 0, 1))
    N.call("apx_gemm", N.APX_F64, 0, 1, m, n, k, Ud.data_ptr(), k, Vd.data_ptr(), k, out.data_ptr(), n, 0,
           ws.data_ptr(), ws.numel(), D.stream_ptr())
    return out.cpu().numpy()


def svd_product_device(Ad, Bd, la, ka, lb, kb, q, order, omega_a, omega_b, out=None):
    """Device-level call (fp64 tensors): returns dict(M, scalars)."""
    m, n = Ad.shape
    p = Bd.shape[1]
    dev = Ad.device
    M = out if out is not None else torch.empty((m, p), dtype=torch.float64, device=dev)
    oa = torch.from_numpy(np.ascontiguousarray(omega_a, dtype=np.float64)).to(dev)
    ob = torch.from_numpy(np.ascontiguousarray(omega_b, dtype=np.float64)).to(dev)
    scal = torch.zeros(N.NSCALARS, dtype=torch.float64, device=dev)
    ws = D.workspace(N.size("apx_svd_first_order_workspace", N.APX_F64, m, n, p, la, lb))
    N.call("apx_svd_first_order", N.APX_F64, Ad.data_ptr(), Bd.data_ptr(), m, n, p, la, ka, lb, kb, q, order,
           oa.data_ptr(), ob.data_ptr(), M.data_ptr(), scal.data_ptr(), ws.data_ptr(), ws.numel(), D.stream_ptr())
    return {"M": M, "scalars": scal, "ws": ws}


def svd_first_order_multiply(A, B, s: int, order: int, seed, power_iterations: int = 0,
                             model: ErrorModel | None = None, components: int | None = None,
                             oversampling: int = 0):
    """svd.py:138-200 -- approximate A @ B through rank-k truncations of both factors.

    Extensions beyond the reference signature (config C1): ``components`` fixes k directly and
    ``oversampling`` p sketches k + p columns, keeping the leading k triplets. With the defaults
    the computation is the reference's."""
    Ah = D.as_host_matrix(A) if not D.is_device(A) else None
    Bh = D.as_host_matrix(B) if not D.is_device(B) else None
    host = Ah is not None
    if host and (np.iscomplexobj(Ah) or np.iscomplexobj(Bh)):
        raise ValueError("randomized_partial_svd expects a real matrix")
    Ad = _dev64(Ah if host else A)
    Bd = _dev64(Bh if host else B)
    m, n = Ad.shape
    if Bd.shape[0] != n:
        raise ValueError(f"dimension mismatch: {tuple(Ad.shape)} x {tuple(Bd.shape)}")
    if order not in (0, 1):
        raise ValueError("order must be 0 or 1")
    if power_iterations < 0:
        raise ValueError("power_iterations must be >= 0")
    p = Bd.shape[1]
    if components is not None:
        if components < 1:
            raise ValueError("components must be >= 1")
        ka, kb = min(components, m, n), min(components, n, p)
    else:
        ka = min(component_count(n, s), m)
        kb = min(component_count(p, s), n)
    la, lb = min(ka + oversampling, m, n), min(kb + oversampling, n, p)
    t0 = time.perf_counter()
    oa = np.random.default_rng([seed, 0]).standard_normal((n, la))
    ob = np.random.default_rng([seed, 1]).standard_normal((p, lb))
    r = svd_product_device(Ad, Bd, la, ka, lb, kb, power_iterations, order, oa, ob)
    sc = r["scalars"].tolist()
    wall = time.perf_counter() - t0
    nA, nB = math.sqrt(max(0.0, sc[N.S_FRO2_A])), math.sqrt(max(0.0, sc[N.S_FRO2_B]))
    ndA = energy_residual(sc[N.S_FRO2_A], sc[N.S_KEPT_A], m * n)  # svd.py:122-130
    ndB = energy_residual(sc[N.S_FRO2_B], sc[N.S_KEPT_B], n * p)
    nM = math.sqrt(max(0.0, sc[N.S_FRO2_M]))
    rep = finish_report("svd", order, ka, nA, nB, ndA, ndB, nM, n, wall, model)
    return D.to_user(r["M"], host), rep
