"""Cycle-truncated and mixed (rSVD x cycles) approximate products -- GPU path.

The reference ships the cycle primitives only (core.py:106-154; the paper marks cycle products
"not demonstrated here"). This module supplies the product with the reference's
conventions:

  * A = sum_j Lambda_j C^j, Lambda_j = diag(cycle_reorder(A, "left")[:, j])  (core.py:123-124)
  * selection = top_indices of the cycle 2-norms (circulant.py:63-70: ties -> lower index)
  * order 0: Ahat . Bhat (zeroth order, the svd convention svd.py:169-172)
  * order 1: Ahat . B + dA . Bhat (first order, svd.py:174-177 / circulant.py:193-198)
  * residual norms from energy differences (circulant.py:130-133)
"""

from __future__ import annotations

import math
import time

import torch

from . import _device as D
from . import _native as N
from .errest import ErrorModel, energy_residual, finish_report


def cycle_product_device(A, B, k_a: int, k_b: int, order: int, force_sel_a=None, force_sel_b=None,
                         out=None):
    """Device-level call: returns dict(M, sel_a, sel_b, scalars) with device tensors.

    A, B: square device tensors of one real dtype (float32 / float64)."""
    n = A.shape[0]
    code = N.APX_F32 if A.dtype == torch.float32 else N.APX_F64
    dev = A.device
    M = out if out is not None else torch.empty((n, n), dtype=A.dtype, device=dev)
    sa = torch.empty(max(k_a, 1), dtype=torch.int32, device=dev)
    sb = torch.empty(max(k_b, 1), dtype=torch.int32, device=dev)
    fa = None if force_sel_a is None else torch.as_tensor(force_sel_a, dtype=torch.int32).to(dev)
    fb = None if force_sel_b is None else torch.as_tensor(force_sel_b, dtype=torch.int32).to(dev)
    scal = torch.zeros(N.NSCALARS, dtype=torch.float64, device=dev)
    ws = D.workspace(N.size("apx_cycle_first_order_workspace", code, n, k_a, k_b, order))
    N.call("apx_cycle_first_order", code, A.data_ptr(), B.data_ptr(), n, k_a, k_b, order,
           D.ptr(fa), D.ptr(fb), M.data_ptr(), sa.data_ptr(), sb.data_ptr(), scal.data_ptr(),
           ws.data_ptr(), ws.numel(), D.stream_ptr())
    return {"M": M, "sel_a": sa[:k_a], "sel_b": sb[:k_b], "scalars": scal, "ws": ws}


def _norms(s, terms: int):
    """(||A||, ||B||, ||dA||, ||dB||, ||M||) from the device scalars; `terms` = entries per operand."""
    nA = math.sqrt(max(0.0, s[N.S_FRO2_A]))
    nB = math.sqrt(max(0.0, s[N.S_FRO2_B]))
    ndA = energy_residual(s[N.S_FRO2_A], s[N.S_KEPT_A], terms)
    ndB = energy_residual(s[N.S_FRO2_B], s[N.S_KEPT_B], terms)
    return nA, nB, ndA, ndB, math.sqrt(max(0.0, s[N.S_FRO2_M]))


def cycle_first_order_multiply(A, B, k: int, order: int, model: ErrorModel | None = None,
                               k_b: int | None = None, force_sel_a=None, force_sel_b=None):
    """Approximate A @ B keeping the k dominant cycles of A (k_b of B, default k).

    Mirrors circulant_first_order_multiply's contract (circulant.py:164-218): square real
    inputs, 0 <= k <= n, order in {0, 1}, returns (M, ApproxReport) with method "cycle".
    numpy in -> numpy float64 out; torch CUDA in -> torch CUDA out (same dtype)."""
    Ad, code_a, host = D.as_device_matrix(A, real_only=True)
    Bd, code_b, _ = D.as_device_matrix(B, real_only=True)
    n = Ad.shape[0]
    if Ad.shape[1] != n or tuple(Bd.shape) != (n, n):
        raise ValueError(f"two square n x n matrices required, got {tuple(Ad.shape)} x {tuple(Bd.shape)}")
    if Bd.dtype != Ad.dtype:
        Bd = Bd.to(Ad.dtype)
    k_b = k if k_b is None else k_b
    if not 0 <= k <= n or not 0 <= k_b <= n:
        raise ValueError(f"k={k} out of range [0, {n}]")
    if order not in (0, 1):
        raise ValueError("order must be 0 or 1")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = cycle_product_device(Ad, Bd, k, k_b, order, force_sel_a, force_sel_b)
    s = r["scalars"].tolist()  # synchronises
    wall = time.perf_counter() - t0
    nA, nB, ndA, ndB, nM = _norms(s, n * n)
    rep = finish_report("cycle", order, k, nA, nB, ndA, ndB, nM, n, wall, model)
    rep.selected_a = r["sel_a"].tolist()
    rep.selected_b = r["sel_b"].tolist()
    return D.to_user(r["M"], host), rep


def draw_sketch(n: int, k: int, seed) -> "np.ndarray":
    """The Gaussian test matrix of randomized_partial_svd for operand A: default_rng([seed, 0])
    (svd.py:161) then rng.standard_normal((n, k)) (svd.py:105-106) -- drawn on the host with
    numpy itself so it is bit-identical to the reference's sketch."""
    import numpy as np

    return np.random.default_rng([seed, 0]).standard_normal((n, k))


def mixed_product_device(A, B, k_svd: int, k_cyc: int, order: int, omega, power_iterations: int = 0,
                         force_sel_b=None, split3: bool = False, out=None, direct: bool = False):
    """Device-level mixed product (config C4). omega: device tensor n x k_svd (A's dtype).

    fp32 order 1 runs the residual plan (M = Q (Bm B) + dA Bhat with dA in scaled f16, see
    csrc/mixed_f16.cu) where the shape allows; ``direct=True`` forces the all-fp32 plan
    (M = A Bhat + Q W with the gather over A)."""
    n = A.shape[0]
    code = N.APX_F32 if A.dtype == torch.float32 else N.APX_F64
    dev = A.device
    M = out if out is not None else torch.empty((n, n), dtype=A.dtype, device=dev)
    sb = torch.empty(max(k_cyc, 1), dtype=torch.int32, device=dev)
    fb = None if force_sel_b is None else torch.as_tensor(force_sel_b, dtype=torch.int32).to(dev)
    scal = torch.zeros(N.NSCALARS, dtype=torch.float64, device=dev)
    ws = D.workspace(N.size("apx_mixed_first_order_workspace", code, n, k_svd, k_cyc, order))
    N.call("apx_mixed_first_order", code, A.data_ptr(), B.data_ptr(), n, k_svd, k_cyc, order,
           power_iterations, omega.data_ptr(), D.ptr(fb), (1 if split3 else 0) | (4 if direct else 0), M.data_ptr(),
           sb.data_ptr(), scal.data_ptr(), ws.data_ptr(), ws.numel(), D.stream_ptr())
    return {"M": M, "sel_b": sb[:k_cyc], "scalars": scal, "ws": ws}


def mixed_first_order_multiply(A, B, k_svd: int, k_cyc: int, order: int, seed,
                               power_iterations: int = 0, model: ErrorModel | None = None,
                               force_sel_b=None, split3: bool = False, out=None, direct: bool = False):
    """Approximate A @ B with A truncated by randomized SVD (rank k_svd, svd.py:83-119) and B by
    its k_cyc dominant cycles (config C4). Returns (M, ApproxReport(method="mixed")).
    ``direct``: see mixed_product_device."""
    Ad, _, host = D.as_device_matrix(A, real_only=True)
    Bd, _, _ = D.as_device_matrix(B, real_only=True)
    n = Ad.shape[0]
    if Ad.shape[1] != n or tuple(Bd.shape) != (n, n):
        raise ValueError(f"two square n x n matrices required, got {tuple(Ad.shape)} x {tuple(Bd.shape)}")
    if Bd.dtype != Ad.dtype:
        Bd = Bd.to(Ad.dtype)
    if order not in (0, 1):
        raise ValueError("order must be 0 or 1")
    if not 1 <= k_svd <= n or not 0 <= k_cyc <= n:
        raise ValueError("component counts out of range")
    if power_iterations < 0:
        raise ValueError("power_iterations must be >= 0")
    omega = torch.from_numpy(draw_sketch(n, k_svd, seed)).to(device=Ad.device, dtype=Ad.dtype)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = mixed_product_device(Ad, Bd, k_svd, k_cyc, order, omega, power_iterations, force_sel_b, split3,
                             direct=direct)
    s = r["scalars"].tolist()
    wall = time.perf_counter() - t0
    nA, nB, ndA, ndB, nM = _norms(s, n * n)
    rep = finish_report("mixed", order, k_svd, nA, nB, ndA, ndB, nM, n, wall, model)
    rep.selected_b = r["sel_b"].tolist()
    return D.to_user(r["M"], host, out), rep
