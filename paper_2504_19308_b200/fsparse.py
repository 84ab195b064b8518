"""Row-wise Fourier sparsification and the sparsified approximate product -- GPU drop-in for the
reference module ``apxmm.fsparse`` (pkg/src/apxmm/fsparse.py). The transforms, per-row top-k
selection and sparse/dense products run in the C-ABI (apx_sfft_first_order, apx_topk_rows,
apx_sparse_rows_multiply, apx_unitary_dft); SparseRowMatrix keeps the reference's host
representation (per-row lists of (column, value))."""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from . import _native as N
from .core import unitary_dft
from .errest import ErrorModel, finish_report

__all__ = [
    "SparseRowMatrix",
    "FourierRowSpectrum",
    "fourier_row_decompose",
    "topk_sparsify",
    "sparse_dense_multiply",
    "fft_sparse_first_order_multiply",
]


@dataclass
class SparseRowMatrix:
    """fsparse.py:33-68 -- entries[i] = [(column, value), ...], columns strictly increasing."""

    rows: int
    cols: int
    entries: list

    def __post_init__(self):
        if self.rows < 0 or self.cols < 0:
            raise ValueError("negative dimensions")
        if len(self.entries) != self.rows:
            raise ValueError("need one entry list per row")
        for i, row in enumerate(self.entries):
            last = -1
            for j, _ in row:
                if not 0 <= j < self.cols:
                    raise ValueError(f"column {j} out of range in row {i}")
                if j <= last:
                    raise ValueError(f"row {i} columns not strictly increasing")
                last = j

    @property
    def nnz(self) -> int:
        return sum(len(r) for r in self.entries)

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.rows, self.cols), dtype=np.complex128)
        for i, row in enumerate(self.entries):
            for j, v in row:
                out[i, j] = v
        return out


@dataclass
class FourierRowSpectrum:
    """fsparse.py:71-89."""

    weights: np.ndarray
    directions: np.ndarray

    def __post_init__(self):
        if self.weights.ndim != 1 or self.directions.ndim != 2:
            raise ValueError("weights must be 1-D, directions 2-D")
        if self.directions.shape[1] != self.weights.size:
            raise ValueError("one direction column per weight required")
        if np.any(self.weights < 0):
            raise ValueError("weights must be nonnegative")


def fourier_row_decompose(A) -> FourierRowSpectrum:
    """fsparse.py:92-105 -- F = W(rows)/sqrt(n), weights sqrt(n)||f_k||, unit directions (zero
    column where the weight vanishes): one row-DFT pass and one column pass on the device
    (apx_fourier_row_decompose)."""
    Ah = D.as_host_matrix(A)
    m, n = Ah.shape
    cplx = np.iscomplexobj(Ah)
    dev = D.require_cuda()
    Ad = torch.from_numpy(np.ascontiguousarray(Ah.astype(np.complex128 if cplx else np.float64))).to(dev)
    weights = torch.empty(n, dtype=torch.float64, device=dev)
    directions = torch.empty((m, n), dtype=torch.complex128, device=dev)
    ws = D.workspace(N.size("apx_fourier_row_decompose_workspace", m, n))
    N.call("apx_fourier_row_decompose", N.APX_C128 if cplx else N.APX_F64, Ad.data_ptr(), m, n, weights.data_ptr(),
           directions.data_ptr(), ws.data_ptr(), ws.numel(), D.stream_ptr())
    return FourierRowSpectrum(weights=weights.cpu().numpy(), directions=directions.cpu().numpy())


def _row_budgets(k, rows: int, cols: int) -> list[int]:
    """fsparse.py:108-118."""
    if np.isscalar(k):
        if k < 0:
            raise ValueError("k must be >= 0")
        return [min(int(k), cols)] * rows
    ks = [int(v) for v in k]
    if len(ks) != rows:
        raise ValueError(f"need one budget per row, got {len(ks)} for {rows} rows")
    if any(v < 0 for v in ks):
        raise ValueError("budgets must be >= 0")
    return [min(v, cols) for v in ks]


def _topk_device(Md: torch.Tensor, budgets: list[int]):
    rows, cols = Md.shape
    kmax = max(budgets) if budgets else 0
    if kmax == 0:
        return np.full((rows, 0), -1, np.int32), np.zeros((rows, 0), np.complex128)
    dev = Md.device
    bud = torch.tensor(budgets, dtype=torch.int32, device=dev)
    sel = torch.empty((rows, kmax), dtype=torch.int32, device=dev)
    vals = torch.empty((rows, kmax), dtype=torch.complex128, device=dev)
    ws = D.workspace(N.size("apx_topk_rows_workspace", rows, cols))
    N.call("apx_topk_rows", Md.data_ptr(), rows, cols, kmax, bud.data_ptr(), sel.data_ptr(), vals.data_ptr(),
           ws.data_ptr(), ws.numel(), D.stream_ptr())
    return sel.cpu().numpy(), vals.cpu().numpy()


def topk_sparsify(M, k) -> SparseRowMatrix:
    """fsparse.py:121-139 -- keep the k largest-modulus entries of each row (ties -> lower
    column; k clamped; per-row budgets allowed)."""
    M = D.as_host_matrix(M)
    rows, cols = M.shape
    budgets = _row_budgets(k, rows, cols)
    dev = D.require_cuda()
    Md = torch.from_numpy(np.ascontiguousarray(M.astype(np.complex128))).to(dev)
    sel, vals = _topk_device(Md, budgets)
    entries = []
    for i in range(rows):
        entries.append([(int(j), complex(v)) for j, v in zip(sel[i], vals[i]) if j >= 0])
    return SparseRowMatrix(rows=rows, cols=cols, entries=entries)


def _to_slots(S: SparseRowMatrix):
    k = max((len(r) for r in S.entries), default=0)
    sel = np.full((S.rows, max(k, 1)), -1, np.int32)
    vals = np.zeros((S.rows, max(k, 1)), np.complex128)
    for i, row in enumerate(S.entries):
        for q, (j, v) in enumerate(row):
            sel[i, q] = j
            vals[i, q] = v
    return sel, vals, max(k, 1)


def _left_multiply(S: SparseRowMatrix, X: np.ndarray) -> np.ndarray:
    dev = D.require_cuda()
    sel, vals, k = _to_slots(S)
    Xd = torch.from_numpy(np.ascontiguousarray(X, dtype=np.complex128)).to(dev)
    p = X.shape[1]
    out = torch.empty((S.rows, p), dtype=torch.complex128, device=dev)
    seld = torch.from_numpy(sel).to(dev)  # keep the device copies alive until the kernel ran
    valsd = torch.from_numpy(vals).to(dev)
    N.call("apx_sparse_rows_multiply", seld.data_ptr(), valsd.data_ptr(), k, S.rows, Xd.data_ptr(), p,
           out.data_ptr(), D.stream_ptr())
    torch.cuda.synchronize()
    return out.cpu().numpy()


def sparse_dense_multiply(S: SparseRowMatrix, B, side: str = "left") -> np.ndarray:
    """fsparse.py:142-165 -- S @ B (left) or B @ S (right) without densifying S."""
    B = D.as_host_matrix(B)
    if side == "left":
        if S.cols != B.shape[0]:
            raise ValueError(f"dimension mismatch: ({S.rows},{S.cols}) x {B.shape}")
        if S.rows == 0:
            return np.zeros((0, B.shape[1]), dtype=np.complex128)
        return _left_multiply(S, B)
    if side == "right":
        if B.shape[1] != S.rows:
            raise ValueError(f"dimension mismatch: {B.shape} x ({S.rows},{S.cols})")
        # B S = (S^T B^T)^T with S^T re-bucketed by its rows (host bookkeeping only)
        buckets = [[] for _ in range(S.cols)]
        for i, row in enumerate(S.entries):
            for j, v in row:
                buckets[j].append((i, v))
        St = SparseRowMatrix(rows=S.cols, cols=S.rows, entries=buckets)
        if St.rows == 0:
            return np.zeros((B.shape[0], 0), dtype=np.complex128)
        return _left_multiply(St, np.ascontiguousarray(B.T)).T
    raise ValueError(f"unknown side {side!r}")


def sfft_product_device(Ad, Bd, code, k: int, order: int, sparsify_cols: bool, out=None):
    """Device-level sfft product (apx_sfft_first_order) on device operands Ad (m x n), Bd (n x p)
    of dtype `code` (APX_F64 / APX_C128): dict(M, sel_a, sel_b, scalars, ka, kb, ws)."""
    m, n = Ad.shape
    p = Bd.shape[1]
    dev = Ad.device
    M = out if out is not None else torch.empty((m, p), dtype=torch.complex128, device=dev)
    scal = torch.zeros(N.NSCALARS, dtype=torch.float64, device=dev)
    ws = D.workspace(N.size("apx_sfft_first_order_workspace", m, n, p, k))
    ka = min(k, n)
    kb = min(k, n if sparsify_cols else p)
    sa = torch.full((m, max(ka, 1)), -1, dtype=torch.int32, device=dev)
    sb = torch.full((p if sparsify_cols else n, max(kb, 1)), -1, dtype=torch.int32, device=dev)
    N.call("apx_sfft_first_order", code, Ad.data_ptr(), Bd.data_ptr(), m, n, p, k, order,
           1 if sparsify_cols else 0, M.data_ptr(), sa.data_ptr(), sb.data_ptr(), scal.data_ptr(),
           ws.data_ptr(), ws.numel(), D.stream_ptr())
    return {"M": M, "sel_a": sa, "sel_b": sb, "scalars": scal, "ka": ka, "kb": kb, "ws": ws}


def fft_sparse_first_order_multiply(A, B, k: int, order: int, sparsify_b: str = "rows",
                                    model: ErrorModel | None = None):
    """fsparse.py:168-240 -- approximate A @ B through top-k sparsified Fourier transforms."""
    Ah = D.as_host_matrix(A)
    Bh = D.as_host_matrix(B)
    n = Ah.shape[1]
    if Bh.shape[0] != n:
        raise ValueError(f"dimension mismatch: {Ah.shape} x {Bh.shape}")
    if k < 0:
        raise ValueError(f"k={k} must be >= 0")
    if order not in (0, 1):
        raise ValueError("order must be 0 or 1")
    if sparsify_b not in ("rows", "cols"):
        raise ValueError(f"unknown sparsify_b {sparsify_b!r}")
    cplx = np.iscomplexobj(Ah) or np.iscomplexobj(Bh)
    code = N.APX_C128 if cplx else N.APX_F64
    dt = np.complex128 if cplx else np.float64
    dev = D.require_cuda()
    Ad = torch.from_numpy(np.ascontiguousarray(Ah.astype(dt))).to(dev)
    Bd = torch.from_numpy(np.ascontiguousarray(Bh.astype(dt))).to(dev)
    m = Ah.shape[0]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = sfft_product_device(Ad, Bd, code, k, order, sparsify_b == "cols")
    M, scal, sa, sb, ka, kb = r["M"], r["scalars"], r["sel_a"], r["sel_b"], r["ka"], r["kb"]
    s = scal.tolist()
    wall = time.perf_counter() - t0
    nA, nB = math.sqrt(max(0.0, s[N.S_FRO2_A])), math.sqrt(max(0.0, s[N.S_FRO2_B]))
    ndA, ndB = math.sqrt(max(0.0, s[N.S_RES2_A])), math.sqrt(max(0.0, s[N.S_RES2_B]))
    rep = finish_report("sfft", order, k, nA, nB, ndA, ndB, math.sqrt(max(0.0, s[N.S_FRO2_M])), n, wall, model)
    rep.selected_a = [[int(j) for j in row if j >= 0] for row in sa.cpu().tolist()] if ka else [[]] * m
    rep.selected_b = [[int(j) for j in row if j >= 0] for row in sb.cpu().tolist()] if kb else []
    return M.cpu().numpy(), rep
