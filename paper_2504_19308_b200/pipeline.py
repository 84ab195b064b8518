"""Pipelined host-to-host mixed products (config C4 served from host memory).

A single call of ``mixed_first_order_multiply`` on pinned host tensors is PCIe-serial: H2D of A
and B (539 MB at n = 8192), the product (~1.1 ms), then D2H of M (268 MB). ``MixedPipeline``
keeps ``depth`` sets of device buffers and three streams (H2D, compute, D2H) so that product i's
result streams back while product i+1's operands stream in (PCIe is full duplex) and product
i+1 computes while product i+2 loads. Every product still copies its full inputs in and its full
result out; nothing is cached between submissions. The numerics are exactly those of
``mixed_first_order_multiply`` (same C-ABI call, same host-drawn sketch).

    pipe = MixedPipeline(n, k_svd=64, k_cyc=64, order=1)
    tickets = [pipe.submit(A_i, B_i, seed_i, out=M_i) for ...]   # pinned host torch tensors
    M, report = pipe.result(tickets[0])
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from . import _native as N
from .cycle import _norms, draw_sketch
from .errest import ErrorModel, finish_report

__all__ = ["MixedPipeline"]


@dataclass
class _Slot:
    A: torch.Tensor
    B: torch.Tensor
    M: torch.Tensor
    omega: torch.Tensor
    omega_host: torch.Tensor
    ws: torch.Tensor
    scal: torch.Tensor
    sel: torch.Tensor
    scal_host: torch.Tensor
    sel_host: torch.Tensor
    ev_in: torch.cuda.Event
    ev_start: torch.cuda.Event
    ev_comp: torch.cuda.Event
    ev_out: torch.cuda.Event
    pending: "Ticket | None" = None


@dataclass
class Ticket:
    slot: int
    seq: int
    out: torch.Tensor
    done: tuple | None = None  # (scalars, selection, device seconds) once collected


class MixedPipeline:
    """Depth-``depth`` pipeline of fp32 mixed products (rSVD rank ``k_svd`` x ``k_cyc`` cycles)."""

    def __init__(self, n: int, k_svd: int, k_cyc: int, order: int = 1, depth: int = 2,
                 power_iterations: int = 0, split3: bool = False, dtype=torch.float32,
                 model: ErrorModel | None = None, direct: bool = False):
        if order not in (0, 1):
            raise ValueError("order must be 0 or 1")
        if not 1 <= k_svd <= n or not 0 <= k_cyc <= n:
            raise ValueError("component counts out of range")
        if power_iterations < 0:
            raise ValueError("power_iterations must be >= 0")
        if dtype not in (torch.float32, torch.float64):
            raise ValueError(f"unsupported dtype {dtype}")
        self.dev = D.require_cuda()
        self.n, self.k_svd, self.k_cyc, self.order = n, k_svd, k_cyc, order
        self.q, self.split3, self.dtype, self.model = power_iterations, split3, dtype, model
        self.flags = (1 if split3 else 0) | (4 if direct else 0)  # direct: the all-fp32 plan
        self.code = N.APX_F32 if dtype == torch.float32 else N.APX_F64
        wsb = N.size("apx_mixed_first_order_workspace", self.code, n, k_svd, k_cyc, order)
        self.slots = []
        for _ in range(max(1, depth)):
            self.slots.append(_Slot(
                A=torch.empty((n, n), dtype=dtype, device=self.dev),
                B=torch.empty((n, n), dtype=dtype, device=self.dev),
                M=torch.empty((n, n), dtype=dtype, device=self.dev),
                omega=torch.empty((n, k_svd), dtype=dtype, device=self.dev),
                omega_host=torch.empty((n, k_svd), dtype=dtype, pin_memory=True),
                ws=D.workspace(wsb),
                scal=torch.zeros(N.NSCALARS, dtype=torch.float64, device=self.dev),
                sel=torch.zeros(max(k_cyc, 1), dtype=torch.int32, device=self.dev),
                scal_host=torch.empty(N.NSCALARS, dtype=torch.float64, pin_memory=True),
                sel_host=torch.empty(max(k_cyc, 1), dtype=torch.int32, pin_memory=True),
                ev_in=torch.cuda.Event(), ev_start=torch.cuda.Event(enable_timing=True),
                ev_comp=torch.cuda.Event(enable_timing=True), ev_out=torch.cuda.Event()))
        self.s_in = torch.cuda.Stream(device=self.dev)
        self.s_comp = torch.cuda.Stream(device=self.dev)
        self.s_out = torch.cuda.Stream(device=self.dev)
        self.seq = 0

    def _check_host(self, X, name):
        if not isinstance(X, torch.Tensor) or X.is_cuda:
            raise ValueError(f"{name}: a host torch tensor is required (pinned for overlap)")
        if tuple(X.shape) != (self.n, self.n) or X.dtype != self.dtype:
            raise ValueError(f"{name}: expected {self.n} x {self.n} {self.dtype}, got {tuple(X.shape)} {X.dtype}")

    def submit(self, A, B, seed, out: torch.Tensor | None = None) -> Ticket:
        """Enqueue one product; returns at once (blocks only while all ``depth`` slots are busy)."""
        self._check_host(A, "A")
        self._check_host(B, "B")
        if out is None:
            out = torch.empty((self.n, self.n), dtype=self.dtype, pin_memory=True)
        self._check_host(out, "out")
        # host work first (the reference's sketch stream, ~6 ms at n = 8192): it overlaps the
        # device work already queued, before this call can block on a busy slot
        omega = torch.from_numpy(np.ascontiguousarray(draw_sketch(self.n, self.k_svd, seed)))
        i = self.seq % len(self.slots)
        sl = self.slots[i]
        if sl.pending is not None:  # the slot's previous product must have fully left the device
            self._collect(sl)
        sl.omega_host.copy_(omega)
        with torch.cuda.stream(self.s_in):
            sl.A.copy_(A, non_blocking=True)
            sl.B.copy_(B, non_blocking=True)
            sl.omega.copy_(sl.omega_host, non_blocking=True)
            sl.ev_in.record(self.s_in)
        with torch.cuda.stream(self.s_comp):
            self.s_comp.wait_event(sl.ev_in)
            sl.ev_start.record(self.s_comp)
            N.call("apx_mixed_first_order", self.code, sl.A.data_ptr(), sl.B.data_ptr(), self.n, self.k_svd,
                   self.k_cyc, self.order, self.q, sl.omega.data_ptr(), None, self.flags,
                   sl.M.data_ptr(), sl.sel.data_ptr(), sl.scal.data_ptr(), sl.ws.data_ptr(), sl.ws.numel(),
                   self.s_comp.cuda_stream)
            sl.ev_comp.record(self.s_comp)
        with torch.cuda.stream(self.s_out):
            self.s_out.wait_event(sl.ev_comp)
            out.copy_(sl.M, non_blocking=True)
            sl.scal_host.copy_(sl.scal, non_blocking=True)
            sl.sel_host.copy_(sl.sel, non_blocking=True)
            sl.ev_out.record(self.s_out)
        t = Ticket(slot=i, seq=self.seq, out=out)
        sl.pending = t
        self.seq += 1
        return t

    def _collect(self, sl: _Slot) -> None:
        sl.ev_out.synchronize()
        t = sl.pending
        t.done = (sl.scal_host.tolist(), sl.sel_host[:self.k_cyc].tolist(),
                  sl.ev_start.elapsed_time(sl.ev_comp) * 1e-3)
        sl.pending = None

    def result(self, t: Ticket):
        """(M on the host, ApproxReport) of a submitted product; waits for its D2H."""
        if t.done is None:
            self._collect(self.slots[t.slot])
        s, sel, wall = t.done  # wall: device time of the product
        nA, nB, ndA, ndB, nM = _norms(s, self.n * self.n)
        rep = finish_report("mixed", self.order, self.k_svd, nA, nB, ndA, ndB, nM, self.n, wall, self.model)
        rep.selected_b = sel
        return t.out, rep
