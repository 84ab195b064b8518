"""Batched independent products on one device: many small products (config C1, n = 512) are each
a chain of ~40 latency-bound kernels that occupy a handful of SMs, so one product at a time
leaves the GPU mostly idle. ``GraphBatch`` launches B independent device-level calls on S
streams inside one CUDA graph (captured once, replayed per batch): the chains run concurrently
and the host pays one graph launch per batch instead of B x 40 kernel launches.

Every device-level entry point of the C-ABI is stream-ordered with a caller-owned workspace and
no global state (include/apx.h), so concurrent calls on different streams are independent.
"""

from __future__ import annotations

from typing import Callable, Sequence

import torch

from . import _device as D
from . import _native as N

__all__ = ["GraphBatch", "SvdProductBatch"]


class GraphBatch:
    """Capture ``calls`` (each a zero-argument function issuing device work on the current
    stream) round-robin over ``streams`` streams into one CUDA graph; ``replay()`` runs them all.
    The calls must only touch preallocated device memory (no allocation, no host copies)."""

    def __init__(self, calls: Sequence[Callable[[], None]], streams: int = 16, warmup: bool = True):
        D.require_cuda()
        self.calls = list(calls)
        self.streams = [torch.cuda.Stream() for _ in range(max(1, min(streams, len(self.calls))))]
        if warmup:  # first calls outside capture (lazy module loads, smem attributes)
            for fn in self.calls[: len(self.streams)]:
                fn()
            torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            cur = torch.cuda.current_stream()
            for i, fn in enumerate(self.calls):
                s = self.streams[i % len(self.streams)]
                s.wait_stream(cur)
                with torch.cuda.stream(s):
                    fn()
            for s in self.streams:
                cur.wait_stream(s)

    def replay(self) -> None:
        self.graph.replay()


class SvdProductBatch:
    """B independent rSVD-truncated products M_b = A_b.B_b (svd_first_order_multiply, fp64) of
    one shape, run as a GraphBatch. Omegas are the caller's sketches (drawn per product with the
    reference's seeds, svd.py:161-162). Outputs: ``M`` (B x m x p) and ``scalars``."""

    def __init__(self, A: torch.Tensor, B: torch.Tensor, la: int, ka: int, lb: int, kb: int, q: int, order: int,
                 omega_a: torch.Tensor, omega_b: torch.Tensor, streams: int = 16):
        if A.dim() != 3 or B.dim() != 3 or A.shape[0] != B.shape[0]:
            raise ValueError("A, B: batched (B x m x n, B x n x p) device tensors")
        if A.dtype != torch.float64 or B.dtype != torch.float64:
            raise ValueError("fp64 operands required")
        nb, m, n = A.shape
        p = B.shape[2]
        if B.shape[1] != n:
            raise ValueError(f"dimension mismatch: {tuple(A.shape)} x {tuple(B.shape)}")
        if order not in (0, 1):
            raise ValueError("order must be 0 or 1")
        dev = A.device
        self.A, self.B = A.contiguous(), B.contiguous()
        self.oa = omega_a.to(dev, torch.float64).contiguous()
        self.ob = omega_b.to(dev, torch.float64).contiguous()
        self.M = torch.empty((nb, m, p), dtype=torch.float64, device=dev)
        self.scalars = torch.zeros((nb, N.NSCALARS), dtype=torch.float64, device=dev)
        wsz = N.size("apx_svd_first_order_workspace", N.APX_F64, m, n, p, la, lb)
        self.ws = [D.workspace(wsz) for _ in range(nb)]

        def make(b):
            def fn():
                N.call("apx_svd_first_order", N.APX_F64, self.A[b].data_ptr(), self.B[b].data_ptr(), m, n, p, la,
                       ka, lb, kb, q, order, self.oa[b].data_ptr(), self.ob[b].data_ptr(), self.M[b].data_ptr(),
                       self.scalars[b].data_ptr(), self.ws[b].data_ptr(), self.ws[b].numel(), D.stream_ptr())
            return fn

        self.batch = GraphBatch([make(b) for b in range(nb)], streams=streams)

    def run(self) -> torch.Tensor:
        self.batch.replay()
        return self.M
