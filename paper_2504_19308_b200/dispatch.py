"""String dispatch of one product -- GPU mirror of the reference's only plugin mechanism,
``cli.run_method`` (pkg/src/apxmm/cli.py:138-158): same method names, keyword arguments, return
value (M, ApproxReport) and ValueError for an unknown method. Every product runs on the device.

Extensions beyond the reference: "cycle" (restated cycle product, configs C2/C5) and "mixed"
(rSVD x cycles, config C4). "lowrank" (``baseline.randomized_outer_product_multiply``) is the
reference's CPU baseline, outside the hot path: it raises NotImplementedError.
"""

from __future__ import annotations

import time

from .circulant import circulant_first_order_multiply
from .core import matmul_naive
from .cycle import cycle_first_order_multiply, mixed_first_order_multiply
from .fsparse import fft_sparse_first_order_multiply
from .report import ApproxReport
from .svd import svd_first_order_multiply

__all__ = ["METHODS", "run_method"]

METHODS = ("naive", "svd", "cd", "sfft", "cycle", "mixed")


def run_method(method: str, order: int, A, B, *, s: int | None = None, k: int | None = None,
               c: int | None = None, seed: int = 0, power_iterations: int = 0,
               sparsify_b: str = "rows", k_svd: int | None = None):
    """Dispatch one approximate (or exact) product. Returns (M, report).

    cli.py:138-158 argument meaning: ``s`` drives the svd component count, ``k`` the circulant /
    sfft / cycle budget, ``seed`` the sketch streams, ``sparsify_b`` the sfft mode. "mixed" uses
    ``k_svd`` (default ``k``) sketch columns for A and ``k`` cycles for B."""
    if method == "naive":
        t0 = time.perf_counter()
        M = matmul_naive(A, B)
        wall = time.perf_counter() - t0
        return M, ApproxReport(method="naive", order=0, k=0, norm_da=0.0, norm_db=0.0, wall_time=wall)
    if method == "lowrank":
        raise NotImplementedError("'lowrank' is the reference's CPU baseline "
                                  "(baseline.randomized_outer_product_multiply), not on the GPU path")
    if method == "svd":
        return svd_first_order_multiply(A, B, s, order, seed, power_iterations=power_iterations)
    if method == "cd":
        return circulant_first_order_multiply(A, B, k, order)
    if method == "sfft":
        return fft_sparse_first_order_multiply(A, B, k, order, sparsify_b=sparsify_b)
    if method == "cycle":
        return cycle_first_order_multiply(A, B, k, order)
    if method == "mixed":
        return mixed_first_order_multiply(A, B, k if k_svd is None else k_svd, k, order, seed,
                                          power_iterations=power_iterations)
    raise ValueError(f"unknown method {method!r}")
