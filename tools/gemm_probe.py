"""Solo timing of the C4 product's n x n GEMM shapes through the debug hook (apx_debug_umma_gemm):
M (+)= Q2 . W2 (n x 128 . 128 x n), one-tile-per-CTA kernel vs the persistent kernel.
    python tools/gemm_probe.py [--n 8192] [--k 128]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2504_19308_b200 import _native as N  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--k", type=int, default=128)
a = ap.parse_args()
n, k = a.n, a.k
dev = torch.device("cuda", 0)
Q = torch.randn(n, k, device=dev)
W = torch.randn(k, n, device=dev)
C = torch.randn(n, n, device=dev)
tk = torch.zeros(4, dtype=torch.int32, device=dev)


def call(layout, bn, acc, ctas=0):
    N.call("apx_debug_umma_gemm", layout, bn, Q.data_ptr(), k, W.data_ptr(), n, C.data_ptr(), n, n, n, k, 1, acc,
           tk.data_ptr() if layout & 128 else None, 0, ctas, None)


def timeit(f, reps=20):
    for _ in range(3):
        f()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        f()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


# Y = A . Omega (n x n . n x 64, 4-way split-K as the residual plan launches it)
A = torch.randn(n, n, device=dev)
Om = torch.randn(n, 64, device=dev)
Yp = torch.empty(4, n, 64, device=dev)
for sp in (1, 2, 4):
    us = timeit(lambda: N.call("apx_debug_umma_gemm", 32 | 2, 64, A.data_ptr(), n, Om.data_ptr(), 64, Yp.data_ptr(),
                               64, n, 64, n, sp, 0, None, 0, 1, None))
    print(f"Y = A.Omega split {sp}: {us:8.1f} us  {4 * n * n / us / 1e3:7.0f} GB/s")
del A
for acc in (0, 1):
    by = (8 if acc else 4) * n * n
    for name, f in [("tile bn128" if acc else "tile bn256", lambda: call(32 | 2, 128 if acc else 256, acc)),
                    ("persist bn128 static", lambda: call(64 | 2, 128, acc)),
                    ("persist bn128 dynamic", lambda: call(128 | 64 | 2, 128, acc)),
                    ("persist bn64 dynamic", lambda: call(128 | 64 | 2, 64, acc))]:
        us = timeit(f)
        print(f"acc={acc} {name:24s} {us:8.1f} us  {by / us / 1e3:7.0f} GB/s")
