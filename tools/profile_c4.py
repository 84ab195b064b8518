"""One C4 product (after warm-up) for ncu launch lists / captures.

    python tools/profile_c4.py [--n 8192] [--reps 1] [--split3 0] [--direct 0]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2504_19308_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--split3", type=int, default=0)
ap.add_argument("--direct", type=int, default=0, help="1: the all-fp32 plan (gather over A)")
a = ap.parse_args()
dev = torch.device("cuda", 0)
A, B = bench.gen_c4(a.n, 1234, dev)
omega = torch.from_numpy(P.cycle.draw_sketch(a.n, 64, 7)).to(dev, torch.float32)
M = torch.empty_like(A)
for _ in range(a.warmup):
    P.mixed_product_device(A, B, 64, 64, 1, omega, 0, None, bool(a.split3), out=M, direct=bool(a.direct))
torch.cuda.synchronize()
for _ in range(a.reps):
    P.mixed_product_device(A, B, 64, 64, 1, omega, 0, None, bool(a.split3), out=M, direct=bool(a.direct))
torch.cuda.synchronize()
print("ok", float(M.double().norm()))
