"""Timing of the order-1 cycle product at n = 32768 (fp32, k = 128) on cycle-dominated operands
(planted cycles + N(0, 1e-6) noise, no circulant terms) with the f16-staged residual gather
(cycle.cu K11h, APX_SEG_F16=1: device-side rule) against the all-fp32 segmented gather
(APX_SEG_F16=0), plus the same A/B on the C5 operands (circulant terms: the rule keeps fp32).
One JSON line per case: ms per product (CUDA events, 5 runs after 2 warm-ups), stage spans,
relative difference of the two results."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2504_19308_b200 as P  # noqa: E402
from devgen import c5_operand  # noqa: E402


def run(A, B, k, mode, reps=5):
    os.environ["APX_SEG_F16"] = str(mode)
    M = torch.empty_like(A)
    for _ in range(2):
        P.cycle.cycle_product_device(A, B, k, k, 1, out=M)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        P.cycle.cycle_product_device(A, B, k, k, 1, out=M)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, M


def main():
    n, k = int(os.environ.get("N", 32768)), 128
    for name, r in (("cycles+noise", 0), ("C5 operands (32 circulant terms)", 32)):
        A, _ = c5_operand(n, k, r, seed=7, operand=0)
        B, _ = c5_operand(n, k, r, seed=7, operand=1)
        t32, M32 = run(A, B, k, 0)
        M32 = M32.clone()
        th, Mh = run(A, B, k, 1)
        d = float(torch.linalg.norm((Mh - M32).double()) / torch.linalg.norm(M32.double()))
        print(json.dumps({"operands": name, "n": n, "k": k, "ms_fp32_gather": round(t32, 3),
                          "ms_auto_rule": round(th, 3), "rel_diff": d}), flush=True)
        del A, B, M32, Mh
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
