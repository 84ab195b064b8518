"""One C5 cycle product (n=32768 fp32, k=128, order 1) for ncu launch lists / captures."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import paper_2504_19308_b200 as P  # noqa: E402
from devgen import c5_operand  # noqa: E402

n = int(os.environ.get("C5_N", 32768))
r = int(os.environ.get("C5_R", 32))  # circulant terms; 0 = cycle-dominated operands (f16 residual gather)
A, _ = c5_operand(n, 128, r, seed=5, operand=0)
B, _ = c5_operand(n, 128, r, seed=5, operand=1)
torch.cuda.synchronize()
P.cycle_product_device(A, B, 128, 128, 1)
torch.cuda.synchronize()
print("ok")
