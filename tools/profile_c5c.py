"""One C5 secondary circulant product (n=32768 fp64 on the device, k=32, order 1) for ncu launch lists."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

from paper_2504_19308_b200 import circulant as PC  # noqa: E402
from paper_2504_19308_b200 import _native as NT  # noqa: E402
from devgen import c5_operand  # noqa: E402

n = int(os.environ.get("C5_N", 32768))
A, _ = c5_operand(n, 128, 32, seed=5, operand=0)
B, _ = c5_operand(n, 128, 32, seed=5, operand=1)
A, B = A.double(), B.double()
torch.cuda.synchronize()
PC.circulant_product_device(A, B, NT.APX_F64, 32, 1)
torch.cuda.synchronize()
print("ok")
