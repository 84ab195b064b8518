"""One C3 circulant product (fp64 n=4096, k=16, order 1) for ncu launch lists."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import oracle as O  # noqa: E402
from paper_2504_19308_b200 import circulant as PC  # noqa: E402

n = int(os.environ.get("C3_N", 4096))
A = torch.from_numpy(O.gen_circulant_operand(n, 16, 5)).cuda()
B = torch.from_numpy(O.gen_circulant_operand(n, 16, 6)).cuda()
PC.circulant_product_device(A, B, 1, 16, 1)
torch.cuda.synchronize()
print("ok")
