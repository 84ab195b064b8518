"""One C2 cycle product (fp64 n=2048, k=32, order 1) for ncu launch lists."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2504_19308_b200 as P  # noqa: E402

n = 2048
A = torch.from_numpy(O.gen_cycle_operand(n, 32, 3)).cuda()
B = torch.from_numpy(O.gen_cycle_operand(n, 32, 4)).cuda()
P.cycle_product_device(A, B, 32, 32, 1)
torch.cuda.synchronize()
print("ok")
