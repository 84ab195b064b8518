"""Device time of one C3 product (circulant fp64 n=4096, k=16, order 1), inputs resident in HBM;
A/B runs of kernel variants set their environment switch before the call."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
from paper_2504_19308_b200 import circulant as PC  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
A = torch.from_numpy(O.gen_circulant_operand(n, 16, 1)).cuda()
B = torch.from_numpy(O.gen_circulant_operand(n, 16, 2)).cuda()
for _ in range(2):
    PC.circulant_product_device(A, B, 1, 16, 1)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(5):
    PC.circulant_product_device(A, B, 1, 16, 1)
e.record()
torch.cuda.synchronize()
print(f"C3 n={n} {s.elapsed_time(e) / 5:.3f} ms (APX_CIRC_DA_INLINE={os.environ.get('APX_CIRC_DA_INLINE', '0')})")
