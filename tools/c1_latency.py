"""Latency of one C1 product (fp64 n=512, l=40 -> k=32, q=2, order 0) on resident inputs, and of
its stages: device events over 20 products after warm-up."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_19308_b200 import genmat as G  # noqa: E402
from paper_2504_19308_b200 import svd as PS  # noqa: E402

n = 512
dev = torch.device("cuda", 0)
sig = 0.9 ** np.arange(n)
A = G.haar_spectrum(n, sig, 1, dev)
B = G.haar_spectrum(n, sig, 2, dev)
oa = np.random.default_rng([0, 0]).standard_normal((n, 40))
ob = np.random.default_rng([0, 1]).standard_normal((n, 40))
for _ in range(3):
    PS.svd_product_device(A, B, 40, 32, 40, 32, 2, 0, oa, ob)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    PS.svd_product_device(A, B, 40, 32, 40, 32, 2, 0, oa, ob)
e.record()
torch.cuda.synchronize()
print(f"C1 one product: {s.elapsed_time(e) / 20:.3f} ms (includes the per-call workspace/omega H2D)")
