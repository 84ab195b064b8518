"""One C1 rSVD product (fp64 n=512, l=40 -> k=32, q=2, order 0) for ncu launch lists."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
from paper_2504_19308_b200 import svd as PS  # noqa: E402

n = 512
A = torch.from_numpy(O.gen_haar_spectrum(n, 0.9 ** np.arange(n), 1)).cuda()
B = torch.from_numpy(O.gen_haar_spectrum(n, 0.9 ** np.arange(n), 2)).cuda()
oa = np.random.default_rng([0, 0]).standard_normal((n, 40))
ob = np.random.default_rng([0, 1]).standard_normal((n, 40))
PS.svd_product_device(A, B, 40, 32, 40, 32, 2, 0, oa, ob)
torch.cuda.synchronize()
print("ok")
