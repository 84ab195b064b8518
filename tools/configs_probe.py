"""Device time of one product for the secondary BASELINE configs (C1, C2, C3, C5) through the
device-level entry points, inputs resident in HBM (parity for these lives in tests/)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2504_19308_b200 as P  # noqa: E402
from paper_2504_19308_b200 import circulant as PC  # noqa: E402
from paper_2504_19308_b200 import svd as PS  # noqa: E402


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


out = {}
dev = torch.device("cuda", 0)
# C1: rSVD fp64 n=512, l=40 -> k=32, q=2, order 0
n = 512
A = torch.from_numpy(O.gen_haar_spectrum(n, 0.9 ** np.arange(n), 1)).to(dev)
B = torch.from_numpy(O.gen_haar_spectrum(n, 0.9 ** np.arange(n), 2)).to(dev)
oa = np.random.default_rng([0, 0]).standard_normal((n, 40))
ob = np.random.default_rng([0, 1]).standard_normal((n, 40))
out["C1_ms"] = timed(lambda: PS.svd_product_device(A, B, 40, 32, 40, 32, 2, 0, oa, ob))
# C1 batched: NB independent products per CUDA-graph replay, concurrent on S streams (batch.py)
NB = int(os.environ.get("C1_BATCH", 128))
sig = 0.9 ** np.arange(n)
Ab = torch.from_numpy(np.stack([O.gen_haar_spectrum(n, sig, 2 * t) for t in range(NB)])).to(dev)
Bb = torch.from_numpy(np.stack([O.gen_haar_spectrum(n, sig, 2 * t + 1) for t in range(NB)])).to(dev)
oab = torch.from_numpy(np.stack([np.random.default_rng([t, 0]).standard_normal((n, 40)) for t in range(NB)]))
obb = torch.from_numpy(np.stack([np.random.default_rng([t, 1]).standard_normal((n, 40)) for t in range(NB)]))
best = None
for S in (16, 32, 64):
    bt = P.SvdProductBatch(Ab, Bb, 40, 32, 40, 32, 2, 0, oab, obb, streams=S)
    ms = timed(bt.run, reps=5, warm=2)
    out[f"C1_batch{NB}_s{S}_ms"] = ms
    best = ms if best is None else min(best, ms)
    del bt
out["C1_batch_products_per_s"] = NB / (best * 1e-3)
del Ab, Bb
# C2: cycle fp64 n=2048, k=32, order 1
n = 2048
A = torch.from_numpy(O.gen_cycle_operand(n, 32, 3)).to(dev)
B = torch.from_numpy(O.gen_cycle_operand(n, 32, 4)).to(dev)
out["C2_ms"] = timed(lambda: P.cycle_product_device(A, B, 32, 32, 1))
# C2 batched: NB2 independent products per CUDA-graph replay on 8 streams (batch.py)
NB2 = 16
A2 = [torch.from_numpy(O.gen_cycle_operand(n, 32, 100 + 2 * t)).to(dev) for t in range(NB2)]
B2 = [torch.from_numpy(O.gen_cycle_operand(n, 32, 101 + 2 * t)).to(dev) for t in range(NB2)]
bt = P.GraphBatch([(lambda a, b: (lambda: P.cycle_product_device(a, b, 32, 32, 1)))(a, b) for a, b in zip(A2, B2)],
                  streams=8)
ms = timed(bt.replay, reps=5, warm=2)
out[f"C2_batch{NB2}_ms"] = ms
out["C2_batch_products_per_s"] = NB2 / (ms * 1e-3)
del bt, A2, B2
# C3: circulant fp64 n=4096, k=16, order 1
n = 4096
A = torch.from_numpy(O.gen_circulant_operand(n, 16, 5)).to(dev)
B = torch.from_numpy(O.gen_circulant_operand(n, 16, 6)).to(dev)
out["C3_ms"] = timed(lambda: PC.circulant_product_device(A, B, 1, 16, 1), reps=3)
del A, B
torch.cuda.empty_cache()
# C5: cycle fp32 n=32768, k=128, order 1 (device generator)
from devgen import c5_operand  # noqa: E402
A, _ = c5_operand(32768, 128, 32, seed=5, operand=0)
B, _ = c5_operand(32768, 128, 32, seed=5, operand=1)
out["C5_cycle_ms"] = timed(lambda: P.cycle_product_device(A, B, 128, 128, 1), reps=2, warm=1)
# C5 secondary: circulant k=32 on the same operands (fp64 on the device, four-step transforms)
from paper_2504_19308_b200 import _native as NT  # noqa: E402
A, B = A.double(), B.double()
torch.cuda.empty_cache()
out["C5_circ_ms"] = timed(lambda: PC.circulant_product_device(A, B, NT.APX_F64, 32, 1), reps=2, warm=1)
print(json.dumps(out))
