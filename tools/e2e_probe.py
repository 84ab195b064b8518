"""e2e (host-to-host) C4 throughput through MixedPipeline for both plans, and the pieces: H2D of
one product's operands alone, the product alone, D2H alone.  python tools/e2e_probe.py"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2504_19308_b200 as P  # noqa: E402

n = 8192
dev = torch.device("cuda", 0)
A, B = bench.gen_c4(n, 1234, dev)
Ah = torch.empty((n, n), dtype=torch.float32, pin_memory=True)
Bh = torch.empty((n, n), dtype=torch.float32, pin_memory=True)
Mh = [torch.empty((n, n), dtype=torch.float32, pin_memory=True) for _ in range(3)]
Ah.copy_(A)
Bh.copy_(B)
out = {}
for direct in (False, True):
    pipe = P.MixedPipeline(n, 64, 64, 1, depth=3, direct=direct)
    for i in range(2):
        pipe.result(pipe.submit(Ah, Bh, 7, out=Mh[i % 3]))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tk = [pipe.submit(Ah, Bh, 7, out=Mh[i % 3]) for i in range(12)]
    for t in tk:
        pipe.result(t)
    torch.cuda.synchronize()
    out["direct" if direct else "resid"] = 12 / (time.perf_counter() - t0)
    del pipe
s = torch.cuda.Stream()
Ad = torch.empty_like(A)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    Ad.copy_(Ah, non_blocking=True)
torch.cuda.synchronize()
out["h2d_GBs"] = 5 * Ah.numel() * 4 / (time.perf_counter() - t0) / 1e9
t0 = time.perf_counter()
for _ in range(12):
    P.cycle.draw_sketch(n, 64, 7)
out["draw_sketch_ms"] = (time.perf_counter() - t0) / 12 * 1e3
print(json.dumps(out))
