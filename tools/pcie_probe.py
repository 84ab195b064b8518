"""PCIe copy bandwidth with pinned host buffers: H2D, D2H, and both directions concurrently."""
import json
import time

import torch

n = 256 * 1024 * 1024 // 4
h1 = torch.empty(n, dtype=torch.float32, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
d1 = torch.empty(n, dtype=torch.float32, device="cuda")
d2 = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
out = {}


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


b = n * 4
out["h2d_GBs"] = b / timed(lambda: d1.copy_(h1, non_blocking=True)) / 1e9
out["d2h_GBs"] = b / timed(lambda: h2.copy_(d2, non_blocking=True)) / 1e9


def both():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


out["duplex_GBs_each"] = b / timed(both) / 1e9
print(json.dumps(out))
