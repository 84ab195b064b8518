"""C4 product: eager launches vs one CUDA-graph replay per product (same buffers)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2504_19308_b200 as P  # noqa: E402

n = 8192
dev = torch.device("cuda", 0)
A, B = bench.gen_c4(n, 1234, dev)
omega = torch.from_numpy(P.cycle.draw_sketch(n, 64, 7)).to(dev, torch.float32)
M = torch.empty_like(A)


def step():
    return P.mixed_product_device(A, B, 64, 64, 1, omega, 0, None, False, out=M)


for _ in range(3):
    r = step()
torch.cuda.synchronize()
ref = M.clone()


def timeit(fn, reps=20):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


eager = timeit(step)
# capture: the C-ABI call allocates nothing; its workspace / outputs must outlive the graph
ws_hold = []
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    step()  # one more warm call on the capture stream
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
with torch.cuda.graph(g):
    ws_hold.append(step())
g.replay()
torch.cuda.synchronize()
same = bool(torch.equal(M, ref))
graph = timeit(g.replay)
print(json.dumps({"eager_ms": eager, "graph_ms": graph, "bitwise_equal": same}))
