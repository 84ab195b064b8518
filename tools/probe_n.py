import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, torch, numpy as np
import paper_2504_19308_b200 as P
from paper_2504_19308_b200 import circulant as PC
dev = torch.device("cuda")
for n in (4096, 5000, 6000, 8192, 16384):
    A = torch.randn(n, n, device=dev, dtype=torch.float64)
    try:
        torch.cuda.synchronize(); t = time.perf_counter()
        r = PC.circulant_product_device(A, A, 1, 16, 1)
        torch.cuda.synchronize(); print("circ", n, "ok", round(time.perf_counter() - t, 3))
    except Exception as e:
        print("circ", n, "FAIL", str(e)[:120])
    del A
    torch.cuda.empty_cache()
for n in (8192, 12000, 16384, 32768):
    x = np.random.default_rng(0).standard_normal((n, 2)) + 0j
    try:
        y = P.unitary_dft(x, "forward", axis=0); print("dft", n, "ok", np.abs(y - np.fft.fft(x, axis=0, norm="ortho")).max())
    except Exception as e:
        print("dft", n, "FAIL", str(e)[:120])
