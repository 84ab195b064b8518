"""Time the C4 Bm = Q^T A GEMM (tcgen05 TF32, layout 7) alone, with and without the in-smem
TF32 rounding fix-up (layout bit 8), at several split counts / grid sizes."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2504_19308_b200 import _native as N  # noqa: E402

n, l = 8192, 64
dev = torch.device("cuda", 0)
A = torch.randn(n, n, device=dev) / n ** 0.5
Q = torch.linalg.qr(torch.randn(n, l, device=dev, dtype=torch.float64))[0].float()
Q = ((Q.view(torch.int32) + 0x1000) & -8192).view(torch.float32).contiguous()  # TF32-rounded, as the C4 plan stores it
lib = N.lib()
st = torch.cuda.current_stream().cuda_stream
for splits in (1, 2, 4):
    C = torch.zeros(splits, l, n, device=dev)
    for lay in (7 | 32, 7 | 8 | 32):
        def run():
            N.call("apx_debug_umma_gemm", lay, 64, A.data_ptr(), n, Q.data_ptr(), l, C.data_ptr(), n, n, l, n,
                   splits, 0, None, 0, 1, st)
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(20):
            run()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 20
        Bm = C.sum(0)
        ref = (Q.double().T @ A.double())
        bias = float((Bm.double().norm() ** 2 - ref.norm() ** 2) / ref.norm() ** 2)
        print(f"splits {splits} layout {lay & 15:2d}: {ms * 1e3:7.1f} us  {n * n * 4 / ms / 1e6:7.0f} GB/s  "
              f"||Bm||^2 rel bias {bias:+.2e}", flush=True)
