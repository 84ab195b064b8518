"""Small invocations of every product path, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): `compute-sanitizer --tool memcheck python tools/sanitize_cases.py`.
Prints one line per case; the sanitizer's summary is the evidence (profiles/r02_sanitizer_*.txt)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_19308_b200 as P  # noqa: E402
from paper_2504_19308_b200 import genmat as G  # noqa: E402
from paper_2504_19308_b200 import sharded as S  # noqa: E402

rng = np.random.default_rng(0)
dev = torch.device("cuda", 0)


def case(name, fn):
    fn()
    torch.cuda.synchronize()
    print("ok", name, flush=True)


if os.environ.get("SAN_SEG"):
    # large-n segmented gathers only (fp32 n = 13312 > 12800: K11s, and its f16-staged variant K11h
    # forced and under the device-side rule); a separate, slower run: SAN_SEG=1
    n = 13312
    As, _ = G.cycle_operand(n, 8, 1, dev, torch.float32)
    Bs, _ = G.cycle_operand(n, 8, 2, dev, torch.float32)
    for mode in ("0", "2", "1"):
        os.environ["APX_SEG_F16"] = mode
        case(f"segmented cycle product fp32 n={n} k=8 APX_SEG_F16={mode}",
             lambda: P.cycle.cycle_product_device(As, Bs, 8, 8, 1))
    print("all cases ok")
    sys.exit(0)

A, _ = G.cycle_operand(256, 20, 1, dev)
B, _ = G.cycle_operand(256, 20, 2, dev)
for order in (0, 1):
    case(f"cycle n=256 order {order}", lambda: P.cycle_first_order_multiply(A, B, 16, order))
A32, B32 = G.c4_operands(512, 3, dev, 32)
case("mixed fp32 n=512 (tcgen05, gather + flags)", lambda: P.mixed_first_order_multiply(A32, B32, 32, 32, 1, 5))
case("mixed fp32 n=512 order 0", lambda: P.mixed_first_order_multiply(A32, B32, 32, 32, 0, 5))
for n in (64, 96):
    X, Y = rng.standard_normal((n, n)), rng.standard_normal((n, n))
    case(f"circulant n={n}", lambda: P.circulant_first_order_multiply(X, Y, 5, 1))
X, Y = rng.standard_normal((300, 300)), rng.standard_normal((300, 300))
for mode in ("rows", "cols"):
    case(f"sfft n=300 k=257 {mode}", lambda: P.fft_sparse_first_order_multiply(X, Y, 257, 1, mode))
case("svd n=64 q=1", lambda: P.svd_first_order_multiply(X[:64, :64], Y[:64, :64], 1, 1, 3, power_iterations=1))
case("rsvd wide l=141 (Householder + global Jacobi)", lambda: P.randomized_partial_svd(X[:160, :150], 1, 4,
                                                                                       components=141))
case("unitary_dft n=700", lambda: P.unitary_dft(rng.standard_normal((4, 700)), "forward", 1))
case("fourier_row_decompose", lambda: P.fourier_row_decompose(rng.standard_normal((8, 64))))
Ac = torch.from_numpy(rng.standard_normal((64, 64))).to(dev)
Bc = torch.from_numpy(rng.standard_normal((64, 64))).to(dev)
case("circulant rows lockstep x2", lambda: S.circulant_lockstep([S.circulant_rows_steps(Ac, Bc, 5, 1, 2, g)
                                                                 for g in range(2)]))
Ar = A32[:256].contiguous()
case("cycle rows lockstep x2", lambda: S.lockstep([S.cycle_rows_steps(A[g * 128:(g + 1) * 128].contiguous(), g * 128,
                                                                       B, 16, 16, 1) for g in range(2)]))
print("all cases ok")
