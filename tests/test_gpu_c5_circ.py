"""Config C5's secondary method at full size: the circulant product (k = 32, order 1) of the
n = 32768 operands of tests/devgen.py (128 cycles + 32 circulant terms + noise), in fp64 on the
device (the four-step transform path: n1 = 128, n2 = 256). The CPU oracle cannot hold these
operands, so the checks are size-independent:

  * the kept components are the R_t of circulant_component (an independent O(n^2) cycle
    average, circulant.py:94-108) -- their norms dominate those of a sample of the others;
  * the first-order identity (AB - M) x = dA (dB x) on a random complex probe, with
    Ahat v = sum_t r_t (*) (w^{t c} v) built from those components (torch.fft circular
    convolutions) and fp64 matvecs: relative error <= 1e-10.
"""
import numpy as np
import pytest
import torch

from devgen import c5_operand

pytestmark = pytest.mark.gpu

N, K, NCYC, NCIRC = 32768, 32, 128, 32


@pytest.fixture(scope="module")
def run():
    from paper_2504_19308_b200 import _native as Nt
    from paper_2504_19308_b200 import circulant as C
    A32, _ = c5_operand(N, NCYC, NCIRC, seed=5, operand=0)
    A = A32.double()
    del A32
    B32, _ = c5_operand(N, NCYC, NCIRC, seed=5, operand=1)
    B = B32.double()
    del B32
    torch.cuda.empty_cache()
    r = C.circulant_product_device(A, B, Nt.APX_F64, K, 1)
    torch.cuda.synchronize()
    del r["ws"]
    torch.cuda.empty_cache()
    yield C, A, B, r
    del A, B, r
    torch.cuda.empty_cache()


def _components(C, X, sel):
    return torch.stack([torch.from_numpy(C.circulant_component(X, int(t))).cuda() for t in sel])


def test_c5_circulant_selection(run):
    C, A, B, r = run
    for X, sel in ((A, r["sel_a"].tolist()), (B, r["sel_b"].tolist())):
        assert sel == sorted(sel) and len(set(sel)) == K
        kept = torch.linalg.norm(_components(C, X, sel), dim=1)
        rng = np.random.default_rng(1)
        others = [int(t) for t in rng.choice(N, 96, replace=False) if int(t) not in set(sel)]
        rest = torch.linalg.norm(_components(C, X, others), dim=1)
        assert float(kept.min()) >= float(rest.max())


def test_c5_circulant_first_order_identity(run):
    C, A, B, r = run
    sa, sb = r["sel_a"].tolist(), r["sel_b"].tolist()
    Ra, Rb = _components(C, A, sa), _components(C, B, sb)
    c = torch.arange(N, device="cuda", dtype=torch.float64)
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    x = torch.complex(torch.randn(N, generator=g, device="cuda", dtype=torch.float64),
                      torch.randn(N, generator=g, device="cuda", dtype=torch.float64))

    def mv(X, v):  # fp64 (complex) matvec, row-chunked
        return torch.cat([X[s:s + 2048].to(torch.complex128) @ v for s in range(0, N, 2048)])

    def hat(R, sel, v):  # sum_t r_t (*) (w^{t c} v), w = exp(2 pi i / n)
        out = torch.zeros_like(v)
        for rt, t in zip(R, sel):
            u = torch.exp(2j * np.pi * ((t * c) % N) / N) * v
            out += torch.fft.ifft(torch.fft.fft(rt) * torch.fft.fft(u))
        return out

    Bx = mv(B, x)
    lhs = mv(A, Bx) - mv(r["M"], x)
    dBx = Bx - hat(Rb, sb, x)
    rhs = mv(A, dBx) - hat(Ra, sa, dBx)
    err = float(torch.linalg.norm(lhs - rhs) / torch.linalg.norm(mv(A, Bx)))
    print(f"C5 circulant n={N} k={K}: first-order identity {err:.3e}")
    assert err < 1e-10
