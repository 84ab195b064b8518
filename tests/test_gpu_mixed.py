"""GPU parity: mixed rSVD x cycles product (config C4) vs the CPU oracle."""
import numpy as np
import pytest
import torch

import oracle as O
from conftest import rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2504_19308_b200 as P
    return P


@pytest.mark.parametrize("order", [0, 1])
def test_mixed_golden_fp64(P, golden, order):
    g = golden("cycle")
    n, ks, kc, seed = (int(v) for v in g["mx_par"])
    M, rep = P.mixed_first_order_multiply(g["mx_A"], g["mx_B"], ks, kc, order, seed)
    assert rep.selected_b == list(g["mx_Jb"])
    assert rel(M, g[f"mx_M{order}"]) < 1e-10


@pytest.mark.parametrize("n,ks,kc,q", [(96, 8, 5, 0), (256, 16, 12, 1), (500, 24, 7, 2)])
@pytest.mark.parametrize("order", [0, 1])
def test_mixed_fp64_vs_oracle(P, n, ks, kc, q, order):
    A = O.gen_haar_spectrum(n, (np.arange(n) + 1.0) ** -1.5, 3 * n)
    B = O.gen_cycle_operand(n, kc + 3, 3 * n + 1)
    M, rep = P.mixed_first_order_multiply(A, B, ks, kc, order, seed=n, power_iterations=q)
    Mo, ro = O.mixed_first_order_multiply(A, B, ks, kc, order, n, power_iterations=q)
    assert rep.selected_b == ro["selected_b"]
    assert rel(M, Mo) < 1e-10
    assert rep.norm_da == pytest.approx(ro["norm_da"], rel=1e-6)
    assert rep.norm_db == pytest.approx(ro["norm_db"], rel=1e-6)


@pytest.mark.parametrize("split3,direct", [(False, False), (False, True), (True, False)])
def test_mixed_fp32_c4_shape(P, split3, direct):
    """C4 structure (sigma_i=(i+1)^-1.5 Haar A; 64-cycle B) at n=1024, fp32 tensors, tol 1e-4:
    the residual plan (default: f16 gather over dA), the all-fp32 plan (direct) and 3xTF32."""
    n, k = 1024, 64
    A = O.gen_haar_spectrum(n, (np.arange(n) + 1.0) ** -1.5, 8).astype(np.float32)
    B = O.gen_cycle_operand(n, 64, 9).astype(np.float32)
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    M, rep = P.mixed_first_order_multiply(Ad, Bd, k, k, 1, seed=4, split3=split3, direct=direct)
    assert M.dtype == torch.float32
    Mo, ro = O.mixed_first_order_multiply(A.astype(np.float64), B.astype(np.float64), k, k, 1, 4)
    assert rep.selected_b == ro["selected_b"]
    err = rel(M.cpu().numpy(), Mo)
    print(f"fp32 mixed n={n} split3={split3} direct={direct}: rel vs oracle {err:.3e}")
    assert err < 1e-4
    assert rep.posterior_estimate == pytest.approx(ro["posterior_estimate"], rel=0.15)


def _device_norms(P, A, B, kc, seed, direct):
    """(||A||^2, ||M||^2) from the device scalars of one product."""
    from paper_2504_19308_b200 import _native as N
    n = A.shape[0]
    omega = torch.from_numpy(P.cycle.draw_sketch(n, 64, seed)).cuda().float()
    r = P.mixed_product_device(A, B, 64, kc, 1, omega, direct=direct)
    s = r["scalars"].tolist()
    return s[N.S_FRO2_A], s[N.S_FRO2_M], r["M"]


@pytest.mark.parametrize("n,kc,seed", [(512, 64, 1), (1536, 40, 2), (2048, 128, 3), (1024, 1, 4)])
def test_mixed_resid_plan_vs_oracle(P, n, kc, seed):
    """Residual plan shapes: thread groups of 128/256/512 columns, k_cyc from 1 to 128 (the f16
    lambda' table's zero padding), ||A||, ||M|| and the selection vs the fp64 oracle."""
    A = O.gen_haar_spectrum(n, (np.arange(n) + 1.0) ** -1.5, seed).astype(np.float32)
    B = O.gen_cycle_operand(n, kc, seed + 50).astype(np.float32)  # dB = the noise: TF32-small
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    M, rep = P.mixed_first_order_multiply(Ad, Bd, 64, kc, 1, seed=seed)
    Md, repd = P.mixed_first_order_multiply(Ad, Bd, 64, kc, 1, seed=seed, direct=True)
    Mo, ro = O.mixed_first_order_multiply(A.astype(np.float64), B.astype(np.float64), 64, kc, 1, seed)
    assert rep.selected_b == ro["selected_b"] == repd.selected_b
    e_r, e_d = rel(M.cpu().numpy(), Mo), rel(Md.cpu().numpy(), Mo)
    print(f"n={n} kc={kc}: residual plan {e_r:.3e}, direct plan {e_d:.3e}")
    assert e_r < 1e-4 and e_d < 1e-4
    # energy difference (3e-4 of ||A||^2): the plans split the Bm GEMM differently
    assert rep.norm_da == pytest.approx(repd.norm_da, rel=2e-2)
    fa, fm, Mr = _device_norms(P, Ad, Bd, kc, seed, False)
    assert fa == pytest.approx(float(np.sum(A.astype(np.float64) ** 2)), rel=1e-6)
    assert fm == pytest.approx(float(torch.sum(Mr.double() ** 2)), rel=1e-6)
    assert fm == pytest.approx(ro["norm_m"] ** 2, rel=2e-4)


def test_mixed_resid_plan_extreme_scales(P):
    """The f16 scalings come from ||A||_F and ||B||_F: operands scaled by powers of two far outside
    f16's range give the same relative result, with no f16 overflow or flush (the scales are
    bounded by the fp32 range finder's Gram matrix, which must stay finite)."""
    n, k = 512, 32
    A = O.gen_haar_spectrum(n, (np.arange(n) + 1.0) ** -1.5, 5).astype(np.float32)
    B = O.gen_cycle_operand(n, k, 6).astype(np.float32)
    Mo, _ = O.mixed_first_order_multiply(A.astype(np.float64), B.astype(np.float64), 64, k, 1, 9)
    for sa, sb in [(2.0 ** 20, 2.0 ** -20), (2.0 ** -24, 1.0), (1.0, 2.0 ** 24), (2.0 ** -12, 2.0 ** -12)]:
        Ad = torch.from_numpy(A * np.float32(sa)).cuda()
        Bd = torch.from_numpy(B * np.float32(sb)).cuda()
        M, rep = P.mixed_first_order_multiply(Ad, Bd, 64, k, 1, seed=9)
        err = rel(M.double().cpu().numpy() / (sa * sb), Mo)
        assert np.isfinite(M.cpu().numpy()).all()
        assert err < 1e-4, (sa, sb, err)


def test_mixed_rank_deficient_sketch_fp64(P):
    """Rank-1 A with a 6-column sketch: CholeskyQR2 breaks down and the device Householder
    fallback must take over (svd.py tests feed such inputs, test_svd.py:56-64)."""
    rng = np.random.default_rng(3)
    n = 64
    A = np.outer(rng.standard_normal(n), rng.standard_normal(n))
    B = O.gen_cycle_operand(n, 4, 2)
    for order in (0, 1):
        M, rep = P.mixed_first_order_multiply(A, B, 6, 4, order, seed=5)
        Mo, ro = O.mixed_first_order_multiply(A, B, 6, 4, order, 5)
        assert rel(M, Mo) < 1e-9


def test_mixed_pipeline_matches_single_calls(P):
    """MixedPipeline (overlapped H2D / compute / D2H) returns exactly the single-call results."""
    n, k = 512, 32
    A = O.gen_haar_spectrum(n, (np.arange(n) + 1.0) ** -1.5, 21).astype(np.float32)
    Bs = [O.gen_cycle_operand(n, 48, 30 + i).astype(np.float32) for i in range(3)]
    Ah = torch.from_numpy(A).pin_memory()
    pipe = P.MixedPipeline(n, k, k, 1, depth=2)
    outs = [torch.empty((n, n), dtype=torch.float32).pin_memory() for _ in Bs]
    tickets = [pipe.submit(Ah, torch.from_numpy(B).pin_memory(), 5 + i, out=o)
               for i, (B, o) in enumerate(zip(Bs, outs))]
    for i, (B, t) in enumerate(zip(Bs, tickets)):
        M, rep = pipe.result(t)
        M1, rep1 = P.mixed_first_order_multiply(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), k, k, 1, 5 + i)
        assert torch.equal(M, M1.cpu())
        assert rep.selected_b == rep1.selected_b
        assert rep.norm_da == rep1.norm_da and rep.norm_db == rep1.norm_db


def test_mixed_resid_plan_falls_back_on_flat_spectrum(P):
    """A with a flat spectrum (Gaussian): the rank-64 approximation leaves most of A in dA, so the
    f16 residual would carry the product at f16 precision (~4e-4). bm_finalize sees the residual
    energy on the device and the plan runs the fp32 gather over dA instead: parity stays < 1e-4."""
    n, k = 1024, 64
    rng = np.random.default_rng(17)
    A = (rng.standard_normal((n, n)) / np.sqrt(n)).astype(np.float32)
    B = O.gen_cycle_operand(n, k, 18).astype(np.float32)
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    M, rep = P.mixed_first_order_multiply(Ad, Bd, 64, k, 1, seed=3)
    Mo, ro = O.mixed_first_order_multiply(A.astype(np.float64), B.astype(np.float64), 64, k, 1, 3)
    assert rep.selected_b == ro["selected_b"]
    err = rel(M.cpu().numpy(), Mo)
    print(f"flat spectrum, residual plan with fp32 fallback: {err:.3e}")
    assert err < 1e-4


FORCE_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import oracle as O
import paper_2504_19308_b200 as P
n = 1024
A = O.gen_haar_spectrum(n, (np.arange(n) + 1.0) ** -1.5, 8).astype(np.float32)
B = O.gen_cycle_operand(n, 64, 9).astype(np.float32)
M, rep = P.mixed_first_order_multiply(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), 64, 64, 1, seed=4)
Mo, _ = O.mixed_first_order_multiply(A.astype(np.float64), B.astype(np.float64), 64, 64, 1, 4)
print(float(np.linalg.norm(M.cpu().numpy() - Mo) / np.linalg.norm(Mo)))
"""


@pytest.mark.parametrize("mode", ["0", "1"])
def test_mixed_resid_plan_forced_modes(mode):
    """APX_RESID_F16=0 forces the fp32 fallback (dA in fp32 into M, in-place fp32 gather, flags set
    after it), =1 the f16 gather: both within tolerance on the C4-structured input."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", FORCE_SCRIPT % root], capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, APX_RESID_F16=mode))
    assert r.returncode == 0, r.stderr[-2000:]
    err = float(r.stdout.strip().splitlines()[-1])
    print(f"APX_RESID_F16={mode}: {err:.3e}")
    assert err < 1e-4
