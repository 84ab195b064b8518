"""The C4 product sharded by rows (paper_2504_19308_b200.sharded, apx_mixed_rows_phase) against the
single-device product and the CPU oracle. Several shards are driven on the one GPU in lockstep
(sharded.lockstep sums each exchange in rank order -- what the NCCL all-reduce does across
ranks); the multi-process protocol itself is covered over gloo in test_dist_cpu.py.

Tolerances: fp32 1e-4 relative Frobenius against the fp64 oracle (north star); against the
single-device GPU product 1e-5 (the Gram and Q^T A sums are split differently); one shard
reproduces the single-device product exactly (same kernels, same order); selections bit-exact.
"""
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


def _operands(n, seed):
    A = O.gen_haar_spectrum(n, (np.arange(n) + 1.0) ** -1.5, seed).astype(np.float32)
    B = O.gen_cycle_operand(n, 64, seed + 1).astype(np.float32)
    return A, B


def _sharded(P, Ad, Bd, omega, world, order=1, k=64):
    from paper_2504_19308_b200 import sharded as S
    n = Ad.shape[0]
    blocks = [S.row_range(n, world, r) for r in range(world)]
    gens = [S.mixed_rows_steps(Ad[r0:r1].contiguous(), Bd, k, k, order, omega, serialize=True)
            for r0, r1 in blocks]
    res = [S.check_breakdown(r) for r in S.lockstep(gens)]
    return torch.cat([r["M"] for r in res], 0), res


@pytest.mark.parametrize("order", [1, 0])
def test_one_shard_equals_single_device(P, order):
    n, k = 1024, 64
    A, B = _operands(n, 40)
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    omega = torch.from_numpy(P.draw_sketch(n, k, 3)).cuda().float()
    ref = P.mixed_product_device(Ad, Bd, k, k, order, omega, direct=True)  # the plan the phases cut
    M, res = _sharded(P, Ad, Bd, omega, 1, order)
    torch.cuda.synchronize()
    assert torch.equal(res[0]["sel_b"], ref["sel_b"])
    assert rel(M.cpu().numpy(), ref["M"].cpu().numpy()) < 1e-6
    s, t = res[0]["scalars"].tolist(), ref["scalars"].tolist()
    for i in (P._native.S_FRO2_A, P._native.S_FRO2_B, P._native.S_KEPT_A, P._native.S_KEPT_B,
              P._native.S_FRO2_M):
        assert s[i] == pytest.approx(t[i], rel=1e-6)


@pytest.mark.parametrize("world", [2, 3, 4])
def test_shards_vs_single_device_and_oracle(P, world):
    n, k = 2048, 64
    A, B = _operands(n, 50 + world)
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    omega = torch.from_numpy(P.draw_sketch(n, k, 7)).cuda().float()
    ref = P.mixed_product_device(Ad, Bd, k, k, 1, omega, direct=True)
    M, res = _sharded(P, Ad, Bd, omega, world)
    for r in res:
        assert torch.equal(r["sel_b"], ref["sel_b"])
    Mh = M.cpu().numpy()
    assert rel(Mh, ref["M"].cpu().numpy()) < 1e-5
    Mo, ro = O.mixed_first_order_multiply(A.astype(np.float64), B.astype(np.float64), k, k, 1, 7)
    assert res[0]["sel_b"].tolist() == ro["selected_b"]
    err = rel(Mh, Mo)
    print(f"sharded world={world} n={n}: rel vs oracle {err:.3e}")
    assert err < 1e-4
    # the rank-summed norms agree with the single-device ones
    s = res[0]["scalars"].tolist()
    t = ref["scalars"].tolist()
    assert s[P._native.S_FRO2_M] == pytest.approx(t[P._native.S_FRO2_M], rel=1e-5)
    assert s[P._native.S_FRO2_A] == pytest.approx(t[P._native.S_FRO2_A], rel=1e-6)


def test_sharded_argument_errors(P):
    from paper_2504_19308_b200 import sharded as S
    n = 1000  # not a multiple of 32
    Ad = torch.zeros((n, n), device="cuda")
    omega = torch.zeros((n, 64), device="cuda")
    with pytest.raises(ValueError):
        S.lockstep([S.mixed_rows_steps(Ad[:500].contiguous(), Ad, 64, 64, 1, omega, serialize=True)])
    with pytest.raises(ValueError):
        next(S.mixed_rows_steps(Ad.double(), Ad.double(), 64, 64, 1, omega))
