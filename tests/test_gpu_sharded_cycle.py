"""The cycle product sharded by rows (configs C2 / C5; sharded.cycle_rows_steps,
apx_cycle_rows_phase): shards driven in lockstep on one GPU (sums in rank order on the device),
checked against the single-device product through the same C-ABI.

  * C2 (fp64 n = 2048, k = 32, orders 1 and 0; shared-memory strip left product) with 1, 2 and 3
    shards, 64-aligned row blocks: rows of M within 1e-12, selections equal, ||M||_F^2 summed;
  * C5-shaped (fp32 n = 16384, k = 64, order 1; the large-n transposed left product restricted
    to the shard's columns, segmented gathers) with 2 and 4 shards: within 1e-6 of the
    single-device product (fp32 tolerance of the path is 1e-4);
  * one shard's rows against the oracle row restatement (oracle.cycle_product_rows).
"""
import numpy as np
import pytest
import torch

import oracle as O
from conftest import rel
from devgen import c5_operand, left_lambdas

pytestmark = pytest.mark.gpu


def _sharded(A, B, k, order, world, align):
    from paper_2504_19308_b200 import sharded as SH
    n = A.shape[0]
    blocks = [SH.cycle_row_range(n, world, r, align) for r in range(world)]
    gens = [SH.cycle_rows_steps(A[r0:r1], r0, B, k, k, order) for r0, r1 in blocks]
    res = SH.lockstep(gens)
    torch.cuda.synchronize()
    return blocks, res


@pytest.mark.parametrize("order", [1, 0])
@pytest.mark.parametrize("world", [1, 2, 3])
def test_sharded_cycle_c2(order, world):
    import paper_2504_19308_b200 as P
    from paper_2504_19308_b200 import _native as N
    n, k = 2048, 32
    A = torch.from_numpy(O.gen_cycle_operand(n, k, 21)).cuda()
    B = torch.from_numpy(O.gen_cycle_operand(n, k, 22)).cuda()
    full = P.cycle_product_device(A, B, k, k, order)
    blocks, res = _sharded(A, B, k, order, world, 64)
    M = torch.cat([r["M"] for r in res])
    err = rel(M.cpu().numpy(), full["M"].cpu().numpy())
    print(f"C2 order {order}, {world} shards: rel vs single device {err:.2e}")
    assert err < 1e-12
    for r in res:
        assert r["sel_a"].tolist() == full["sel_a"].tolist()
        assert r["sel_b"].tolist() == full["sel_b"].tolist()
    s_full = full["scalars"].cpu().numpy()
    s0 = res[0]["scalars"].cpu().numpy()
    for idx in (N.S_FRO2_A, N.S_FRO2_B, N.S_KEPT_A, N.S_KEPT_B, N.S_FRO2_M):
        assert s0[idx] == pytest.approx(s_full[idx], rel=1e-9)


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_cycle_c5_shape(world):
    import paper_2504_19308_b200 as P
    n, k = 16384, 64
    A, JA = c5_operand(n, k, 8, seed=13, operand=0)
    B, JB = c5_operand(n, k, 8, seed=13, operand=1)
    full = P.cycle_product_device(A, B, k, k, 1)
    blocks, res = _sharded(A, B, k, 1, world, 128)
    M = torch.cat([r["M"] for r in res])
    err = float(torch.linalg.norm((M - full["M"]).double()) / torch.linalg.norm(full["M"].double()))
    print(f"C5-shaped n={n}, {world} shards: rel vs single device {err:.2e}")
    assert err < 1e-6
    for r in res:
        assert r["sel_a"].tolist() == JA and r["sel_b"].tolist() == JB
    # the last shard's edge rows against the oracle row restatement
    r0, r1 = blocks[-1]
    rows = np.array([r0, r0 + 1, r1 - 2, r1 - 1])
    Rt = torch.from_numpy(rows).cuda()
    Mo = O.cycle_product_rows(rows, A[Rt].double().cpu().numpy(), JA,
                              [B[(Rt - j) % n].double().cpu().numpy() for j in JA], JB,
                              left_lambdas(B, JB).double().cpu().numpy())
    err_o = rel(res[-1]["M"][torch.from_numpy(rows - r0).cuda()].double().cpu().numpy(), Mo)
    print(f"  rows vs oracle {err_o:.2e}")
    assert err_o < 1e-4
