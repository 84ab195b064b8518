"""Row-sharded circulant and sfft products driven in lockstep on one GPU
(sharded.circulant_lockstep / lockstep): every shard runs the real device phases; the exchanges
are rank-order sums and, for the circulant product, the term1 redistribution (the all-to-all).

  * circulant: selections identical to the single-device product and the rows of M BITWISE equal
    to it (every per-row / per-column computation is the single-device kernel); oracle parity
    1e-10 (near ties resolved by forcing the GPU's selection);
  * sfft: rows within 1e-12 of the single-device product and 1e-10 of the oracle.
"""
import numpy as np
import pytest
import torch

import oracle as O
from conftest import rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    from paper_2504_19308_b200 import sharded as S
    return S


@pytest.mark.parametrize("n,k,world", [(64, 6, 2), (512, 16, 3), (1024, 16, 4), (4096, 16, 2)])
@pytest.mark.parametrize("order", [0, 1])
def test_circulant_rows_lockstep(S, n, k, world, order):
    from paper_2504_19308_b200 import _native as N
    from paper_2504_19308_b200 import circulant as C
    A = torch.from_numpy(O.gen_circulant_operand(n, 16, 7 * n)).cuda()
    B = torch.from_numpy(O.gen_circulant_operand(n, 16, 7 * n + 1)).cuda()
    ref = C.circulant_product_device(A, B, N.APX_F64, k, order)
    res = S.circulant_lockstep([S.circulant_rows_steps(A, B, k, order, world, g) for g in range(world)])
    torch.cuda.synchronize()
    for r in res:
        assert r["sel_a"].tolist() == ref["sel_a"].tolist()
        assert r["sel_b"].tolist() == ref["sel_b"].tolist()
    M = torch.cat([r["M"] for r in res])
    assert torch.equal(M, ref["M"]), float((M - ref["M"]).abs().max())
    s, sr = res[0]["scalars"].tolist(), ref["scalars"].tolist()
    for slot in (N.S_FRO2_A, N.S_FRO2_B, N.S_KEPT_A, N.S_KEPT_B):
        assert s[slot] == sr[slot]
    assert s[N.S_FRO2_M] == pytest.approx(sr[N.S_FRO2_M], rel=1e-12)
    if n <= 1024:
        Mo, _ = O.circulant_first_order_multiply(A.cpu().numpy(), B.cpu().numpy(), k, order,
                                                 ref["sel_a"].tolist(), ref["sel_b"].tolist())
        assert rel(M.cpu().numpy(), Mo) < 1e-10


def test_circulant_rows_complex_and_k0(S):
    from paper_2504_19308_b200 import _native as N
    from paper_2504_19308_b200 import circulant as C
    rng = np.random.default_rng(3)
    n = 128
    A = torch.from_numpy(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))).cuda()
    B = torch.from_numpy(rng.standard_normal((n, n))).cuda()
    for k in (0, 5):
        ref = C.circulant_product_device(A, B.to(torch.complex128), N.APX_C128, k, 1)
        res = S.circulant_lockstep([S.circulant_rows_steps(A, B, k, 1, 2, g) for g in range(2)])
        assert torch.equal(torch.cat([r["M"] for r in res]), ref["M"])


@pytest.mark.parametrize("mode", ["rows", "cols"])
@pytest.mark.parametrize("world", [2, 3])
def test_sfft_rows_lockstep(S, mode, world):
    from paper_2504_19308_b200 import _native as N
    from paper_2504_19308_b200.fsparse import sfft_product_device
    rng = np.random.default_rng(world)
    n, m, p, k = 256, 300, 200, 12
    A = torch.from_numpy(rng.standard_normal((m, n))).cuda()
    B = torch.from_numpy(rng.standard_normal((n, p))).cuda()
    ref = sfft_product_device(A, B, N.APX_F64, k, 1, mode == "cols")
    cuts = [round(g * m / world) for g in range(world + 1)]
    res = S.lockstep([S.sfft_rows_steps(A[cuts[g]:cuts[g + 1]], B, k, 1, mode) for g in range(world)])
    M = torch.cat([r["M"] for r in res])
    assert rel(M.cpu().numpy(), ref["M"].cpu().numpy()) < 1e-12
    s, sr = res[0]["scalars"].tolist(), ref["scalars"].tolist()
    for slot in (N.S_FRO2_A, N.S_RES2_A, N.S_FRO2_M, N.S_FRO2_B, N.S_RES2_B):
        assert s[slot] == pytest.approx(sr[slot], rel=1e-12)
    sel = torch.cat([r["sel_a"] for r in res])
    assert torch.equal(sel, ref["sel_a"])
