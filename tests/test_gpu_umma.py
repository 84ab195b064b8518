"""Kernel-level check of the tcgen05 TF32 GEMM (all operand layouts used by the mixed product).
Inputs are rounded to TF32 so the only difference from the fp64 reference is fp32 accumulation."""
import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def tf32(x):
    b = x.astype(np.float32).view(np.uint32) & np.uint32(0xFFFFE000)
    return b.view(np.float32)


def run(layout, bn, M, N, K, splits=1, accumulate=0, mask=None, mod_n=1, trans_out=False):
    from paper_2504_19308_b200 import _native as Nn
    rng = np.random.default_rng(layout * 1000 + bn + M + N + K)
    a = tf32(rng.standard_normal((M, K)))
    b = tf32(rng.standard_normal((K, N)))
    L = layout & 7
    A_st = a.T.copy() if L & 1 else a            # MN-major A is stored [k][m]
    B_st = b.copy() if L & 2 else b.T.copy()     # MN-major B stored [k][n], else [n][k]
    dA = torch.from_numpy(A_st).cuda()
    dB = torch.from_numpy(B_st).cuda()
    ldc = M if L & 4 else N
    rows_c = N if L & 4 else M
    C0 = rng.standard_normal((rows_c, ldc)).astype(np.float32) if accumulate else np.zeros((rows_c, ldc), np.float32)
    dC = torch.from_numpy(np.tile(C0, (splits, 1))).cuda()
    dm = None
    if mask is not None:
        dm = torch.tensor(mask, dtype=torch.int32).cuda()
    if layout & 128:  # persistent GEMM with dynamic tiles: the ticket counter rides in mask_j
        dm = torch.zeros(4, dtype=torch.int32).cuda()
    Nn.call("apx_debug_umma_gemm", layout, bn, dA.data_ptr(), A_st.shape[1], dB.data_ptr(), B_st.shape[1],
            dC.data_ptr(), ldc, M, N, K, splits, accumulate, None if dm is None else dm.data_ptr(),
            0 if mask is None else len(mask), mod_n, None)
    if layout & 128:
        assert int(dm[0]) >= 1  # the producers claimed tiles (and each its terminating ticket)
    torch.cuda.synchronize()
    C = dC.cpu().numpy().reshape(splits, rows_c, ldc)
    a64 = a.astype(np.float64)
    if mask is not None:  # drop (m,k) with (k - m) mod n in mask
        m_idx = np.arange(M)[:, None]
        k_idx = np.arange(K)[None, :]
        a64 = np.where(np.isin((k_idx - m_idx) % mod_n, mask), 0.0, a64)
    ref = a64 @ b.astype(np.float64)
    got = C.sum(axis=0) if splits > 1 else C[0]
    if L & 4:
        got = got.T
    if accumulate:
        ref = ref + (C0.T if L & 4 else C0)
    return float(np.linalg.norm(got - ref) / np.linalg.norm(ref))


@pytest.mark.parametrize("layout", range(8))
def test_umma_layouts_bn64(layout):
    assert run(layout, 64, 256, 64, 96) < 1e-5


@pytest.mark.parametrize("layout", [0, 2])
@pytest.mark.parametrize("bn", [128, 256])
def test_umma_wide(layout, bn):
    assert run(layout, bn, 384, 512, 64) < 1e-5


def test_umma_ragged_and_split():
    assert run(1, 64, 200, 50, 333, splits=3) < 1e-5
    assert run(0, 64, 130, 64, 77, splits=2) < 1e-5


def test_umma_accumulate():
    assert run(2, 128, 256, 256, 64, accumulate=1) < 1e-5


def test_umma_masked_mn_a():
    # A operand = dB^T with cycles {0, 3, 17} of a 256-cycle pattern masked
    assert run(1, 64, 256, 64, 256, mask=[0, 3, 17], mod_n=256) < 1e-5


# ---- TMA + warp-specialized variant (layout bit 32) ----
@pytest.mark.parametrize("layout", range(8))
def test_umma_tma_layouts_bn64(layout):
    assert run(32 | layout, 64, 256, 64, 96) < 1e-5


@pytest.mark.parametrize("layout", [0, 2])
@pytest.mark.parametrize("bn", [128, 256])
def test_umma_tma_wide(layout, bn):
    assert run(32 | layout, bn, 384, 512, 64) < 1e-5


def test_umma_tma_ragged_split_mask():
    assert run(32 | 1, 64, 256, 64, 336, splits=3) < 1e-5
    assert run(32 | 5, 64, 256, 64, 256, splits=2) < 1e-5
    assert run(32 | 1, 64, 256, 64, 256, mask=[0, 3, 17], mod_n=256) < 1e-5
    assert run(32 | 2, 256, 256, 512, 64, accumulate=1) < 1e-5


@pytest.mark.parametrize("layout", [0, 2])
def test_umma_tma_staged_c_accumulate(layout):
    """BN 128 with K <= 64 runs a 2-stage ring and stages the C tile through it (cp.async) for the
    read-modify-write epilogue; ragged M/N exercise the zero-fill and the store guards."""
    assert run(32 | layout, 128, 384, 512, 64, accumulate=1) < 1e-5
    assert run(32 | layout, 128, 200, 260, 40, accumulate=1) < 1e-5
    assert run(32 | layout, 128, 256, 256, 128, accumulate=1) < 1e-5  # 4-stage ring: L2-prefetch path



@pytest.mark.parametrize("bn", [64, 128])
@pytest.mark.parametrize("accumulate", [0, 1])
def test_umma_persistent_tile_loop(bn, accumulate):
    """Persistent double-buffered GEMM (gemm_persist_kernel): few CTAs walking many tiles (TMEM
    buffer reuse, ring phases across tiles), static and dynamic (ticket + shared tile queue) tile
    order, K = 128 and 64, ragged M and K."""
    for dyn in (0, 128):
        for ctas in (1, 3, 0):
            assert run(dyn | 64 | 2, bn, 512, 512, 128, accumulate=accumulate, mod_n=ctas) < 1e-5
        assert run(dyn | 64 | 2, bn, 300, 256, 64, accumulate=accumulate, mod_n=5) < 1e-5
        assert run(dyn | 64 | 2, bn, 256, 384, 40, accumulate=accumulate, mod_n=2) < 1e-5
