"""Batched independent products (batch.py): config C1 (fp64 n = 512, k = 32, p = 8, q = 2,
order 0) for B operand pairs run concurrently on several streams inside one CUDA graph.
Every item must equal the single-product device call bitwise (same kernels, same inputs, its own
workspace), item 0 must match the oracle composition at 1e-10, and a replay must reproduce the
first run bitwise."""
import numpy as np
import pytest
import torch

import oracle as O
from conftest import rel

pytestmark = pytest.mark.gpu


def test_svd_product_batch_c1():
    import paper_2504_19308_b200 as P
    from paper_2504_19308_b200 import svd as PS
    n, nb = 512, 12
    sig = 0.9 ** np.arange(n)
    As = [O.gen_haar_spectrum(n, sig, 2 * t) for t in range(nb)]
    Bs = [O.gen_haar_spectrum(n, sig, 2 * t + 1) for t in range(nb)]
    oas = [np.random.default_rng([t, 0]).standard_normal((n, 40)) for t in range(nb)]
    obs = [np.random.default_rng([t, 1]).standard_normal((n, 40)) for t in range(nb)]
    dev = torch.device("cuda", 0)
    A = torch.from_numpy(np.stack(As)).to(dev)
    B = torch.from_numpy(np.stack(Bs)).to(dev)
    batch = P.SvdProductBatch(A, B, 40, 32, 40, 32, 2, 0, torch.from_numpy(np.stack(oas)),
                              torch.from_numpy(np.stack(obs)), streams=5)
    M = batch.run().clone()
    torch.cuda.synchronize()
    for t in range(nb):
        r = PS.svd_product_device(A[t], B[t], 40, 32, 40, 32, 2, 0, oas[t], obs[t])
        torch.cuda.synchronize()
        assert torch.equal(r["M"], M[t]), t
    Mo, _ = O.svd_first_order_multiply(As[0], Bs[0], None, 0, 0, power_iterations=2, components=32, oversampling=8)
    assert rel(M[0].cpu().numpy(), Mo) < 1e-10
    M2 = batch.run()
    torch.cuda.synchronize()
    assert torch.equal(M2, M)
