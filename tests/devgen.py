"""On-device synthetic operands for the large configs (test / bench input synthesis only).

C5: N(0, noise^2) + `ncyc` planted cycles with N(0,1) diagonals + `r` terms
diag(d_i) Circ(c_i), d_i ~ U(0.5, 1.5), c_i the smooth real circulant column of
oracle.gen_circulant_operand. n = 32768 fp32 is 4 GiB per operand, so everything is generated
on the GPU (torch Philox keyed by (seed, operand)); shifts, d_i and c_i are drawn on the host with
numpy streams default_rng([seed, 103, n, operand]).
"""
import numpy as np
import torch

import oracle as O


def c5_operand(n: int, ncyc: int, r: int, seed: int, operand: int, noise: float = 1e-3,
               dtype=torch.float32, device="cuda"):
    """Returns (A device tensor, planted shifts sorted ascending)."""
    rng = np.random.default_rng([seed, 103, n, operand])
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) * 1000003 + operand)
    A = torch.empty((n, n), device=device, dtype=dtype)
    for s in range(0, n, 2048):  # chunked: one 2^30-element normal_ launch faults (torch 2.11)
        A[s:s + 2048].normal_(0.0, noise, generator=g)
    shifts = rng.choice(n, size=ncyc, replace=False)
    i = torch.arange(n, device=device)
    flat = A.view(-1)
    for j in shifts:
        lam = torch.randn(n, generator=g, device=device, dtype=dtype)
        flat.index_add_(0, i * n + (i - int(j)) % n, lam)
    for _ in range(r):
        d = torch.from_numpy(rng.uniform(0.5, 1.5, n)).to(device, dtype)
        c = torch.from_numpy(O.apx_oracle._smooth_circulant_column(rng, n)).to(device, dtype)
        # Circ(c)[i, k] = c[(i - k) % n], built per 2048-row chunk as a row-flipped Hankel view
        # y[q + k] of y[q] = c[(s + cs - 1 - q) % n] (chunks keep torch's kernels in int32 range)
        for s in range(0, n, 2048):
            cs = min(2048, n - s)
            q = torch.arange(cs + n - 1, device=device)
            y = c[(s + cs - 1 - q) % n].contiguous()
            T = y.as_strided((cs, n), (1, 1)).flip(0)
            A[s:s + cs].addcmul_(d[s:s + cs, None], T)
            del T
    return A, sorted(int(j) for j in shifts)


def left_lambdas(A, J):
    """lam[t][i] = A[i, (i - J[t]) % n] (core.py:123-124 left layout), on the device."""
    n = A.shape[0]
    i = torch.arange(n, device=A.device)
    return torch.stack([A[i, (i - int(j)) % n] for j in J])
