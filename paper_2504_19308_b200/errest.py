"""Error estimates (reference errest.py:35-154).

The a-priori / posterior formulas are O(1) host arithmetic on norms the device already reduced;
they stay in Python. ``sketch_norm_estimate`` runs its two thin GEMMs and the reduction on the
device through the C-ABI (apx_sketch_norm).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

_CASES = ("mean-zero", "unsigned", "custom")


@dataclass(frozen=True)
class ErrorModel:
    """errest.py:35-66 -- entry-distribution model for the a-priori denominator."""

    case: str
    n: int
    c: float | None = None

    def __post_init__(self):
        if self.case not in _CASES:
            raise ValueError(f"unknown case {self.case!r}")
        if self.n < 1:
            raise ValueError("n must be >= 1")
        if self.case == "custom":
            if self.c is None or not 0.0 < self.c <= 1.0:
                raise ValueError("custom model needs c in (0, 1]")
        elif self.c is not None:
            raise ValueError(f"case {self.case!r} takes no c")

    def product_constant(self) -> float:
        if self.case == "mean-zero":
            return 1.0 / math.sqrt(self.n)
        if self.case == "unsigned":
            return 0.75
        return float(self.c)


def apriori_relative_error(normA: float, normB: float, norm_dA: float, norm_dB: float,
                           model: ErrorModel) -> float:
    """errest.py:108-124."""
    if normA <= 0 or normB <= 0:
        raise ValueError("normA and normB must be > 0")
    if norm_dA < 0 or norm_dB < 0:
        raise ValueError("residual norms must be >= 0")
    return (norm_dA * norm_dB / math.sqrt(model.n)) / (model.product_constant() * normA * normB)


def posterior_relative_error(norm_dA: float, norm_dB: float, norm_M: float, n: int) -> float:
    """errest.py:127-136."""
    if norm_M <= 0:
        raise ValueError("norm_M must be > 0")
    if norm_dA < 0 or norm_dB < 0:
        raise ValueError("residual norms must be >= 0")
    if n < 1:
        raise ValueError("n must be >= 1")
    return norm_dA * norm_dB / (math.sqrt(n) * norm_M)


def energy_residual(total_sq: float, kept_sq: float, terms: int) -> float:
    """||dA|| from energies, sqrt(max(0, ||A||^2 - kept)) (svd.py:122-130, circulant.py:130-133).

    ||A||^2 and the kept energy are two fixed-order device sums over the same `terms` squares in
    different bases, each exact to about eps * log2(terms) * ||A||^2. A difference inside that
    rounding bound carries no information -- an exactly representable operand (a circulant matrix
    kept whole, reference test_circulant.py:136-142) lands there -- and is reported as 0, the value
    the reference's max(0, .) clamp gives when its own rounding happens to fall below zero."""
    diff = total_sq - kept_sq
    if diff <= 4.0 * 2.220446049250313e-16 * math.log2(max(2, terms)) * abs(total_sq):
        return 0.0
    return math.sqrt(diff)


def finish_report(method: str, order: int, k: int, normA: float, normB: float, norm_da: float,
                  norm_db: float, norm_m: float, n: int, wall: float, model: ErrorModel | None):
    """Assemble the ApproxReport exactly like the tail of every reference multiply
    (svd.py:180-199, circulant.py:200-218, fsparse.py:221-240)."""
    from .report import ApproxReport

    if model is None:
        model = ErrorModel(case="mean-zero", n=n)
    apriori = (apriori_relative_error(normA, normB, norm_da, norm_db, model)
               if normA > 0 and normB > 0 else None)
    posterior = posterior_relative_error(norm_da, norm_db, norm_m, n) if norm_m > 0 else None
    return ApproxReport(method=method, order=order, k=k, norm_da=norm_da, norm_db=norm_db,
                        apriori_estimate=apriori, posterior_estimate=posterior, wall_time=wall)


def sketch_norm_estimate(A, B, k: int, seed) -> float:
    """errest.py:139-154 -- ||A (B G)||_F^2 / k with G ~ N(0,1) of shape (cols(B), k) drawn by
    ``np.random.default_rng(seed)`` exactly as the reference draws it; the two fp64 GEMMs and the
    sum of squares run on the device (apx_sketch_norm). Complex operands go through their real
    embeddings A' = [[Ar, -Ai], [Ai, Ar]], B' = [[Br], [Bi]], for which ||A'(B'G)|| = ||A(BG)||."""
    import numpy as np
    import torch

    from . import _device as D
    from . import _native as N
    from .core import as_matrix

    A = as_matrix(A)
    B = as_matrix(B)
    if A.shape[1] != B.shape[0]:
        raise ValueError(f"dimension mismatch: {A.shape} x {B.shape}")
    if k < 1:
        raise ValueError("k must be >= 1")
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((B.shape[1], k))
    if np.iscomplexobj(A) or np.iscomplexobj(B):
        Ar, Ai = A.real, (A.imag if np.iscomplexobj(A) else np.zeros_like(A.real))
        Br, Bi = B.real, (B.imag if np.iscomplexobj(B) else np.zeros_like(B.real))
        A = np.block([[Ar, -Ai], [Ai, Ar]])
        B = np.concatenate([Br, Bi], axis=0)
    m, n = A.shape
    p = B.shape[1]
    dev = D.require_cuda()
    Ad = torch.from_numpy(np.ascontiguousarray(A, dtype=np.float64)).to(dev)
    Bd = torch.from_numpy(np.ascontiguousarray(B, dtype=np.float64)).to(dev)
    Gd = torch.from_numpy(np.ascontiguousarray(G)).to(dev)
    out = torch.zeros(1, dtype=torch.float64, device=dev)
    ws = D.workspace(N.size("apx_sketch_norm_workspace", m, n, p, k))
    N.call("apx_sketch_norm", Ad.data_ptr(), Bd.data_ptr(), m, n, p, Gd.data_ptr(), k, out.data_ptr(),
           ws.data_ptr(), ws.numel(), D.stream_ptr())
    return float(out.item() / k)
