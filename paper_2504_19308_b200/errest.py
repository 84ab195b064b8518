"""Host-side scalar error estimates that end every multiply (reference errest.py:35-136).

These are O(1) host arithmetic on norms the device already reduced; they stay in Python.
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
