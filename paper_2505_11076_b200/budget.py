"""Middle-dimension rule used to size every benchmark/test configuration.

Restates /root/reference/pkg/src/dbf/budget.py:113-142 (``middle_dim``, ``storage_bits``).  The
reference's budgeting pipeline (channel scores, allocation, re-factorization) is out of scope
(SURVEY.md §2 rows 8-9); only the k rule that fixes the layer shapes is needed here.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass


def middle_dim(n: int, m_dim: int, bits: float, granularity: int = 32) -> int:
    """budget.py:113-132: largest multiple of ``granularity`` with at most ``bits`` sign bits
    per weight, never below ``granularity`` itself (warns when clamped)."""
    if bits <= 0:
        raise ValueError(f"bits must be > 0, got {bits}")
    if granularity < 1:
        raise ValueError(f"granularity must be >= 1, got {granularity}")
    raw = bits * n * m_dim / (n + m_dim)
    k = int(raw // granularity) * granularity
    if k < granularity:
        warnings.warn(
            f"budget of {bits} bits/weight for {n}x{m_dim} is below one "
            f"granularity block; clamping k to {granularity}",
            stacklevel=2,
        )
        return granularity
    return k


@dataclass(frozen=True)
class StorageBits:
    total: int
    bits_per_weight: float
    scale_share: float


def storage_bits(n: int, k: int, m_dim: int, scale_width_bits: int = 16) -> StorageBits:
    """budget.py:135-142."""
    if min(n, k, m_dim) < 1:
        raise ValueError("dims must be >= 1")
    scale_bits = (n + k + m_dim) * scale_width_bits
    total = n * k + k * m_dim + scale_bits
    weights = n * m_dim
    return StorageBits(total, total / weights, scale_bits / weights)
