"""Middle-dimension rule used to size every benchmark/test configuration.

Restates /root/reference/pkg/src/dbf/budget.py:113-142 (``middle_dim``, ``storage_bits``) and the
greedy layer-wise allocation (``allocate``, budget.py:187-261) that sizes the non-uniform k sweep of
the benchmark (BASELINE configs[4]).  Computing channel scores from calibration data and the
re-factorization are out of scope.
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


def allocate_middle_dims(layers, scores, target_bpw: float, floor_bpw: float = 0.0,
                         granularity: int = 32) -> dict:
    """Per-layer middle dimensions under a global sign-bit budget: a restatement of the reference's
    greedy ``allocate`` (/root/reference/pkg/src/dbf/budget.py:187-261), used to build the
    non-uniform layer-wise k configurations of the benchmark (BASELINE configs[4]).

    ``layers``: sequence of (name, n, m_dim); ``scores``: name -> nonnegative channel scores (their
    length is the layer's source k).  Channels are kept per layer in descending score order, in
    whole granularity blocks competing globally on score mass per sign bit (each channel costs
    n + m_dim bits), above a per-layer floor; a block that does not fit is skipped.  Ties break by
    (layer name, channel index).  Returns name -> k_new."""
    import numpy as np

    if granularity < 1:
        raise ValueError(f"granularity must be >= 1, got {granularity}")
    names = [nm for nm, _, _ in layers]
    if len(set(names)) != len(names) or set(names) != set(scores):
        raise ValueError("layers and scores must match one-to-one by name")
    cost = {nm: n + m for nm, n, m in layers}
    wts = {nm: n * m for nm, n, m in layers}
    budget = target_bpw * sum(wts.values())
    slack = budget * 1e-12
    k_src = {nm: int(np.asarray(scores[nm]).size) for nm in names}

    def floor_k(nm):
        if floor_bpw <= 0:
            return 0
        k = int(np.ceil(floor_bpw * wts[nm] / cost[nm] / granularity)) * granularity
        return min(k, k_src[nm])

    floors = {nm: floor_k(nm) for nm in names}
    used = float(sum(floors[nm] * cost[nm] for nm in names))
    if used > budget + slack:
        raise ValueError(f"floor of {floor_bpw} bits/weight is infeasible under target {target_bpw}: "
                         f"short by {used - budget:.0f} bits")
    blocks = []
    for nm in names:
        sc = np.sort(np.asarray(scores[nm], dtype=np.float64))[::-1]
        for j in range(floors[nm], k_src[nm] - granularity + 1, granularity):
            mass = float(sc[j:j + granularity].sum())
            blocks.append((-mass / (granularity * cost[nm]), nm, j))
    blocks.sort()
    kept = dict(floors)
    for _, nm, j in blocks:
        if kept[nm] != j:
            continue
        c = granularity * cost[nm]
        if used + c <= budget + slack:
            kept[nm] = j + granularity
            used += c
    return kept
