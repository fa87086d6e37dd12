"""Range partitioning by duty ratios -- drop-in for ``hetoc.passes.partition``.

Reference: pkg/src/hetoc/passes/partition.py:13-31.  The computation runs in
the engine's C ABI (``hb_partition_range``), the same code that splits a batch
across GPUs inside ``hb_hash_fixed`` / ``hb_hash_varlen``, so the Python view
and the engine can never disagree on shard bounds.
"""

from __future__ import annotations

import ctypes
import math

from .. import _native


def round_half_up(x: float) -> int:  # partition.py:13-14
    return math.floor(x + 0.5)


def partition_range(lb: int, ub: int, ratios: list[float]) -> list[tuple[int, int]]:
    """Per-ratio sub-ranges of [lb, ub): disjoint, ordered, union exact (partition.py:17-31)."""
    if lb > ub:
        raise ValueError(f"range [{lb}, {ub}) is inverted")
    if not ratios:
        raise ValueError("need at least one ratio")
    k = len(ratios)
    r = (ctypes.c_double * k)(*[float(x) for x in ratios])
    b = (ctypes.c_int64 * (k + 1))()
    _native.check(_native.lib().hb_partition_range(int(lb), int(ub), r, k, b), "hb_partition_range")
    bounds = list(b)
    return list(zip(bounds, bounds[1:]))
