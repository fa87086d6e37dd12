"""Multi-process (one rank per GPU) sharding of a hash batch.

The batch shards by message range -- ``partition_range(0, n, [1/world]*world)``
(pkg/src/hetoc/passes/partition.py:17-31, as lower_loop applies it,
pkg/src/hetoc/passes/lower_hyper_for.py:207-254) -- and each rank hashes its
slice with no data-path collective.  The only collective is the optional
digest gather (north_star: "NCCL is needed only for an optional device-side
gather"), an all-gather over ``torch.distributed`` (NCCL over NVLink on GPUs,
gloo in the CPU tests).
"""

from __future__ import annotations

from .passes.partition import partition_range


def shard_bounds(n: int, world: int) -> list[tuple[int, int]]:
    """Equal-ratio message-range shards of [0, n) for `world` ranks."""
    if world < 1:
        raise ValueError("world must be >= 1")
    return partition_range(0, n, [1.0 / world] * world)


def shard_for_rank(n: int, world: int, rank: int) -> tuple[int, int]:
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    return shard_bounds(n, world)[rank]


def gather_digests(local, n_total: int, group=None):
    """All-gather per-rank (n_i, dlen) uint8 digest slices into the full
    (n_total, dlen) array on every rank (dst_off = s_i*dlen, the copy-out rule
    of _emit_dev_launch, lower_hyper_for.py:316)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    bounds = shard_bounds(n_total, world)
    rows = max(hi - lo for lo, hi in bounds) if bounds else 0
    dlen = local.shape[1]
    rank = dist.get_rank(group)
    lo, hi = bounds[rank]
    if local.shape[0] != hi - lo:
        raise ValueError(f"rank {rank} holds {local.shape[0]} digests, shard is [{lo}, {hi})")
    padded = torch.zeros((rows, dlen), dtype=torch.uint8, device=local.device)
    padded[: hi - lo] = local
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded, group=group)
    return torch.cat([p[: b - a] for p, (a, b) in zip(parts, bounds)], dim=0)
