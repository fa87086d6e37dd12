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


class P2PDigestGather:
    """Fused hash + gather with the peer mapping set up once.

    Every rank hashes its shard -- global rows ``[lo, hi)`` of
    ``shard_bounds(n_total, world)``, the (hi-lo, L) CUDA tensor ``msgs_local``
    -- and the hash kernel stores its digests straight into the root's
    (n_total, dlen) buffer through a CUDA IPC mapping (P2P stores over NVLink 5
    / NVSwitch when the ranks sit on different GPUs).  Only the 64-byte memory
    handle (at construction) and barriers go through ``torch.distributed``.
    ``launch()`` enqueues one hash pass on the current stream; ``out`` is the
    full digest tensor on the root (None elsewhere), complete after
    ``torch.cuda.synchronize()`` + a barrier.
    """

    def __init__(self, alg: str, msgs_local, n_total: int, root: int = 0, group=None):
        import ctypes

        import torch
        import torch.distributed as dist

        from . import _native
        from .crypto.batch import DIGEST_LEN, _check_alg

        _check_alg(alg)
        self.alg, self.group, self.root = alg, group, root
        world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        self.lo, self.hi = shard_bounds(n_total, world)[self.rank]
        if (msgs_local.dim() != 2 or msgs_local.shape[0] != self.hi - self.lo or not msgs_local.is_cuda
                or msgs_local.dtype != torch.uint8):
            raise ValueError(f"rank {self.rank} must pass its shard [{self.lo}, {self.hi}) as a 2-D uint8 CUDA tensor")
        self.msgs = msgs_local.contiguous()
        self.dlen = DIGEST_LEN[alg]
        self.gpu = self.msgs.device.index
        self.lib = _native.lib()
        self.out, self.mapped = None, None
        handle = [None]
        if self.rank == root:
            self.out = torch.empty((n_total, self.dlen), dtype=torch.uint8, device=self.msgs.device)
            h = (ctypes.c_uint8 * 64)()
            off = ctypes.c_uint64(0)
            _native.check(self.lib.hb_ipc_handle(self.out.data_ptr(), h, ctypes.byref(off)), "hb_ipc_handle")
            handle[0] = (bytes(h), off.value)
        torch.cuda.synchronize(self.gpu)  # the root's buffer exists before anyone maps it
        dist.broadcast_object_list(handle, src=root, group=group)
        if self.rank == root:
            self.base = self.out.data_ptr()
        else:
            ptr = ctypes.c_void_p()
            h = (ctypes.c_uint8 * 64).from_buffer_copy(handle[0][0])
            _native.check(self.lib.hb_ipc_open(self.gpu, h, ctypes.byref(ptr)), "hb_ipc_open")
            self.mapped = ptr.value
            self.base = self.mapped + handle[0][1]

    def launch(self, stream=None):
        import torch

        from . import _native

        if self.hi <= self.lo:
            return
        s = stream if stream is not None else torch.cuda.current_stream(self.gpu).cuda_stream
        rc = self.lib.hb_hash_fixed_dev(_native.ALG_ID[self.alg], self.gpu, self.msgs.data_ptr(), self.hi - self.lo,
                                        self.msgs.shape[1], self.base + self.lo * self.dlen, s, 0)
        _native.check(rc, "hb_hash_fixed_dev")

    def close(self):
        import ctypes

        if self.mapped is not None:
            self.lib.hb_ipc_close(self.gpu, ctypes.c_void_p(self.mapped))
            self.mapped = None


def hash_fixed_gather_p2p(alg: str, msgs_local, n_total: int, root: int = 0, group=None):
    """One fused hash + gather pass (see :class:`P2PDigestGather`); returns the
    full digest tensor on the root, None elsewhere."""
    import torch
    import torch.distributed as dist

    g = P2PDigestGather(alg, msgs_local, n_total, root, group)
    try:
        g.launch()
        torch.cuda.synchronize(g.gpu)  # this rank's digest stores have landed in the root's buffer
        dist.barrier(group=group)
    finally:
        g.close()
    return g.out
