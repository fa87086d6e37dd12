"""world_size-2 gloo test of the N>1 host path: message-range shards
(partition_range) hashed independently per rank, then the optional digest
gather, reproduce the single-rank result.  CPU only: the per-rank "kernel"
here is the oracle (a test stand-in; on GPUs each rank calls the engine)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2407_09333_b200.distributed import gather_digests, shard_bounds, shard_for_rank


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, L, q):
    import torch.distributed as dist

    import oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard_for_rank(n, world, rank)
        # the bytes of global messages [lo, hi): counter-based, shard-independent
        mine = oracle.fill_random((hi - lo) * L, 17, lo * L).reshape(hi - lo, L)
        res = {}
        for alg in ("sha1", "md5", "sm3"):
            local = torch.from_numpy(oracle.batch_fixed(alg, mine))
            full = gather_digests(local, n)
            res[alg] = full.numpy().copy()
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [1001, 7, 1])
def test_two_rank_shard_and_gather(n):
    import oracle

    L = 40  # multiple of 8 so every shard starts on a generator word
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, L, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    data = oracle.fill_random(n * L, 17).reshape(n, L)
    for alg in ("sha1", "md5", "sm3"):
        ref = oracle.batch_fixed(alg, data)
        for r in range(world):
            assert np.array_equal(got[r][alg], ref), (alg, r)


def test_shard_bounds_rules():
    assert shard_bounds(10, 2) == [(0, 5), (5, 10)]
    assert shard_bounds(1 << 24, 8)[-1] == ((1 << 24) * 7 // 8, 1 << 24)
    assert shard_bounds(3, 8)[0] == (0, 0)  # empty shards are legal
    with pytest.raises(ValueError):
        shard_for_rank(10, 2, 2)


def _p2p_worker(rank, world, port, n, L, q):
    import torch.distributed as dist

    import oracle
    from paper_2407_09333_b200.distributed import hash_fixed_gather_p2p, shard_for_rank

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ngpu = torch.cuda.device_count()
        dev = torch.device("cuda", rank % ngpu)
        lo, hi = shard_for_rank(n, world, rank)
        res = {}
        for alg in ("sha1", "md5", "sm3"):
            mine = torch.from_numpy(oracle.fill_random((hi - lo) * L, 23, lo * L).reshape(hi - lo, L)).to(dev)
            full = hash_fixed_gather_p2p(alg, mine, n)
            if rank == 0:
                res[alg] = full.cpu().numpy()
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_fused_p2p_gather(world):
    """The fused gather: every rank's hash kernel stores its digests straight
    into rank 0's buffer through a CUDA IPC mapping (P2P over NVLink between
    GPUs; here the ranks may share one GPU -- the mapping is the same).  Only the
    64-byte handle and a barrier go through torch.distributed (gloo)."""
    import oracle

    n, L = 100003, 64
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_p2p_worker, args=(r, world, port, n, L, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    data = oracle.fill_random(n * L, 23).reshape(n, L)
    for alg in ("sha1", "md5", "sm3"):
        assert np.array_equal(got[0][alg], oracle.batch_fixed(alg, data, threads=8)), alg


@pytest.mark.gpu
def test_bench_multirank_path():
    """bench.py under torchrun with 2 ranks (gloo test hook: ranks share the
    visible GPU): sharding, max-over-ranks timing and the fused P2P gather run
    and print one JSON line whose end-to-end digests match the device run."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, HB_BENCH_BACKEND="gloo")
    for extra in (["--workload", "sha1_64"], ["--workload", "md5_1k", "--msgs", "65536", "--gather", "p2p"]):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(root, "bench.py"),
               "--gpus", "2", "--steps", "3", "--warmup", "3", "--e2e-steps", "2"] + extra
        r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
        assert line["n_gpus"] == 2 and line["value"] > 0 and line["e2e"]["matches_device_run"], line
