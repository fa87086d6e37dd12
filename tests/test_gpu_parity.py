"""Parity of the B200 engine with the CPU oracle and the reference golden
vectors.  Every call goes through the C ABI (libhetoc_b200.so).  Bit-exact is
the bar: digests are integer/byte results."""

import ctypes
import hashlib

import numpy as np
import pytest

import oracle
from paper_2407_09333_b200 import _native
from paper_2407_09333_b200.crypto import (
    MessageBatch,
    UnknownAlgorithmError,
    batch_digest,
    batch_digest_varlen,
    digest,
    digest_sha1_accel,
    gen_messages,
    hash_batch,
    hash_decimal,
    md5,
    sha1,
    sm3,
)

pytestmark = pytest.mark.gpu
ALGS = ("sha1", "md5", "sm3")
FLAGS = {"tma": 0, "direct": _native.HB_FLAG_NO_TMA}
ZC_DEFAULT = 256 << 10  # $HB_ZERO_COPY_MAX default (hb_internal.h)


@pytest.fixture(autouse=True)
def _ring_unless_zero_copy(request, monkeypatch):
    """These tests cover kernel shapes (TMA tiles, the length sort, exact-size
    device buffers) that small host calls no longer reach: small untimed calls
    take the zero-copy path (kernels reading mapped host memory, direct loads,
    unsorted).  So every test here runs with $HB_ZERO_COPY_MAX=0 unless it is
    marked zero_copy; the zero-copy path has its own tests below."""
    if request.node.get_closest_marker("zero_copy") is None:
        monkeypatch.setenv("HB_ZERO_COPY_MAX", "0")
        _native.reload_tuning()
    yield
    monkeypatch.undo()
    _native.reload_tuning()


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_device_visible_and_native_loaded():
    assert _native.device_count() >= 1
    info = _native.device_info(0)
    assert info["cc_major"] == 10, info  # sm_100


@pytest.mark.zero_copy
def test_kats(golden):
    for row in golden("kats.json"):
        assert digest(row["alg"], bytes.fromhex(row["msg_hex"])).hex() == row["digest"]
    assert sha1(b"abc").hex() == "a9993e364706816aba3e25717850c26c9cd0d89d"
    assert md5(b"").hex() == "d41d8cd98f00b204e9800998ecf8427e"
    assert sm3(b"abc").hex() == "66c7f0f462eeedd9d1f2d46bdc10e4e24167c4875cf2f7a2297da02b8f4ba8e0"
    assert digest_sha1_accel(b"").hex() == "da39a3ee5e6b4b0d3255bfef95601890afd80709"


@pytest.mark.zero_copy
def test_digest_small_every_length():
    """crypto.digest's one-launch path (hb_digest_small): every length 0..300,
    the 55/56/64-byte padding edges of later blocks, both parameter sizes
    (<=256 and <=4096 B) and the limit, against the oracle; one byte past the
    limit takes the varlen path and must agree too."""
    lens = list(range(301)) + [439, 440, 447, 448, 511, 512, 1000, 2047, 2048, 4031, 4032, 4095, 4096, 4097, 6000]
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    data = oracle.fill_random(int(off[-1]), 61)
    lib = _native.lib()
    k0 = _native.launch_count()
    for alg in ALGS:
        ref = oracle.batch_varlen(alg, data, off, 8)
        for i, L in enumerate(lens):
            m = data[int(off[i]):int(off[i + 1])].tobytes()
            assert digest(alg, m).data == ref[i].tobytes(), (alg, L)
        out = ctypes.create_string_buffer(32)
        assert lib.hb_digest_small(_native.ALG_ID[alg], data.ctypes.data, 4096, out, 0) == _native.HB_OK
        assert out.raw[:ref.shape[1]] == oracle.batch_varlen(alg, data[:4096], np.array([0, 4096], np.uint64))[0].tobytes()
        assert "k_digest_small" in _native.last_kernel_name()
    assert _native.launch_count() > k0
    assert lib.hb_digest_small(1, b"a", 1, ctypes.create_string_buffer(16), _native.device_count()) == _native.HB_ERR_NODEV


@pytest.mark.zero_copy
@pytest.mark.parametrize("zc_max", ["65536", "262144"])
def test_small_batch_zero_copy(hb_env, zc_max):
    """Small untimed single-GPU calls read mapped host memory directly
    (small_batch in hb_engine.cu).  Against the oracle and against the chunk
    ring (HB_ZERO_COPY_MAX=0) at the size limits: input bytes, 128 KiB of
    digests, 64 KiB of offsets; varlen with offsets[0] != 0; every kernel
    family (TMA widths fall back to the direct loads)."""
    cases = [(1, 64), (5, 0), (4096, 16), (4096, 32), (1024, 64), (64, 1024), (63, 1000), (16, 4096), (1, 65536), (4000, 7)]
    for alg in ALGS:
        for n, L in cases:
            data = oracle.fill_random(n * L, n + L).reshape(n, L)
            ref = oracle.batch_fixed(alg, data, threads=8)
            hb_env.set(HB_ZERO_COPY_MAX=zc_max)
            assert np.array_equal(batch_digest(alg, data), ref), (alg, n, L)
            hb_env.set(HB_ZERO_COPY_MAX=0)
            assert np.array_equal(batch_digest(alg, data), ref), (alg, n, L)
        rng = np.random.default_rng(5)
        for n in (1, 7, 1000, 8190, 8191):
            lens = rng.integers(0, 40, n)
            off = (np.concatenate([[0], np.cumsum(lens)]) + 13).astype(np.uint64)
            data = oracle.fill_random(int(off[-1]) + 5, n)
            ref = oracle.batch_varlen(alg, data, off, 8)
            hb_env.set(HB_ZERO_COPY_MAX=zc_max)
            assert np.array_equal(batch_digest_varlen(alg, data, off), ref), (alg, n)
            hb_env.set(HB_ZERO_COPY_MAX=0)
            assert np.array_equal(batch_digest_varlen(alg, data, off), ref), (alg, n)


@pytest.mark.zero_copy
def test_small_call_error_leaves_engine_usable():
    """A small call rejected at launch (an A/B-only flag on the shipped
    library) raises, and the next calls on the same slots still succeed: the
    slot goes back to the pool and the non-sticky error is cleared."""
    if _native.built_with_ab():
        pytest.skip("the A/B library accepts the A/B varlen flags")
    data = oracle.fill_random(300, 4)
    off = np.array([0, 100, 300], np.uint64)
    for _ in range(3):
        with pytest.raises(RuntimeError, match="A/B"):
            batch_digest_varlen("md5", data, off, flags=_native.HB_FLAG_VARLEN_WORDS)
        assert np.array_equal(batch_digest_varlen("md5", data, off), oracle.batch_varlen("md5", data, off))
        assert digest("sm3", b"abc").hex().startswith("66c7f0f4")


@pytest.mark.zero_copy
def test_small_batch_concurrent_callers():
    """Pool threads issuing small batches at once (hash_batch / _fast_digest
    slices) each lease their own zero-copy slot: no crossed digests."""
    from concurrent.futures import ThreadPoolExecutor

    jobs = [(ALGS[i % 3], 1 + (i * 37) % 900, (16, 64, 100, 1024)[i % 4]) for i in range(240)]
    datas = [oracle.fill_random(n * L, i).reshape(n, L) for i, (_, n, L) in enumerate(jobs)]
    with ThreadPoolExecutor(16) as ex:
        got = list(ex.map(lambda k: batch_digest(jobs[k][0], datas[k]), range(len(jobs))))
    for (alg, n, L), d, g in zip(jobs, datas, got):
        assert np.array_equal(g, oracle.batch_fixed(alg, d)), (alg, n, L)


@pytest.mark.zero_copy
def test_digest_small_concurrent_callers():
    """Pool threads calling digest at once (the executor's per-index
    crypto.digest) each get their own stream/slot: no crossed results."""
    from concurrent.futures import ThreadPoolExecutor

    msgs = [bytes([i % 251]) * (i % 700) for i in range(2000)]
    with ThreadPoolExecutor(16) as ex:
        got = list(ex.map(lambda m: digest("sm3", m).data, msgs))
    off = np.concatenate([[0], np.cumsum([len(m) for m in msgs])]).astype(np.uint64)
    ref = oracle.batch_varlen("sm3", np.frombuffer(b"".join(msgs), np.uint8), off, 8)
    assert got == [r.tobytes() for r in ref]


def test_boundary_lengths_single(golden):
    for row in golden("boundary.json"):
        m = np.frombuffer(bytes.fromhex(row["msg_hex"]), np.uint8).reshape(1, -1)
        for alg in ALGS:
            for fl in FLAGS.values():
                assert batch_digest(alg, m, flags=fl)[0].tobytes().hex() == row[alg], (alg, row["len"], fl)


def test_fixed_golden_batches(golden):
    for row in golden("fixed_batches.json"):
        n, L = row["n"], row["msg_len"]
        data = oracle.fill_random(n * L, row["seed"]).reshape(n, L)
        for alg in ALGS:
            for fl in FLAGS.values():
                out = batch_digest(alg, data, flags=fl)
                assert sha(out) == row[alg], (alg, n, L, fl)


@pytest.mark.zero_copy
@pytest.mark.parametrize("path", ["ring", "zero_copy"])
@pytest.mark.parametrize("alg", ALGS)
def test_every_width_0_to_300(alg, path, hb_env):
    # every tail shape r = L % 64 (incl. 55/56/63/64/65 boundaries), partial warps/CTAs (n=133);
    # the ring reaches the TMA tiles from L = 144, the zero-copy path the direct loads at every width
    hb_env.set(HB_ZERO_COPY_MAX=0 if path == "ring" else ZC_DEFAULT)
    for L in range(0, 301):
        n = 133
        data = oracle.fill_random(n * L, 77 + L).reshape(n, L)
        ref = oracle.batch_fixed(alg, data, threads=4)
        for name, fl in FLAGS.items():
            got = batch_digest(alg, data, flags=fl)
            assert np.array_equal(got, ref), (alg, L, name)


@pytest.mark.parametrize("alg", ALGS)
def test_large_widths(alg):
    for L in (1024, 1040, 4096, 4100, 65536, 65537):
        n = 70
        data = oracle.fill_random(n * L, L).reshape(n, L)
        ref = oracle.batch_fixed(alg, data, threads=8)
        for fl in FLAGS.values():
            assert np.array_equal(batch_digest(alg, data, flags=fl), ref), (alg, L)


def test_non_uint8_and_noncontiguous_input():
    base = oracle.fill_random(64 * 200, 5).reshape(64, 200)
    view = base[:, 3:67]  # non-contiguous rows
    for alg in ALGS:
        assert np.array_equal(batch_digest(alg, view), oracle.batch_fixed(alg, np.ascontiguousarray(view)))
    wide = base[:, :16].astype(np.int64) + 512  # cast mod 256 like batch.py:133
    assert np.array_equal(batch_digest("md5", wide), oracle.batch_fixed("md5", base[:, :16]))


def test_varlen_golden(golden):
    for row in golden("varlen_batches.json"):
        lens = np.array(row["lens"], np.uint64)
        off = np.zeros(len(lens) + 1, np.uint64)
        off[1:] = np.cumsum(lens)
        data = oracle.fill_random(int(off[-1]), row["seed"])
        for alg in ALGS:
            assert sha(batch_digest_varlen(alg, data, off)) == row[alg]


def _varlen_random_case():
    rng = np.random.default_rng(12)
    n = 20000  # above the sort threshold
    lens = rng.integers(0, 4097, n).astype(np.uint64)
    lens[::97] = 0
    off = np.zeros(n + 1, np.uint64)
    off[1:] = np.cumsum(lens) + 5  # non-zero base offset
    off[0] = 5
    data = oracle.fill_random(int(off[-1]) + 3, 99)
    return data, off


@pytest.mark.parametrize("sort", ["default", "window", "global"])
@pytest.mark.parametrize("alg", ALGS)
def test_varlen_random_sorted_and_unsorted(alg, sort, hb_env):
    """The shipped varlen path: windowed (MD5 default) or global length sort,
    or none (HB_FLAG_NO_SORT), per-thread 128-bit-load kernel."""
    if sort != "default":
        hb_env.set(HB_VARLEN_SORT=sort)
    data, off = _varlen_random_case()
    ref = oracle.batch_varlen(alg, data, off, threads=8)
    for fl in (0, _native.HB_FLAG_NO_SORT, _native.HB_FLAG_VARLEN_COOP_OFF,
               _native.HB_FLAG_VARLEN_COOP_OFF | _native.HB_FLAG_NO_SORT):
        assert np.array_equal(batch_digest_varlen(alg, data, off, flags=fl), ref), fl
        assert "k_varlen16" in _native.last_kernel_name()


def test_varlen_ab_flags_rejected_in_default_build():
    if _native.built_with_ab():
        pytest.skip("A/B library loaded")
    data, off = _varlen_random_case()
    for fl in (_native.HB_FLAG_VARLEN_WORDS, _native.HB_FLAG_VARLEN_COOP):
        with pytest.raises(RuntimeError, match="HB_AB"):
            batch_digest_varlen("md5", data, off, flags=fl)


@pytest.mark.ab
@pytest.mark.parametrize("sort", ["window4096", "window16384", "global", "prefetch", "bulk", "ld32", "ld16"])
@pytest.mark.parametrize("alg", ALGS)
def test_varlen_ab_arms(alg, sort, hb_env):
    env = {"HB_VARLEN_SORT": "global" if sort == "global" else "window"}
    if sort.startswith("window"):
        env["HB_SORT_WINDOW"] = sort[6:]
    if sort == "prefetch":
        env["HB_VARLEN_PREFETCH"] = "1"
    if sort == "bulk":
        env["HB_VARLEN_BULK"] = "2"
    if sort.startswith("ld"):
        env["HB_VARLEN_LD"] = sort[2:]
    hb_env.set(**env)
    data, off = _varlen_random_case()
    ref = oracle.batch_varlen(alg, data, off, threads=8)
    for fl in (0, _native.HB_FLAG_NO_SORT, _native.HB_FLAG_VARLEN_WORDS,
               _native.HB_FLAG_VARLEN_WORDS | _native.HB_FLAG_NO_SORT, _native.HB_FLAG_VARLEN_COOP_OFF,
               _native.HB_FLAG_VARLEN_COOP_OFF | _native.HB_FLAG_NO_SORT, _native.HB_FLAG_VARLEN_COOP,
               _native.HB_FLAG_VARLEN_COOP | _native.HB_FLAG_NO_SORT):
        assert np.array_equal(batch_digest_varlen(alg, data, off, flags=fl), ref), fl


def test_engine_chunking_and_pinned(hb_env):
    # many sub-batches (the _run_group contract, executor.py:603-699) and pinned vs pageable host buffers
    n, L = 5000, 200
    data = oracle.fill_random(n * L, 31).reshape(n, L)
    ref = {a: oracle.batch_fixed(a, data, threads=8) for a in ALGS}
    hb_env.set(HB_CHUNK_BYTES=64 * 1024)
    lib = _native.lib()
    p = lib.hb_alloc_pinned(n * L)
    assert p
    try:
        pinned = np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_uint8)), shape=(n * L,)).reshape(n, L)
        pinned[:] = data
        for alg in ALGS:
            t = {}
            assert np.array_equal(batch_digest(alg, data, timing=t), ref[alg])
            assert t["chunks"] > 10 and t["h2d_bytes"] == n * L
            assert np.array_equal(batch_digest(alg, pinned), ref[alg])
            assert np.array_equal(batch_digest(alg, data, flags=_native.HB_FLAG_SYNC_H2D), ref[alg])
    finally:
        lib.hb_free_pinned(p)
    # varlen chunking including one message bigger than the chunk budget
    lens = np.array([10, 200000, 3, 0, 70000] + [100] * 3000, np.uint64)
    off = np.zeros(len(lens) + 1, np.uint64)
    off[1:] = np.cumsum(lens)
    vdata = oracle.fill_random(int(off[-1]), 8)
    for alg in ALGS:
        assert np.array_equal(batch_digest_varlen(alg, vdata, off), oracle.batch_varlen(alg, vdata, off, 8))


def test_engine_pipelined_chunks(hb_env):
    """Chunk pipelining of host-buffer calls: a shard whose digests reach
    HB_PIPE_MIN_OUT is cut into >= HB_PIPE_CHUNKS chunks of >= HB_MIN_CHUNK_BYTES
    (H2D of chunk k+1 overlaps kernel + D2H of chunk k); a 4 MiB batch of
    64-byte messages stays one chunk by default.  The digests are the oracle's
    either way (fixed, varlen, decimal)."""
    n, L = 65536, 64
    data = oracle.fill_random(n * L, 37).reshape(n, L)
    lens = np.random.default_rng(3).integers(0, 129, 40000).astype(np.uint64)
    off = np.zeros(len(lens) + 1, np.uint64)
    off[1:] = np.cumsum(lens)
    vdata = oracle.fill_random(int(off[-1]), 9)
    for alg in ALGS:
        ref = oracle.batch_fixed(alg, data, threads=8)
        vref = oracle.batch_varlen(alg, vdata, off, 8)
        dref = oracle.batch_fixed(alg, oracle.gen_decimal(10**6, 300000, 9), threads=8)
        for env, chunks in (({}, (1, 1)), ({"HB_PIPE_MIN_OUT": "1", "HB_MIN_CHUNK_BYTES": str(1 << 20)}, (4, 4)),
                            ({"HB_PIPE_MIN_OUT": "1", "HB_MIN_CHUNK_BYTES": "65536", "HB_PIPE_CHUNKS": "16"}, (16, 16)),
                            ({"HB_PIPE_MIN_OUT": "1", "HB_PIPE_CHUNKS": "1"}, (1, 1))):
            hb_env.reset(("HB_PIPE_MIN_OUT", "HB_MIN_CHUNK_BYTES", "HB_PIPE_CHUNKS"), **env)
            t = {}
            assert np.array_equal(batch_digest(alg, data, timing=t), ref)
            assert chunks[0] <= t["chunks"] <= chunks[1], (alg, env, t["chunks"])
            assert np.array_equal(batch_digest_varlen(alg, vdata, off), vref)
            assert np.array_equal(hash_decimal(alg, 10**6, 300000, 9), dref)


@pytest.mark.parametrize("pair", ["0", "1"])
def test_small_rows_pairs(pair, hb_env):
    """Compile-time-width kernel with two rows per thread (HB_SMALL_PAIR, MD5,
    >= 2^20 rows): odd row counts (the last thread's second row missing) and
    every short width, all rows against the oracle."""
    hb_env.set(HB_SMALL_PAIR=pair)
    for L in (16, 32, 48, 64, 128):
        n = (1 << 20) + 1
        data = oracle.fill_random(n * L, 53 + L).reshape(n, L)
        for alg in ALGS:
            assert np.array_equal(batch_digest(alg, data, gpus=[0]), oracle.batch_fixed(alg, data, threads=16)), (alg, L)


@pytest.mark.parametrize("L", [64, 1024])
def test_pdl_stream_order(L):
    """Programmatic dependent launch keeps stream order: (1) a torch kernel
    writes the messages right before each hash launch; (2) a chain of hash
    launches where each consumes the previous one's digests as its messages
    (the producer triggers its dependents before storing them, so only
    griddepcontrol.wait's completion semantics make this correct).  Small
    (k_fixed_small) and TMA (k_fixed_tma_ws) shapes, no synchronisation
    between the launches."""
    import torch

    from paper_2407_09333_b200 import device

    for n in (20000, 70000):  # MD5: the 4+1-warp tile below 2^16 messages, single-warp tiles above
        buf = torch.empty((n, L), dtype=torch.uint8, device="cuda:0")
        outs = []
        for k in range(6):
            buf.fill_(k + 1)
            outs.append(device.hash_fixed("md5", buf))
        torch.cuda.synchronize()
        for k, o in enumerate(outs):
            ref = oracle.batch_fixed("md5", np.full((1, L), k + 1, np.uint8))
            assert np.array_equal(o.cpu().numpy(), np.repeat(ref, n, axis=0)), (n, k)
    per = L // 32  # SM3 digests per L-byte row of the next round
    rows = per ** 3 if L > 64 else 1 << 14
    data = oracle.fill_random(rows * L, 41).reshape(rows, L)
    cur = torch.from_numpy(data).cuda()
    ref = data
    while rows >= per:
        rows //= per
        cur = device.hash_fixed("sm3", cur).reshape(rows, L)
        ref = oracle.batch_fixed("sm3", ref, threads=8).reshape(rows, L)
    torch.cuda.synchronize()
    assert np.array_equal(cur.cpu().numpy(), ref)


@pytest.mark.parametrize("bind", ["1", "0"])
def test_multi_shard_numa_binding(bind, hb_env):
    """A multi-GPU call (here two shards on GPU 0) hands its shards to the
    per-GPU worker threads, each pinned to its GPU's local CPUs (sysfs
    local_cpulist); the digests are unchanged and the caller's own affinity is
    untouched."""
    import os

    hb_env.set(HB_BIND_NUMA=bind)
    n, L = 30001, 200
    data = oracle.fill_random(n * L, 43).reshape(n, L)
    before = os.sched_getaffinity(0)
    for alg in ALGS:
        assert np.array_equal(batch_digest(alg, data, gpus=[0, 0]), oracle.batch_fixed(alg, data, threads=8))
    assert os.sched_getaffinity(0) == before


def test_bind_host_to_gpu():
    """NVML's GPU-local core set becomes this process's affinity (bench.py
    does this per rank before allocating pinned buffers)."""
    import os

    from paper_2407_09333_b200.device import bind_host_to_gpu

    before = os.sched_getaffinity(0)
    try:
        cores = bind_host_to_gpu(0)
        assert cores, "NVML returned no CPU affinity for GPU 0"
        assert set(cores) <= before and os.sched_getaffinity(0) == set(cores)
    finally:
        os.sched_setaffinity(0, before)


def test_hash_batch_and_thread_invariance():
    b = gen_messages(0, 3)
    for alg in ALGS:
        one = hash_batch(alg, b, threads=1)
        eight = hash_batch(alg, b, threads=8)
        assert one == eight
        assert [d.data for d in one] == [oracle.digest(alg, b.message(i)) for i in range(3)]


def test_ratio_invariance_style_sharding():
    # SPEC.md:505 analogue: output independent of how [0,n) is split over devices
    n = _native.device_count()
    data = oracle.fill_random(10**5 * 9, 4).reshape(10**5, 9)
    for alg in ALGS:
        ref = oracle.batch_fixed(alg, data, threads=8)
        assert np.array_equal(batch_digest(alg, data, gpus=[0]), ref)
        assert np.array_equal(batch_digest(alg, data, gpus=list(range(n)) + [0]), ref)  # uneven split, repeated dev


@pytest.mark.parametrize("dec_run", ["1", "0"])
def test_decimal_workload(golden, dec_run, hb_env):
    """HB_DEC_RUN=1 (default): runs-of-ten kernel for widths 2..10 below
    v ~ 1.07e10, the one-message-per-thread kernel elsewhere; 0: the latter only."""
    hb_env.set(HB_DEC_RUN=dec_run)
    # the FMA digit path of the one-message kernel ends at index 2^30; straddle it at every width it serves
    for w in range(1, 10):
        for start, cnt in ((max(0, 10**w - 300), min(300, 10**w)), (2**30 - 150, 300)):
            if start + cnt > 10**w:
                continue
            for alg in ALGS:
                assert np.array_equal(hash_decimal(alg, start, cnt, w),
                                      oracle.batch_fixed(alg, oracle.gen_decimal(start, cnt, w))), (alg, w, start)
    _decimal_common(golden)


def _decimal_common(golden):
    # the 32-bit digit path ends exactly at index 2^32 - 1; straddle it
    start, cnt = 2**32 - 150, 300
    for alg in ALGS:
        assert np.array_equal(hash_decimal(alg, start, cnt, 10), oracle.batch_fixed(alg, oracle.gen_decimal(start, cnt, 10)))
    for row in golden("decimal_batches.json"):
        for alg in ALGS:
            out = hash_decimal(alg, row["start"], row["count"], row["width"])
            assert sha(out) == row[alg]
    for w in list(range(1, 21)) + [25]:
        cnt = min(300, 10**w)
        start = max(0, min(10**w - cnt, 10**w // 3, 2**63))
        msgs = oracle.gen_decimal(start, cnt, w) if w <= 20 else gen_messages(start, cnt, w).as_array()
        for alg in ALGS:
            assert np.array_equal(hash_decimal(alg, start, cnt, w), oracle.batch_fixed(alg, msgs)), (alg, w)


@pytest.mark.ab
@pytest.mark.parametrize("dec_run", ["1", "0"])
@pytest.mark.parametrize("variant", ["1", "fma_digits"])
def test_decimal_workload_ab(golden, variant, dec_run, hb_env):
    hb_env.set(HB_DEC_RUN=dec_run, HB_FMA_DIGITS="0")
    if variant == "fma_digits":
        hb_env.set(HB_FMA_DIGITS="1")
        for w, v in [(w, v) for w in range(1, 10) for v in ("1", "3")]:
            hb_env.set(HB_CONST_VARIANT=v)
            for start, cnt in ((max(0, 10**w - 300), min(300, 10**w)), (2**30 - 150, 300)):
                if start + cnt > 10**w:
                    continue
                for alg in ALGS:
                    assert np.array_equal(hash_decimal(alg, start, cnt, w),
                                          oracle.batch_fixed(alg, oracle.gen_decimal(start, cnt, w))), (alg, w, start)
    else:
        hb_env.set(HB_CONST_VARIANT=variant)
    _decimal_common(golden)


def test_decimal_range_checked():
    """gen_messages' range rule at the C ABI: indices past 10^width
    or a 64-bit wrap are rejected, not silently reduced."""
    lib = _native.lib()
    out = np.empty((10, 16), np.uint8)
    for start, count, width in ((10**9 - 5, 10, 9), (2**64 - 5, 10, 20), (0, 101, 2)):
        rc = lib.hb_hash_decimal(1, start, count, width, out.ctypes.data, None, 0, 0, None)
        assert rc == _native.HB_ERR_INVAL, (start, count, width)
        rc = lib.hb_hash_decimal_dev(1, 0, start, count, width, None, None)
        assert rc == _native.HB_ERR_INVAL
    with pytest.raises(ValueError):
        hash_decimal("md5", 2**64 - 5, 10, 20)


def _decimal_ragged_cases():
    for w in (2, 3, 4, 8, 9, 10):
        for r in range(10):
            for cnt in (c for c in (1, 2, 9, 10, 11, 19, 21, 1283) if c <= 10**w):
                yield w, max(0, min(10**w - cnt, 10**(w - 1) + 37 * 10 + r)), cnt
    for start, cnt in ((10**10 - 1000, 1000), (10**10 - 1001, 1001), (10**10 - 37, 37), (2**32 - 15, 40)):
        yield 10, start, cnt


def test_decimal_runs_ragged():
    """Runs-of-ten kernel: every start residue mod 10 x short counts (first and
    last thread partial, one thread both), the end of the width-10 range and
    the 2^32 boundary (u = v / 10 stays below 2^30 for every width <= 10)."""
    for w, start, cnt in _decimal_ragged_cases():
        for alg in ALGS:
            assert np.array_equal(hash_decimal(alg, start, cnt, w),
                                  oracle.batch_fixed(alg, oracle.gen_decimal(start, cnt, w))), (alg, w, start, cnt)


@pytest.mark.ab
@pytest.mark.parametrize("variant", ["1", "3", "pair", "nopair"])
def test_decimal_runs_ragged_ab(variant, hb_env):
    if variant in ("pair", "nopair"):  # two messages per compression call (MD5 default) or one
        hb_env.set(HB_DEC_PAIR="1" if variant == "pair" else "0")
    else:
        hb_env.set(HB_CONST_VARIANT=variant)
    for w, start, cnt in _decimal_ragged_cases():
        for alg in ALGS:
            assert np.array_equal(hash_decimal(alg, start, cnt, w),
                                  oracle.batch_fixed(alg, oracle.gen_decimal(start, cnt, w))), (alg, w, start, cnt)


def test_error_mapping():
    with pytest.raises(UnknownAlgorithmError):
        digest("sha3", b"")
    with pytest.raises(RuntimeError):
        batch_digest("md5", np.zeros((2, 4), np.uint8), gpus=[999])
    with pytest.raises(ValueError):
        batch_digest_varlen("md5", np.zeros(10, np.uint8), np.array([0, 5, 3], np.uint64))


def test_device_api_torch_streams():
    import torch

    from paper_2407_09333_b200 import device

    n, L = 4099, 512
    buf = torch.empty(n * L, dtype=torch.uint8, device="cuda:0")
    device.fill_random(buf, 1234)
    host = oracle.fill_random(n * L, 1234)
    assert np.array_equal(buf.cpu().numpy(), host)
    msgs = buf.view(n, L)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for alg in ALGS:
            for fl in FLAGS.values():
                out = device.hash_fixed(alg, msgs, flags=fl)
                s.synchronize()
                assert np.array_equal(out.cpu().numpy(), oracle.batch_fixed(alg, host.reshape(n, L), 8))
    # unaligned device rows (L=100 and a 1-byte offset base) go through the generic kernel
    raw = torch.empty(1 + 300 * 100, dtype=torch.uint8, device="cuda:0")
    device.fill_random(raw, 5)
    v = raw[1:].view(300, 100)
    h = raw.cpu().numpy()[1:].reshape(300, 100)
    for alg in ALGS:
        assert np.array_equal(device.hash_fixed(alg, v).cpu().numpy(), oracle.batch_fixed(alg, h))
    # varlen on device with a non-zero base offset
    lens = torch.randint(0, 3000, (5000,), generator=torch.Generator().manual_seed(1))
    off = torch.zeros(5001, dtype=torch.int64)
    off[1:] = torch.cumsum(lens, 0)
    off += 16
    data = torch.empty(int(off[-1]) + 4, dtype=torch.uint8, device="cuda:0")
    device.fill_random(data, 6)
    hdata = data.cpu().numpy()
    d_off = off.cuda()
    for alg in ALGS:
        got = device.hash_varlen(alg, data[16:], d_off).cpu().numpy()
        ref = oracle.batch_varlen(alg, hdata, off.numpy().astype(np.uint64), 8)
        assert np.array_equal(got, ref)


def test_full_size_sampled_and_cross_path():
    """At a BASELINE-scale batch (2^22 x 1 KiB = 4 GiB on device): the TMA and
    direct-load kernels agree bit-for-bit on every row, and a random sample of
    rows equals the oracle on the same counter-generated bytes."""
    import torch

    from paper_2407_09333_b200 import device

    n, L = 1 << 22, 1024
    buf = torch.empty(n * L, dtype=torch.uint8, device="cuda:0")
    device.fill_random(buf, 2)
    msgs = buf.view(n, L)
    rng = np.random.default_rng(0)
    rows = np.unique(np.concatenate([rng.integers(0, n, 2048), [0, 1, n - 1]]))
    for alg in ALGS:
        a = device.hash_fixed(alg, msgs)
        b = device.hash_fixed(alg, msgs, flags=_native.HB_FLAG_NO_TMA)
        torch.cuda.synchronize()
        assert torch.equal(a, b)
        got = a.cpu().numpy()[rows]
        sample = np.stack([oracle.fill_random(L, 2, int(r) * L) for r in rows])
        assert np.array_equal(got, oracle.batch_fixed(alg, sample, 8))
    del buf


@pytest.mark.ab
@pytest.mark.parametrize("cfg", ["1x3", "2x2", "2x3", "ws2", "ws3", "ws2x2", "ws3x2", "ws3u", "ws3x2u", "ws3n",
                                 "w1x1", "w1x2", "w1x4", "w1x4s2", "w1x2p", "ws3v6", "w1x2s4", "w1x2s2", "w1x3", "w1x4p"])
def test_tma_tile_configs_and_variants(cfg, hb_env):
    """Every compiled TMA tile configuration x round variant is bit-exact
    (the tuned default is only one of them; $HB_TMA_CFG/$HB_VARIANT select)."""
    variants = {"1x3": ["0", "1", "2", "3"], "ws3": ["0", "1", "2", "3", "4", "5", "6", "7"],
                "w1x1": ["1", "3"], "w1x2": ["1", "3", "4"], "w1x4": ["1", "3", "5"], "w1x4s2": ["1"],
                "w1x2p": ["1", "4", "6"], "ws3v6": ["6"], "w1x2s4": ["1"], "w1x2s2": ["1"], "w1x3": ["1"], "w1x4p": ["1"]}.get(
        cfg, ["1", "3"] if cfg.endswith("x2") and cfg.startswith("ws") else ["0", "1"] if cfg.startswith("ws")
        else ["0", "1", "2"])
    hb_env.set(HB_TMA_CFG=cfg)
    for L in (16, 48, 64, 112, 128, 1024, 1040):
        n = 333
        data = oracle.fill_random(n * L, 7 * L + 1).reshape(n, L)
        refs = {a: oracle.batch_fixed(a, data, threads=8) for a in ALGS}
        for v in variants:
            hb_env.set(HB_VARIANT=v)
            for alg in ALGS:
                assert np.array_equal(batch_digest(alg, data), refs[alg]), (cfg, v, alg, L)


def test_duty_ratio_invariance():
    """SPEC.md:505 on the GPU: 10^5 x 9-byte generated messages give bit-identical
    digests for every duty-ratio split on the 0.02 grid (two bindings here map to
    GPU 0 and, when present, GPU 1; on one GPU both bindings share it)."""
    n_dev = _native.device_count()
    gpus = [0, 1 if n_dev > 1 else 0]
    msgs = gen_messages(0, 10**5).as_array()
    for alg in ALGS:
        ref = oracle.batch_fixed(alg, msgs, threads=8)
        for k in range(0, 51):
            x = k / 50
            got = batch_digest(alg, msgs, gpus=gpus, ratios=[x, 1.0 - x])
            assert np.array_equal(got, ref), (alg, x)


GEOMETRY_KEYS = ("HB_SMALL_N", "HB_DIRECT_MAX_L", "HB_NO_SMALL_KERNEL", "HB_CONST_VARIANT", "HB_CHAIN_N",
                 "HB_MD5_NB3_N")


def _geometry_arms(alg, arms, hb_env):
    for L in (16, 32, 48, 64, 96, 128, 144, 1024):
        n = 3001
        data = oracle.fill_random(n * L, 5 * L + 3).reshape(n, L)
        ref = oracle.batch_fixed(alg, data, threads=8)
        for env in arms:
            hb_env.reset(GEOMETRY_KEYS, **env)
            assert np.array_equal(batch_digest(alg, data), ref), (alg, L, env)


@pytest.mark.parametrize("alg", ALGS)
def test_batch_geometry_dispatch_matches(alg, hb_env):
    """The fixed-width dispatch picks a kernel shape by batch geometry (direct
    loads for short rows, one message per thread below $HB_SMALL_N, the tuned
    tiles otherwise); every shape must give the oracle's digests."""
    _geometry_arms(alg, [{}, {"HB_SMALL_N": "0", "HB_DIRECT_MAX_L": "0"},
                         {"HB_SMALL_N": str(1 << 40), "HB_DIRECT_MAX_L": "0"},
                         # MD5's single-warp two- and three-messages-per-thread tiles at every width
                         {"HB_CHAIN_N": "0", "HB_DIRECT_MAX_L": "0"},
                         {"HB_CHAIN_N": "0", "HB_MD5_NB3_N": "0", "HB_DIRECT_MAX_L": "0"}], hb_env)


@pytest.mark.ab
@pytest.mark.parametrize("alg", ALGS)
def test_batch_geometry_dispatch_ab(alg, hb_env):
    _geometry_arms(alg, [{"HB_NO_SMALL_KERNEL": "1"}, {"HB_CONST_VARIANT": "0"}, {"HB_SMALL_CTA": "32"}], hb_env)


def _every_length_cases():
    lens = np.array([L for L in range(261) for _ in range(3)], np.uint64)
    np.random.default_rng(5).shuffle(lens)
    for shift in (0, 1, 3, 7, 13):
        off = np.zeros(len(lens) + 1, np.uint64)
        off[1:] = np.cumsum(lens)
        off += np.uint64(shift)
        yield shift, off, oracle.fill_random(int(off[-1]) + 5, 17 + shift)


@pytest.mark.zero_copy
@pytest.mark.parametrize("path", ["ring", "zero_copy"])
@pytest.mark.parametrize("alg", ALGS)
def test_varlen_every_length_and_alignment(alg, path, hb_env):
    """Every length 0..260 (x3, shuffled, so message starts take every
    alignment mod 16) in one batch and in partial warps (n not a multiple of
    32), with several leading offsets, sorted and unsorted (the ring: device
    buffers, length sort from 1,024 messages) and through the small-call
    zero-copy path (mapped host memory, unsorted)."""
    hb_env.set(HB_ZERO_COPY_MAX=0 if path == "ring" else ZC_DEFAULT)
    for shift, off, buf in _every_length_cases():
        ref = oracle.batch_varlen(alg, buf, off, threads=8)
        for k in (len(off) - 1, 31, 33, 1):
            for fl in (0, _native.HB_FLAG_NO_SORT, _native.HB_FLAG_VARLEN_COOP_OFF):
                got = batch_digest_varlen(alg, buf, off[: k + 1], flags=fl)
                assert np.array_equal(got, ref[:k]), (alg, shift, k, fl)


@pytest.mark.ab
@pytest.mark.parametrize("alg", ALGS)
def test_varlen_every_length_and_alignment_ab(alg, hb_env):
    C = _native.HB_FLAG_VARLEN_COOP
    hb_env.set(HB_ZERO_COPY_MAX=0)  # device buffers and the length sort, as the arms were measured
    for shift, off, buf in _every_length_cases():
        ref = oracle.batch_varlen(alg, buf, off, threads=8)
        for k in (len(off) - 1, 31, 33, 1):
            assert np.array_equal(batch_digest_varlen(alg, buf, off[: k + 1], flags=C), ref[:k]), (alg, shift, k)
        for env, fl in (({"HB_VC_STAGES": "3"}, C), ({"HB_VC_STAGES": "2"}, C), ({"HB_VC_PF": "128"}, C),
                        ({"HB_VC_PF": "0"}, C), ({"HB_VARLEN_PREFETCH": "1"}, 0), ({"HB_VARLEN_BULK": "3"}, 0),
                        ({"HB_VARLEN_BULK": "5"}, 0), ({"HB_VARLEN_LD": "32"}, 0), ({"HB_VARLEN_LD": "16"}, 0),
                        ({"HB_VARLEN_LD": "32", "HB_VARLEN_Q": "4"}, 0),
                        # lean block loop: runtime / per-class realignment, round variants, L2 policies
                        ({"HB_VARLEN_KERNEL": "40"}, 0), ({"HB_VARLEN_KERNEL": "41"}, 0),
                        ({"HB_VARLEN_KERNEL": "42"}, 0), ({"HB_VARLEN_KERNEL": "44"}, 0),
                        ({"HB_VARLEN_KERNEL": "46"}, 0), ({"HB_VARLEN_KERNEL": "47"}, 0),
                        ({"HB_VARLEN_KERNEL": "48"}, 0), ({"HB_VARLEN_KERNEL": "49"}, 0),
                        ({"HB_VARLEN_KERNEL": "50"}, 0), ({"HB_VARLEN_KERNEL": "51"}, 0),
                        ({"HB_VARLEN_KERNEL": "52"}, 0), ({"HB_VARLEN_KERNEL": "53"}, 0),
                        ({"HB_VARLEN_KERNEL": "54"}, 0), ({"HB_VARLEN_KERNEL": "55"}, 0),
                        ({"HB_VARLEN_KERNEL": "56"}, 0)):
            hb_env.set(**env)
            got = batch_digest_varlen(alg, buf, off, flags=fl)
            assert np.array_equal(got, ref), (alg, shift, env)
            hb_env.clear(*env)


def test_hash_batch_var_message_batch():
    """§8(f) row 3: a mixed-length batch through hash_batch is the scalar
    digest of every message (the reference's only variable-length path)."""
    from paper_2407_09333_b200.crypto import VarMessageBatch

    rng = np.random.default_rng(3)
    msgs = [bytes(rng.integers(0, 256, int(L), dtype=np.uint8)) for L in rng.integers(0, 300, 2500)]
    b = VarMessageBatch.from_messages(msgs)
    for alg in ALGS:
        got = hash_batch(alg, b, threads=4)
        ref = oracle.batch_varlen(alg, np.frombuffer(b.data, np.uint8), b.offsets_array(), threads=8)
        assert [d.data for d in got] == [bytes(r) for r in ref]
        assert all(d.alg == alg for d in got)


def test_fixed_hash_graph_replay():
    """CUDA-graph capture of a device-resident launch: replays after refilling
    the bound input in place give the oracle's digests."""
    import torch

    from paper_2407_09333_b200 import device

    n, L = 65536, 64
    buf = torch.empty(n * L, dtype=torch.uint8, device="cuda:0")
    for alg in ALGS:
        g = None
        for seed in (1, 2, 3):
            device.fill_random(buf, seed)
            if g is None:
                g = device.FixedHashGraph(alg, buf.view(n, L))
                assert g.kernels_per_replay >= 1
            out = g.replay()
            torch.cuda.synchronize()
            rows = np.array([0, 1, 777, n - 1])
            sample = np.stack([oracle.fill_random(L, seed, int(r) * L) for r in rows])
            assert np.array_equal(out.cpu().numpy()[rows], oracle.batch_fixed(alg, sample)), (alg, seed)


@pytest.mark.parametrize("late", ["1", "0"])
def test_input_ready_shared_out_order(late, hb_env):
    """HB_FLAG_INPUT_READY launches compute before griddepcontrol.wait
    ($HB_LATE_WAIT=1: consecutive batches overlap) and store only after it, so
    back-to-back launches over DIFFERENT inputs into the SAME digest buffer
    leave exactly the last launch's digests -- for the compile-time-width
    kernel, the 4+1-warp tile and the single-warp tiles (2 and 3 messages per
    thread), sub-wave grids (released at entry) and multi-wave ones."""
    import torch

    from paper_2407_09333_b200 import device

    hb_env.set(HB_LATE_WAIT=late)
    flag = _native.HB_FLAG_INPUT_READY
    for alg, n, L, env in (("sha1", 65536, 64, {}), ("md5", 20000, 1024, {}), ("md5", 70000, 1024, {}),
                           ("md5", 300000, 256, {}), ("md5", 70000, 320, {"HB_MD5_NB3_N": "0"}),
                           ("sm3", 9000, 512, {}), ("sm3", 65536, 1024, {})):
        hb_env.set(HB_LATE_WAIT=late, **env)
        d = {"sha1": 20, "md5": 16, "sm3": 32}[alg]
        copies = []
        for k in range(6):
            b = torch.empty(n * L, dtype=torch.uint8, device="cuda:0")
            device.fill_random(b, 300 + k)
            copies.append(b.view(n, L))
        out = torch.empty((n, d), dtype=torch.uint8, device="cuda:0")
        torch.cuda.synchronize()
        for rep in range(3):
            for c in copies:
                device.hash_fixed(alg, c, out=out, flags=flag)
        torch.cuda.synchronize()
        full = oracle.batch_fixed(alg, copies[-1].cpu().numpy(), threads=8)
        assert np.array_equal(out.cpu().numpy(), full), (alg, n, L, env, late)
        hb_env.clear(*env)


def test_input_ready_early_start():
    """HB_FLAG_INPUT_READY: back-to-back launches over rotating, already
    written inputs start reading before the previous grid completes (early
    loads, early release of the next grid for sub-wave grids); every pass's
    digests equal the oracle's, for the compile-time-width kernel, the TMA
    ring (sub-wave and multi-wave grids, ragged last CTA) and a one-block
    message.  A fill kernel that rewrites the input right before a flagged
    launch is ordered by a plain (unflagged) launch in between."""
    import torch

    from paper_2407_09333_b200 import device

    flag = _native.HB_FLAG_INPUT_READY
    for alg, n, L in (("sha1", 65536, 64), ("md5", 65536, 1024), ("sm3", 1000, 256), ("md5", 300000, 256),
                      ("sha1", 4099, 48), ("md5", 70000, 16)):
        d = {"sha1": 20, "md5": 16, "sm3": 32}[alg]
        copies = []
        for k in range(3):
            b = torch.empty(n * L, dtype=torch.uint8, device="cuda:0")
            device.fill_random(b, 100 + k)
            copies.append(b.view(n, L))
        outs = [torch.empty((n, d), dtype=torch.uint8, device="cuda:0") for _ in copies]
        for rep in range(2):
            for b, o in zip(copies, outs):
                device.hash_fixed(alg, b, out=o, flags=flag)
        g = device.FixedHashGraph(alg, copies, flags=flag, repeats=2)
        g.replay()
        torch.cuda.synchronize()
        for k, o in enumerate(outs):
            rows = np.array([0, 1, n // 2, n - 1])
            sample = np.stack([oracle.fill_random(L, 100 + k, int(r) * L) for r in rows])
            ref = oracle.batch_fixed(alg, sample)
            assert np.array_equal(o.cpu().numpy()[rows], ref), (alg, n, L, k)
        last = len(copies) - 1
        assert np.array_equal(g.out.cpu().numpy()[rows], ref), (alg, n, L, "graph")
        full = oracle.batch_fixed(alg, copies[0].cpu().numpy(), threads=8)
        assert np.array_equal(outs[0].cpu().numpy(), full), (alg, n, L, "full")
        # rewrite an input, then hash it unflagged: the result follows the new bytes
        device.fill_random(copies[last].view(-1), 555)
        device.hash_fixed(alg, copies[last], out=outs[last])
        torch.cuda.synchronize()
        sample = np.stack([oracle.fill_random(L, 555, int(r) * L) for r in rows])
        assert np.array_equal(outs[last].cpu().numpy()[rows], oracle.batch_fixed(alg, sample))


def test_varlen_input_ready_sort_overlap():
    """HB_FLAG_INPUT_READY on varlen launches: MD5's windowed sort starts while
    the preceding kernel drains (no griddepcontrol.wait), released by the
    previous varlen hash kernel once its threads have read their permutation
    entries -- here three different batches back to back on ONE scratch buffer
    (each sort overwrites the permutation the previous hash kernel read), after
    a fixed-width launch, with no synchronisation in between; every digest
    equals the oracle's."""
    import torch

    from paper_2407_09333_b200 import device

    flag = _native.HB_FLAG_INPUT_READY
    rng = np.random.default_rng(31)
    cases = []
    for k, (n, maxlen) in enumerate(((20000, 3000), (70000, 700), (5000, 9000))):
        lens = rng.integers(0, maxlen + 1, n).astype(np.int64)
        off = np.zeros(n + 1, np.int64)
        off[1:] = np.cumsum(lens)
        host = oracle.fill_random(int(off[-1]), 70 + k)
        cases.append((torch.from_numpy(host).cuda(), torch.from_numpy(off).cuda(), host, off))
    scratch = torch.empty(int(_native.lib().hb_varlen_scratch_bytes(70000)), dtype=torch.uint8, device="cuda:0")
    fixed = torch.zeros((100000, 1024), dtype=torch.uint8, device="cuda:0")
    for alg in ALGS:
        torch.cuda.synchronize()
        outs = []
        for rep in range(2):
            device.hash_fixed(alg, fixed, flags=flag)
            for d, o, _, _ in cases:
                outs.append(device.hash_varlen(alg, d, o, scratch=scratch, flags=flag, offset_base=0))
        torch.cuda.synchronize()
        for k, (_, _, host, off) in enumerate(cases):
            ref = oracle.batch_varlen(alg, host, off.astype(np.uint64), threads=8)
            for rep in range(2):
                assert np.array_equal(outs[rep * len(cases) + k].cpu().numpy(), ref), (alg, k, rep)


def test_out_argument_reuse_and_pinned():
    """Digests written into a caller buffer (pageable or page-locked) equal a fresh result."""
    import ctypes

    n, L = 3000, 100
    data = oracle.fill_random(n * L, 77).reshape(n, L)
    lib = _native.lib()
    hp = lib.hb_alloc_pinned(n * 32)
    try:
        pinned = np.ctypeslib.as_array(ctypes.cast(hp, ctypes.POINTER(ctypes.c_uint8)), shape=(n * 32,))
        for alg in ALGS:
            d = {"sha1": 20, "md5": 16, "sm3": 32}[alg]
            ref = oracle.batch_fixed(alg, data, threads=8)
            for out in (np.empty((n, d), np.uint8), pinned[: n * d].reshape(n, d)):
                got = batch_digest(alg, data, out=out)
                assert got is out and np.array_equal(out, ref)
            dec = hash_decimal(alg, 5, n, 9, out=np.empty((n, d), np.uint8))
            assert np.array_equal(dec, oracle.batch_fixed(alg, gen_messages(5, n, 9).as_array(), threads=8))
    finally:
        lib.hb_free_pinned(hp)


def test_concurrent_callers_thread_safe():
    """The reference calls the boundary from pool threads (_fast_digest,
    executor.py:596-599; hash_batch's ThreadPool, batch.py:310-313): concurrent
    engine calls from many threads (GIL released in ctypes) must each get
    their own correct digests."""
    from concurrent.futures import ThreadPoolExecutor

    jobs = []
    for k in range(24):
        alg = ALGS[k % 3]
        n, L = 500 + 37 * k, [64, 100, 1024, 9, 200][k % 5]
        data = oracle.fill_random(n * L, 1000 + k).reshape(n, L)
        jobs.append((alg, data, oracle.batch_fixed(alg, data, threads=4)))
    lens = np.random.default_rng(9).integers(0, 3000, 1500).astype(np.uint64)
    off = np.zeros(len(lens) + 1, np.uint64)
    off[1:] = np.cumsum(lens)
    vdata = oracle.fill_random(int(off[-1]), 55)
    vref = {a: oracle.batch_varlen(a, vdata, off, threads=4) for a in ALGS}

    def run(j):
        alg, data, ref = jobs[j]
        ok = np.array_equal(batch_digest(alg, data), ref)
        return ok and np.array_equal(batch_digest_varlen(alg, vdata, off), vref[alg])

    with ThreadPoolExecutor(max_workers=8) as ex:
        assert all(ex.map(run, range(len(jobs))))


@pytest.mark.parametrize("ld", ["16", pytest.param("32", marks=pytest.mark.ab)])
def test_varlen_last_message_at_buffer_end(ld, hb_env):
    """The wide loads never read past the data buffer: the batch's last message
    ends exactly at the end of a device allocation whose size is not a
    multiple of 32 (checked with every tail length 0..95)."""
    import torch

    from paper_2407_09333_b200 import device

    hb_env.set(HB_VARLEN_LD=ld)
    for tail in range(0, 96):
        lens = np.array([100, 37, 64 + tail], np.int64)
        off = np.zeros(4, np.int64)
        off[1:] = np.cumsum(lens)
        total = int(off[-1])
        host = oracle.fill_random(total, 400 + tail)
        data = torch.from_numpy(host).cuda()  # exactly `total` bytes
        d_off = torch.from_numpy(off).cuda()
        for alg in ALGS:
            got = device.hash_varlen(alg, data, d_off, offset_base=0).cpu().numpy()
            assert np.array_equal(got, oracle.batch_varlen(alg, host, off.astype(np.uint64))), (alg, tail, ld)


def test_accel_generic_equivalence_1e6():
    """the accelerated SHA-1 path equals the generic one on 10^6
    random messages (here both are the GPU kernel; the oracle is the judge)."""
    n, L = 10**6, 23
    data = oracle.fill_random(n * L, 265).reshape(n, L)
    ref = oracle.batch_fixed("sha1", data, threads=8)
    assert np.array_equal(batch_digest("sha1", data, accel=True), ref)
    assert np.array_equal(batch_digest("sha1", data, accel=False), ref)
    assert [d.data for d in hash_batch("sha1", MessageBatch(n, L, data.tobytes()), accel=True)[:1000]] == \
        [bytes(r) for r in ref[:1000]]


# ------------------------------------------------------------ engine (r2) --
def test_small_default_call_runs_on_one_gpu():
    """A drop-in call with the default device set ("all GPUs") on a small
    batch -- 4 KiB, the size of the reference executor's per-thread
    _fast_digest slices -- runs on exactly one GPU (no fan-out, no worker
    hand-off); an explicit list with two shards goes to the GPU workers."""
    data = oracle.fill_random(64 * 64, 3).reshape(64, 64)
    for alg in ALGS:
        t = {}
        got = batch_digest(alg, data, timing=t)
        assert np.array_equal(got, oracle.batch_fixed(alg, data))
        assert t["shards"] == 1 and bin(t["device_mask"]).count("1") == 1, t
        t = {}
        assert np.array_equal(batch_digest(alg, data, gpus=[0, 0], timing=t), oracle.batch_fixed(alg, data))
        assert t["shards"] == 2 and t["device_mask"] == 1, t


def test_timing_is_a_union_of_busy_intervals(hb_env):
    """hb_timing's per-stage times are unions of the chunk ring's busy
    intervals (overlapping slots are not double-counted), each at most the
    call's wall time; the per-chunk timeline has one span per stage and chunk."""
    n, L = 1 << 16, 1024
    data = oracle.fill_random(n * L, 21).reshape(n, L)
    for env in ({}, {"HB_CHUNK_BYTES": 4 << 20}):
        hb_env.reset(("HB_CHUNK_BYTES",), **env)
        t = {}
        out = batch_digest("md5", data, timing=t, gpus=[0])
        assert t["chunks"] >= (16 if env else 1)
        for k in ("h2d_ms", "kernel_ms", "d2h_ms"):
            assert 0 < t[k] <= t["total_ms"] * 1.05 + 0.05, (k, t)
        spans = _native.last_timeline()
        kern = [s for s in spans if s["stage"] == "kernel"]
        assert len(kern) == t["chunks"]
        assert all(s["t1_ms"] >= s["t0_ms"] for s in spans)
        assert np.array_equal(out[:7], oracle.batch_fixed("md5", data[:7]))


def test_engine_tuning_reload(hb_env):
    data = oracle.fill_random(4000 * 256, 8).reshape(4000, 256)
    t = {}
    batch_digest("sha1", data, timing=t, gpus=[0])
    assert t["chunks"] == 1
    hb_env.set(HB_CHUNK_BYTES=65536)
    t = {}
    assert np.array_equal(batch_digest("sha1", data, timing=t, gpus=[0]), oracle.batch_fixed("sha1", data))
    assert t["chunks"] == -(-4000 // 256), t


def test_engine_budget():
    b = _native.engine_budget(0)
    info = _native.device_info(0)
    assert 0 < b["budget_bytes"] <= info["total_mem"]
    assert 0 < b["chunk_cap_bytes"] <= 256 << 20


@pytest.mark.parametrize("n,L,expect,expect_md5", [(1 << 18, 1024, "k_fixed_tma_ws", "k_fixed_tma_w1"),
                                                   (4096, 1024, "k_fixed_tma_ws", "k_fixed_tma_ws"),
                                                   (4096, 64, "k_fixed_small", "k_fixed_small"),
                                                   (4096, 96, "k_fixed_direct", "k_fixed_direct"),
                                                   (4096, 100, "k_generic", "k_generic")])
def test_last_kernel_name(n, L, expect, expect_md5):
    """hb_last_kernel_name names the kernel that actually ran (what the bench
    reports as roofline.kernel), for the device and host-buffer paths."""
    import torch

    from paper_2407_09333_b200 import device

    msgs = torch.zeros((n, L), dtype=torch.uint8, device="cuda:0")
    device.hash_fixed("sha1", msgs)
    name = _native.last_kernel_name()
    assert name.startswith(f"void hb::{expect}<") or expect in name, name
    batch_digest("md5", np.zeros((n, L), np.uint8), gpus=[0, 0])  # two shards on the workers
    assert expect_md5 in _native.last_kernel_name()
    device.hash_decimal("md5", 0, 1000, 9)
    assert "k_decimal_run" in _native.last_kernel_name()


def test_device_wrappers_reject_bad_buffers():
    """the device-resident wrappers check what the kernels will
    dereference (offsets on the data's device, contiguous inputs, an `out`
    of the right shape, dtype, device and alignment)."""
    import torch

    from paper_2407_09333_b200 import device

    msgs = torch.zeros((100, 64), dtype=torch.uint8, device="cuda:0")
    with pytest.raises(ValueError):
        device.hash_fixed("md5", msgs, out=torch.empty((99, 16), dtype=torch.uint8, device="cuda:0"))
    with pytest.raises(ValueError):
        device.hash_fixed("md5", msgs, out=torch.empty((100, 16), dtype=torch.int32, device="cuda:0"))
    with pytest.raises(ValueError):
        big = torch.empty(100 * 16 + 1, dtype=torch.uint8, device="cuda:0")
        device.hash_fixed("md5", msgs, out=big[1:].view(100, 16))
    with pytest.raises(ValueError):
        device.hash_fixed("md5", msgs, out=torch.empty((100, 16), dtype=torch.uint8))
    data = torch.zeros(1000, dtype=torch.uint8, device="cuda:0")
    with pytest.raises(ValueError):
        device.hash_varlen("md5", data, torch.tensor([0, 10, 20]))
    with pytest.raises(ValueError):
        device.hash_varlen("md5", data[::2], torch.tensor([0, 10, 20], device="cuda:0"))
    ok = device.hash_varlen("md5", data, torch.tensor([0, 10, 20], device="cuda:0"))
    torch.cuda.synchronize()
    assert np.array_equal(ok.cpu().numpy(), oracle.batch_varlen("md5", np.zeros(20, np.uint8),
                                                               np.array([0, 10, 20], np.uint64)))
