"""The B200 runtime for lowered *hyper* hash programs.

CPU tests: the lowering restatement reproduces the reference compiler's
printed output byte for byte on every golden case, and the printed form
round-trips through the parser (and, when the reference package is importable
in the authoring container, through the ``HirModule`` adapter).
GPU tests: every golden program executes on the B200 with the reference
simulator's output bytes, batch counts and copied bytes.
"""

import hashlib
import os
import sys

import numpy as np
import pytest

from paper_2407_09333_b200.crypto import gen_messages
from paper_2407_09333_b200.runtime import (
    DeviceSpec,
    DeviceTable,
    ExecError,
    LoweringError,
    ProgramError,
    Workload,
    execute,
    execute_batched,
    from_hir,
    lower_hash_batch,
    parse,
    run_point,
)

REF_SRC = "/root/reference/pkg/src"


def cases(golden):
    return golden("lowered.json")["cases"]


def table(case, ordinals=None):
    host = DeviceSpec("host", kind="host", threads=4, sha_accel=case["host_sha_accel"])
    accels = tuple(DeviceSpec(d, kind="cuda", ordinal=(ordinals or {}).get(d, 0), mem_bytes=m,
                              sha_accel=d in case["accel_sha"]) for d, m in case["mem_bytes"].items())
    return DeviceTable(host, accels)


def test_parse_format_roundtrip(golden):
    for c in cases(golden):
        prog = parse(c["text"], ["msgs", "out"])
        assert prog.format() == c["text"], c["name"]


def test_lowering_matches_reference_compiler(golden):
    """lower_hash_batch == run_pipeline(build_hash_module(...)) printed, every case."""
    for c in cases(golden):
        prog = lower_hash_batch(c["alg"], c["count"], c["width"], c["bindings"], table(c))
        assert prog.format() == c["text"], c["name"]


def test_lowering_rejects_bad_ratios():
    t = DeviceTable(DeviceSpec("host", kind="host"), (DeviceSpec("gpu0"),))
    with pytest.raises(LoweringError):
        lower_hash_batch("md5", 10, 9, [("gpu0", 0.5)], t)
    with pytest.raises(ValueError):
        lower_hash_batch("nope", 10, 9, [("gpu0", 1.0)], t)


def test_parser_rejects_non_hash_programs():
    bad = 'func @main(%0: buf<i8, 9>) {\n  %1 = load %0[%0] : i8\n  return\n}\n'
    with pytest.raises(ProgramError):
        parse(bad)
    body = ('func @main(%0: buf<i64, 4>) {\n  par.loop %1 = 0 to 4 device("gpu0") {\n'
            '    store %1, %0[%1]\n    yield\n  }\n  return\n}\n')
    with pytest.raises(ProgramError):
        parse(body)


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference package not present (authoring container only)")
def test_hir_adapter_matches_text(golden):
    sys.path.insert(0, REF_SRC)
    try:
        from hetoc.hir.parser import parse as ref_parse
    finally:
        sys.path.remove(REF_SRC)
    for c in cases(golden):
        mod = ref_parse(c["text"])
        mod.functions[0].param_names = ["msgs", "out"]
        assert from_hir(mod).format() == c["text"], c["name"]


# ---------------------------------------------------------------- on the GPU
def _gpu_table(case):
    from paper_2407_09333_b200 import _native

    n = _native.device_count()
    return table(case, {d: i % n for i, d in enumerate(case["mem_bytes"])})


@pytest.mark.gpu
def test_golden_programs_execute_on_gpu(golden):
    for c in cases(golden):
        if c["name"] == "md5_host_share":
            continue
        msgs = gen_messages(0, c["count"], c["width"]).data
        for prog in (parse(c["text"], ["msgs", "out"]),
                     lower_hash_batch(c["alg"], c["count"], c["width"], c["bindings"], table(c))):
            rep = execute_batched(prog, _gpu_table(c), {"msgs": msgs})
            assert hashlib.sha256(rep.outputs["out"]).hexdigest() == c["out_sha256"], c["name"]
            for d in c["mem_bytes"]:
                assert rep.batch_count[d] == c["batch_count"][d], (c["name"], d)
                assert rep.bytes_copied[d] == c["bytes_copied"][d], (c["name"], d)
            assert rep.max_wall() > 0 and all(v >= 0 for v in rep.compute_s.values())


@pytest.mark.gpu
def test_host_share_and_capacity_errors(golden):
    by = {c["name"]: c for c in cases(golden)}
    c = by["md5_host_share"]
    with pytest.raises(ExecError, match="no CPU hash path"):
        execute_batched(c["text"], _gpu_table(c), {"msgs": gen_messages(0, c["count"], c["width"]).data},
                        param_names=["msgs", "out"])
    c = by["sha1_many_batches_accel"]  # over capacity without batching: the arena refuses (arena.py:40-44)
    with pytest.raises(ExecError, match="over capacity"):
        execute(c["text"], _gpu_table(c), {"arg0": gen_messages(0, c["count"], c["width"]).data})


@pytest.mark.gpu
def test_run_point_gpu_splits():
    import oracle
    from paper_2407_09333_b200 import _native

    n = _native.device_count()
    w = Workload("sm3", 20011, 9)
    ref = oracle.batch_fixed("sm3", gen_messages(0, w.count, w.width).as_array(), threads=8).tobytes()
    host = DeviceSpec("host", kind="host", threads=os.cpu_count() or 1)
    for mem in (1 << 30, 100000):  # one batch, then many sub-batches per GPU
        devs = DeviceTable(host, tuple(DeviceSpec(f"gpu{i}", ordinal=i % n, mem_bytes=mem) for i in range(2)))
        for ratios in ((0.5, 0.5), (0.0, 1.0), (0.93, 0.07)):
            r = run_point(w, devs, ratios, keep_digests=True)
            assert r.digests == ref, (mem, ratios)
            if mem == 100000 and ratios == (0.5, 0.5):
                assert all(b > 1 for b in r.batches.values())


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference package not present (authoring container only)")
def test_from_reference_device_table():
    """A reference DeviceTable maps onto GPUs with its capacities kept; a
    host-mapped accelerator is refused (no CPU hash path)."""
    from paper_2407_09333_b200.runtime import DeviceConfigError, from_reference

    sys.path.insert(0, REF_SRC)
    try:
        from hetoc.runtime.devices import DeviceSpec as RSpec, DeviceTable as RTable
    finally:
        sys.path.remove(REF_SRC)
    ref = RTable(RSpec("host", kind="host", threads=8, sha_accel=True),
                 (RSpec("gpu0", mem_bytes=5000), RSpec("gpu1", mem_bytes=1 << 20, sha_accel=True)))
    t = from_reference(ref, {"gpu1": 3})
    assert [(a.id, a.kind, a.ordinal, a.mem_bytes, a.sha_accel) for a in t.accels] == \
        [("gpu0", "cuda", 0, 5000, False), ("gpu1", "cuda", 3, 1 << 20, True)]
    assert t.host.sha_accel and t.host.threads == 8
    with pytest.raises(DeviceConfigError):
        from_reference(RTable(RSpec("host", kind="host"), (RSpec("acc", host_mapped=True),)))


@pytest.mark.parametrize("make", [
    lambda: DeviceSpec(""),
    lambda: DeviceSpec("g", kind="simulated_accel"),
    lambda: DeviceSpec("g", threads=0),
    lambda: DeviceSpec("g", mem_bytes=0),
    lambda: DeviceSpec("g", ordinal=-1),
    lambda: DeviceTable(DeviceSpec("h", kind="cuda")),
    lambda: DeviceTable(DeviceSpec("h", kind="host"), (DeviceSpec("h"),)),
    lambda: DeviceTable(DeviceSpec("h", kind="host"), (DeviceSpec("g"), DeviceSpec("g", ordinal=1))),
    lambda: DeviceTable(DeviceSpec("h", kind="host"), (DeviceSpec("g", kind="host"),)),
    lambda: DeviceTable(DeviceSpec("h", kind="host")).resolve("gpu9"),
])
def test_device_table_rejects(make):
    """Every malformed spec or table, and an unknown id, raises DeviceConfigError."""
    from paper_2407_09333_b200.runtime import DeviceConfigError
    with pytest.raises(DeviceConfigError):
        make()


# ------------------------------------------------- variable length (§8(f) 3)
def _var_table(mem=1 << 30, k=3, ordinals=None):
    host = DeviceSpec("host", kind="host", threads=4)
    return DeviceTable(host, tuple(DeviceSpec(f"gpu{i}", kind="cuda", ordinal=(ordinals or {}).get(i, 0),
                                              mem_bytes=mem) for i in range(k)))


def _var_batch(n, seed, maxlen=3000, base=0):
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, maxlen + 1, n).astype(np.int64)
    lens[::53] = 0
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum(lens)
    off += base
    return off


def test_varlen_lowering_structure_and_roundtrip():
    """Offsets re-based per shard: binding j's group copies bytes
    [offsets[s], offsets[e]) and offsets [s, e] and launches with
    offset_base = offsets[s]; digests go back to s*dlen.  Printed text
    round-trips through the parser."""
    from paper_2407_09333_b200.passes import partition_range
    from paper_2407_09333_b200.runtime import VarDigestLoop, lower_hash_batch_varlen

    off = _var_batch(1000, 1, base=7)
    ratios = [0.25, 0.5, 0.25]
    prog = lower_hash_batch_varlen("sm3", off, [(f"gpu{i}", r) for i, r in enumerate(ratios)], _var_table())
    text = prog.format()
    assert parse(text, ["msgs", "offsets", "out"]).format() == text
    assert "crypto.digest_varlen" in text and "msg_len" not in text
    launches = [o for o in prog.ops if o.opcode == "dev.launch"]
    bounds = partition_range(0, 1000, ratios)
    assert len(launches) == 3
    for op, (s, e) in zip(launches, bounds):
        assert isinstance(op.body, VarDigestLoop)
        assert (op.attrs["lb"], op.attrs["ub"], op.attrs["offset"]) == (0, e - s, s)
        assert op.body.offset_base == off[s]
    copies = [o for o in prog.ops if o.opcode == "hyper.memcpy"]
    data_in = [c for c in copies if c.operands[0] == 0]
    assert [(c.attrs["src_off"], c.attrs["count"]) for c in data_in] == \
        [(int(off[s]), int(off[e] - off[s])) for s, e in bounds]
    outs = [c for c in copies if c.operands[1] == 2]
    assert [c.attrs["dst_off"] for c in outs] == [s * 32 for s, _ in bounds]
    # bindings with an empty range are dropped, host bindings refused
    p2 = lower_hash_batch_varlen("md5", off, [("gpu0", 1.0), ("gpu1", 0.0)], _var_table())
    assert sum(o.opcode == "dev.launch" for o in p2.ops) == 1
    with pytest.raises(LoweringError):
        lower_hash_batch_varlen("md5", off, [("host", 1.0)], _var_table())
    with pytest.raises(LoweringError):
        lower_hash_batch_varlen("md5", np.array([5, 3]), [("gpu0", 1.0)], _var_table())


@pytest.mark.gpu
@pytest.mark.parametrize("alg", ["sha1", "md5", "sm3"])
def test_varlen_program_on_gpus(alg):
    """Varlen programs across 3 device bindings (one per GPU when present),
    unbatched and with over-capacity groups cut into sub-batches, bit-exact
    against the oracle (itself pinned to the reference's scalar digest)."""
    import oracle
    from paper_2407_09333_b200 import _native
    from paper_2407_09333_b200.runtime import lower_hash_batch_varlen

    nd = _native.device_count()
    off = _var_batch(6000, 2, base=0)
    data = oracle.fill_random(int(off[-1]), 31)
    ref = oracle.batch_varlen(alg, data, off.astype(np.uint64), threads=8).tobytes()
    ords = {i: i % nd for i in range(3)}
    for mem, ratios in ((1 << 30, (0.2, 0.5, 0.3)), (400000, (0.2, 0.5, 0.3)), (150000, (0.0, 1.0, 0.0))):
        devs = _var_table(mem, ordinals=ords)
        prog = lower_hash_batch_varlen(alg, off, [(f"gpu{i}", r) for i, r in enumerate(ratios)], devs)
        inputs = {"msgs": data, "offsets": off}
        if mem == 1 << 30:
            rep = execute(prog, devs, inputs)
            assert rep.outputs["out"] == ref
        rep = execute_batched(prog.format(), devs, inputs, param_names=["msgs", "offsets", "out"])
        assert rep.outputs["out"] == ref, (alg, mem, ratios)
        if mem < (1 << 30):
            assert max(rep.batch_count.values()) > 1, rep.batch_count
        launched = sum(rep.batch_count.values())
        assert launched >= sum(r > 0 for r in ratios)


@pytest.mark.gpu
def test_varlen_program_golden(golden):
    """The reference's scalar digest per message (tests/golden/varlen_batches.json,
    made by tests/golden/make_golden.py from hetoc.crypto.digest) through a
    lowered two-GPU varlen program."""
    import oracle
    from paper_2407_09333_b200 import _native
    from paper_2407_09333_b200.runtime import lower_hash_batch_varlen

    nd = _native.device_count()
    devs = _var_table(1 << 30, k=2, ordinals={0: 0, 1: 1 % nd})
    for row in golden("varlen_batches.json"):
        lens = np.array(row["lens"], np.int64)
        off = np.zeros(len(lens) + 1, np.int64)
        off[1:] = np.cumsum(lens)
        data = oracle.fill_random(int(off[-1]), row["seed"])
        for alg in ("sha1", "md5", "sm3"):
            prog = lower_hash_batch_varlen(alg, off, [("gpu0", 0.4), ("gpu1", 0.6)], devs)
            rep = execute_batched(prog, devs, {"msgs": data, "offsets": off})
            assert hashlib.sha256(rep.outputs["out"]).hexdigest() == row[alg], (alg, len(lens))


def test_sweep_grid_and_records():
    """ratio_grid equals the reference's (sweep.py:39-48); split_ratios puts x
    on the first binding; argmin skips failed points; CSV skips them too."""
    from paper_2407_09333_b200.runtime import RunRecord, ratio_grid, records_to_csv, split_ratios, sweep_argmin

    for step in (0.02, 0.1, 0.25, 0.3, 1.0):
        xs = ratio_grid(step)
        assert xs[0] == 0.0 and xs[-1] == 1.0 and xs == sorted(xs)
    if os.path.isdir(REF_SRC):
        sys.path.insert(0, REF_SRC)
        try:
            from hetoc.scheduler.sweep import ratio_grid as ref_grid
        finally:
            sys.path.remove(REF_SRC)
        for step in (0.02, 0.07, 0.1, 0.25, 0.3, 1.0):
            assert ratio_grid(step) == ref_grid(step)
    for bad in (0.0, -0.1, 1.5):
        with pytest.raises(ValueError):
            ratio_grid(bad)
    assert split_ratios(0.25, 3) == (0.25, 0.375, 0.375)
    with pytest.raises(ValueError):
        split_ratios(0.5, 1)
    recs = [RunRecord((0.0, 1.0), 2.0, {"a": 1.0, "b": 2.0}, {"a": 0, "b": 3}, 10, "md5"),
            RunRecord((0.5, 0.5), 1.0, {"a": 1.0, "b": 1.0}, {"a": 2, "b": 2}, 10, "md5"),
            RunRecord((1.0, 0.0), float("nan"), {}, {}, 10, "md5", error="boom")]
    assert sweep_argmin(recs).ratio_first == 0.5
    csv = records_to_csv(recs).splitlines()
    assert csv[0] == "ratio_first,wall_s,accel_s,batches,n_data,alg" and len(csv) == 3
    assert csv[2] == "0.5,1,1;1,2;2,10,md5"
    with pytest.raises(ValueError):
        sweep_argmin(recs[2:])


@pytest.mark.gpu
def test_sweep_gpu_ratio_grid():
    """The reference's duty-ratio sweep (sweep.py:75-99) over two GPU bindings
    (aliasing GPU 0 on a one-GPU box): every point runs, the extremes put the
    whole batch on one binding, and each point's digests equal the oracle's."""
    import oracle
    from paper_2407_09333_b200 import _native
    from paper_2407_09333_b200.runtime import split_ratios, sweep, sweep_argmin

    n = _native.device_count()
    w = Workload("md5", 30011, 9)
    host = DeviceSpec("host", kind="host", threads=os.cpu_count() or 1)
    devs = DeviceTable(host, tuple(DeviceSpec(f"gpu{i}", ordinal=i % n, mem_bytes=1 << 20) for i in range(2)))
    recs = sweep(w, devs, step=0.25)
    assert [r.ratio_first for r in recs] == [0.0, 0.25, 0.5, 0.75, 1.0]
    assert all(r.error is None and r.wall_s > 0 for r in recs)
    assert recs[0].batches["gpu0"] == 0 and recs[-1].batches["gpu1"] == 0
    best = sweep_argmin(recs)
    ref = oracle.batch_fixed("md5", gen_messages(0, w.count, w.width).as_array(), threads=8).tobytes()
    assert run_point(w, devs, split_ratios(best.ratio_first, 2), keep_digests=True).digests == ref
