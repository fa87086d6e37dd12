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
