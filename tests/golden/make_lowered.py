"""Golden lowered programs, made by running the REFERENCE's compiler and
simulated runtime (authoring container only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_lowered.py

For each case: ``crypto.hash_batch`` over the paper workload
(``gen_messages(0, count, width)``) is built as ``scheduler/workload.py``'s
``build_hash_module`` does (any number of device bindings), lowered with
``run_pipeline`` and printed with ``print_module``; the reference's own
``execute_batched`` then runs it against simulated accelerators with the same
capacities.  Stored: the printed program, the SHA-256 of the reference's
``out`` buffer, its per-device batch counts and bytes copied.  The B200 runtime
must reproduce the text (``runtime.lowering``), parse it, and -- on a GPU --
produce the same bytes and batch counts (``tests/test_runtime.py``).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from hetoc.crypto.batch import DIGEST_LEN, gen_messages  # noqa: E402
from hetoc.hir.core import Buffer, DeviceBinding, FuncBuilder, HirModule  # noqa: E402
from hetoc.hir.printer import print_module  # noqa: E402
from hetoc.passes.pipeline import run_pipeline  # noqa: E402
from hetoc.runtime.devices import DeviceSpec, DeviceTable  # noqa: E402
from hetoc.runtime.executor import execute_batched  # noqa: E402

# name, alg, count, width, bindings [(id, ratio)], device capacities {id: mem_bytes}, host sha_accel, accel sha ids
CASES = [
    ("md5_one_gpu", "md5", 1000, 9, [("gpu0", 1.0)], {"gpu0": 1 << 30}, False, ()),
    ("sm3_two_gpus_batched", "sm3", 1000, 9, [("gpu0", 0.3), ("gpu1", 0.7)], {"gpu0": 5000, "gpu1": 1 << 20},
     False, ()),
    ("sha1_many_batches_accel", "sha1", 5000, 9, [("gpu0", 1.0)], {"gpu0": 20000}, True, ("gpu0",)),
    ("md5_three_gpus_w64", "md5", 777, 64, [("gpu0", 0.25), ("gpu1", 0.25), ("gpu2", 0.5)],
     {"gpu0": 1 << 20, "gpu1": 9000, "gpu2": 1 << 20}, False, ()),
    ("sha1_zero_share", "sha1", 300, 12, [("gpu0", 0.0), ("gpu1", 1.0)], {"gpu0": 1 << 20, "gpu1": 1 << 20},
     True, ()),
    ("sm3_tiny_split", "sm3", 3, 9, [("gpu0", 0.5), ("gpu1", 0.5)], {"gpu0": 1 << 20, "gpu1": 1 << 20}, False, ()),
    ("sha1_uneven_ratios_w20", "sha1", 4099, 20, [("gpu0", 0.37), ("gpu1", 0.63)],
     {"gpu0": 50000, "gpu1": 77777}, False, ()),
    ("md5_host_share", "md5", 200, 9, [("host", 0.5), ("gpu0", 0.5)], {"gpu0": 1 << 20}, False, ()),
]


def build(alg, count, width, bindings):
    b = FuncBuilder("main", [Buffer("i8", count * width), Buffer("i8", count * DIGEST_LEN[alg])])
    b.func.param_names = ["msgs", "out"]
    msgs, out = b.func.params
    b.op("crypto.hash_batch", [msgs, out],
         attrs={"alg": alg, "count": count, "msg_len": width, "shared": False,
                "devices": [DeviceBinding(d, r) for d, r in bindings]})
    return HirModule([b.build()])


def main():
    cases = []
    for name, alg, count, width, bindings, mems, host_sha, accel_sha in CASES:
        host = DeviceSpec("host", kind="host", threads=4, sha_accel=host_sha)
        accels = tuple(DeviceSpec(d, threads=1, mem_bytes=m, sha_accel=d in accel_sha) for d, m in mems.items())
        devs = DeviceTable(host, accels)
        low = run_pipeline(build(alg, count, width, bindings), devices=devs)
        text = print_module(low)
        rep = execute_batched(low, devs, {"msgs": gen_messages(0, count, width).data})
        cases.append({"name": name, "alg": alg, "count": count, "width": width,
                      "bindings": [[d, r] for d, r in bindings], "mem_bytes": mems, "host_sha_accel": host_sha,
                      "accel_sha": list(accel_sha), "text": text,
                      "out_sha256": hashlib.sha256(rep.outputs["out"]).hexdigest(),
                      "batch_count": rep.batch_count, "bytes_copied": rep.bytes_copied})
        print(name, rep.batch_count)
    with open(os.path.join(HERE, "lowered.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_lowered.py (reference run_pipeline + execute_batched)",
                   "cases": cases}, f, indent=1)


if __name__ == "__main__":
    main()
