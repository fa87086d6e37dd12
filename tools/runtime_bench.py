"""The runtime for lowered hyper programs at scale: crypto.hash_batch over the
paper workload (gen_messages, 9 digits) lowered onto the GPU(s) and executed
with capacity sub-batching; device-measured time vs the direct engine call.

usage: python tools/runtime_bench.py [alg] [count]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_09333_b200 import _native  # noqa: E402
from paper_2407_09333_b200.crypto import batch_digest, gen_messages  # noqa: E402
from paper_2407_09333_b200.runtime import DeviceSpec, DeviceTable, Workload, run_point  # noqa: E402

alg = sys.argv[1] if len(sys.argv) > 1 else "sha1"
count = int(sys.argv[2]) if len(sys.argv) > 2 else 20_000_000
w = Workload(alg, count, 9)
msgs = w.message_bytes()
ref = batch_digest(alg, np.frombuffer(msgs, np.uint8).reshape(count, 9))
t0 = time.perf_counter()
batch_digest(alg, np.frombuffer(msgs, np.uint8).reshape(count, 9))
direct_s = time.perf_counter() - t0
ng = _native.device_count()
host = DeviceSpec("host", kind="host", threads=os.cpu_count() or 1)
for cap in (1 << 40, 64 << 20):  # one launch group vs sub-batches of <= 64 MiB
    devs = DeviceTable(host, tuple(DeviceSpec(f"gpu{i}", ordinal=i % ng, mem_bytes=cap) for i in range(max(1, ng))))
    run_point(w, devs, message_bytes=msgs)  # warm
    t0 = time.perf_counter()
    r = run_point(w, devs, message_bytes=msgs, keep_digests=True)
    wall = time.perf_counter() - t0
    ok = r.digests == ref.tobytes()
    print(json.dumps({"alg": alg, "count": count, "cap_bytes": cap, "batches": r.batches, "device_wall_s": round(r.wall_s, 4),
                      "host_wall_s": round(wall, 3), "direct_engine_s": round(direct_s, 3),
                      "msgs_per_s_device": round(count / r.wall_s / 1e6, 1), "bit_exact": ok}), flush=True)

# breakdown of the sub-batched run: device kernel / copy time vs span
from paper_2407_09333_b200.runtime import execute_batched, lower_hash_batch  # noqa: E402

devs = DeviceTable(host, (DeviceSpec("gpu0", ordinal=0, mem_bytes=64 << 20),))
prog = lower_hash_batch(alg, count, 9, [("gpu0", 1.0)], devs)
t0 = time.perf_counter()
rep = execute_batched(prog, devs, {"msgs": msgs})
print(json.dumps({"span_s": round(rep.wall_time["gpu0"], 4), "kernels_s": round(rep.compute_s["gpu0"], 4),
                  "copies_s": round(rep.charge_s["gpu0"], 4), "host_s": round(time.perf_counter() - t0, 3),
                  "batches": rep.batch_count["gpu0"]}), flush=True)
