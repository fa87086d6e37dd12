"""Small-batch latency: the chunk ring (H2D copy -> kernel -> D2H copy) against
the zero-copy path (the kernel reads the batch from mapped pinned host memory
and stores digests there; hb_engine.cu small_batch), both through
hb_hash_fixed / hb_hash_varlen with pageable numpy buffers (the reference call
shape), untimed, one GPU.  Median per-call wall time of K calls, us; the
crossover sets the default $HB_ZERO_COPY_MAX.

usage: python tools/zero_copy_probe.py [alg n L] ...
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_09333_b200 import _native  # noqa: E402
from paper_2407_09333_b200.crypto import batch_digest, batch_digest_varlen  # noqa: E402

args = sys.argv[1:]
cases = [(args[i], int(args[i + 1]), int(args[i + 2])) for i in range(0, len(args), 3)] or [
    ("md5", 1, 64), ("md5", 64, 64), ("md5", 64, 1024), ("sha1", 1024, 64), ("md5", 256, 1024), ("sm3", 4096, 32),
    ("md5", 2048, 64), ("md5", 128, 1024), ("md5", 4096, 64), ("md5", 512, 1024), ("md5", 16384, 16),
    ("md5", 2048, 256), ("md5", 1024, 1024), ("sha1", 65536, 64)]
ARMS = {"ring": "0", "zc": str(16 << 20)}


def med(f, k):
    for _ in range(5):
        f()
    ts = []
    for _ in range(k):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    return ts[k // 2] * 1e6


for alg, n, L in cases:
    data = np.random.default_rng(n + L).integers(0, 256, (n, L), dtype=np.uint8)
    off = np.arange(n + 1, dtype=np.uint64) * L
    res = {"alg": alg, "n": n, "L": L, "KiB": round(n * L / 1024, 1)}
    outs = {}
    for arm, v in ARMS.items():
        os.environ["HB_ZERO_COPY_MAX"] = v
        _native.reload_tuning()
        k = 300 if n * L <= (256 << 10) else 60
        res[arm + "_us"] = round(med(lambda: batch_digest(alg, data), k), 1)
        res[arm + "_varlen_us"] = round(med(lambda: batch_digest_varlen(alg, data.reshape(-1), off), k), 1)
        outs[arm] = batch_digest(alg, data)
        res[arm + "_kernel"] = _native.last_kernel_name().split("(")[0].replace("void hb::", "")
    assert np.array_equal(outs["ring"], outs["zc"])
    print(json.dumps(res), flush=True)
os.environ.pop("HB_ZERO_COPY_MAX")
