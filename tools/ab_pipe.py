"""A/B of the host-buffer engine's chunk pipelining ($HB_PIPE_CHUNKS: a shard
is cut into at least this many chunks of >= $HB_MIN_CHUNK_BYTES so H2D,
kernel and D2H of consecutive chunks overlap).  End to end through the public
API with pinned host input and output, interleaved rounds, digests compared
across arms."""
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_09333_b200 import crypto  # noqa: E402

DLEN = {"md5": 16, "sha1": 20, "sm3": 32}
# arm "P" or "P@M": HB_PIPE_CHUNKS=P, HB_MIN_CHUNK_BYTES=M MiB and no digest-size threshold
# (engine defaults otherwise)
ARMS = os.environ.get("AB_ARMS", "1,4@1,4@4,4@8,4@16").split(",")
CASES = [("sha1", 65536, 64), ("sha1", 1 << 17, 64), ("sha1", 1 << 18, 64), ("sha1", 1 << 19, 64),
         ("sha1", 1 << 20, 64), ("sm3", 1 << 19, 64), ("md5", 1 << 16, 1024), ("md5", 1 << 20, 1024)]
if os.environ.get("AB_CASES") == "small":
    CASES = [("sha1", 16384, 64), ("sha1", 65536, 64), ("md5", 65536, 64), ("sha1", 1 << 17, 64), ("md5", 4096, 1024)]


def pinned(shape):
    return torch.empty(shape, dtype=torch.uint8, pin_memory=True).numpy()


for alg, n, L in CASES:
    src = pinned((n, L))
    src[:] = np.random.default_rng(n + L).integers(0, 256, (n, L), dtype=np.uint8)
    out = pinned((n, DLEN[alg]))
    ref, times = None, {}
    reps = max(3, min(50, int(2e8 // (n * L))))
    for _ in range(3):
        for arm in ARMS:
            os.environ["HB_PIPE_CHUNKS"] = arm.split("@")[0]
            os.environ.pop("HB_MIN_CHUNK_BYTES", None)
            os.environ.pop("HB_PIPE_MIN_OUT", None)
            if "@" in arm:  # explicit floor: split regardless of the digest-size threshold
                os.environ["HB_MIN_CHUNK_BYTES"] = str(int(float(arm.split("@")[1]) * (1 << 20)))
                os.environ["HB_PIPE_MIN_OUT"] = "1"
            crypto.batch_digest(alg, src, out=out)
            t0 = time.perf_counter()
            for _ in range(reps):
                crypto.batch_digest(alg, src, out=out)
            dt = (time.perf_counter() - t0) / reps
            if ref is None:
                ref = out.copy()
            assert np.array_equal(out, ref), (alg, n, L, arm)
            times.setdefault(arm, []).append(dt)
    for arm, ts in times.items():
        ms = statistics.median(ts) * 1e3
        print(json.dumps({"alg": alg, "n": n, "L": L, "arm": arm, "ms": round(ms, 4),
                          "GBps": round(n * L / ms / 1e6, 2)}), flush=True)
