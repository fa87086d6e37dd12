"""A/B of the kernel shapes at small messages / small batches (kernel-only,
interleaved rounds, bit-exact cross-check): default dispatch, the direct
per-thread-load kernel (HB_FLAG_NO_TMA), and the 4-warp tiles forced
(HB_SMALL_N=0).  Prints one JSON line per (alg, n, L, arm)."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_09333_b200 import _native, device  # noqa: E402

DLEN = {"md5": 16, "sha1": 20, "sm3": 32}
POINTS = [(1 << 24, 16), (1 << 24, 32), (1 << 24, 64), (1 << 24, 128)] if os.environ.get("AB_SHORT_ONLY") else \
    [(1 << 24, 16), (1 << 24, 32), (1 << 24, 64), (1 << 24, 128), (1 << 22, 256),
     (1 << 16, 1024), (1 << 16, 65536), (1 << 12, 65536), (1 << 14, 16384), (1 << 17, 4096)]
ARMS = {"default": ({}, 0), "const_v1": ({"HB_CONST_VARIANT": "1"}, 0), "direct": ({"HB_NO_SMALL_KERNEL": "1"}, _native.HB_FLAG_NO_TMA), "ws_forced": ({"HB_SMALL_N": "0", "HB_DIRECT_MAX_L": "0"}, 0),
        "small_forced": ({"HB_SMALL_N": str(1 << 40), "HB_DIRECT_MAX_L": "0"}, 0)}
if os.environ.get("AB_ARMS"):  # {name: {env}} (flags 0)
    ARMS = {k: (v, 0) for k, v in json.loads(os.environ["AB_ARMS"]).items()}
if os.environ.get("AB_POINTS"):  # n:L,n:L,...
    POINTS = [tuple(int(x) for x in p.split(":")) for p in os.environ["AB_POINTS"].split(",")]
KEYS = sorted({k for env, _ in ARMS.values() for k in env} | {"HB_SMALL_N", "HB_DIRECT_MAX_L", "HB_NO_SMALL_KERNEL",
                                                              "HB_CONST_VARIANT"})
rounds = int(os.environ.get("AB_ROUNDS", 3))
for n, L in POINTS:
    buf = torch.empty(n * L, dtype=torch.uint8, device="cuda:0")
    device.fill_random(buf, 7)
    msgs = buf.view(n, L)
    steps = max(3, min(50, int(2e9 // (n * L))))
    for alg in sys.argv[1:] or ["md5", "sha1", "sm3"]:
        ref, times = None, {}
        for _ in range(rounds):
            for arm, (env, flags) in ARMS.items():
                for k in KEYS:
                    os.environ.pop(k, None)
                os.environ.update(env)
                _native.reload_tuning()  # the library parses $HB_* once
                out = torch.empty((n, DLEN[alg]), dtype=torch.uint8, device="cuda:0")
                device.hash_fixed(alg, msgs, out=out, flags=flags)
                torch.cuda.synchronize()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                for _ in range(steps):
                    device.hash_fixed(alg, msgs, out=out, flags=flags)
                e.record()
                torch.cuda.synchronize()
                if ref is None:
                    ref = out.clone()
                assert torch.equal(out, ref), (alg, n, L, arm)
                times.setdefault(arm, []).append(s.elapsed_time(e) / steps)
        for k in ("HB_SMALL_N", "HB_DIRECT_MAX_L", "HB_NO_SMALL_KERNEL", "HB_CONST_VARIANT"):
            os.environ.pop(k, None)
        for arm, ts in times.items():
            ms = statistics.median(ts)
            print(json.dumps({"alg": alg, "n": n, "L": L, "arm": arm, "ms": round(ms, 5),
                              "GBps": round(n * L / ms / 1e6, 1)}), flush=True)
    del buf, msgs
    torch.cuda.empty_cache()
