"""Generic A/B of environment knobs on a fixed-width batch (kernel-only,
interleaved rounds, digests cross-checked against the first arm).

usage: AB_ARMS='{"base": {}, "x": {"HB_TMA_L2": "128"}}' python tools/ab_env.py md5 [n] [L] [steps]
"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_09333_b200 import device  # noqa: E402

alg = sys.argv[1] if len(sys.argv) > 1 else "md5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 24
L = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
arms = json.loads(os.environ.get("AB_ARMS", '{"base": {}}'))
keys = sorted({k for env in arms.values() for k in env})
buf = torch.empty(n * L, dtype=torch.uint8, device="cuda:0")
device.fill_random(buf, 2)
msgs = buf.view(n, L)
out = torch.empty((n, {"md5": 16, "sha1": 20, "sm3": 32}[alg]), dtype=torch.uint8, device="cuda:0")
ref, times = None, {}
for _ in range(int(os.environ.get("AB_ROUNDS", 3))):
    for name, env in arms.items():
        for k in keys:
            os.environ.pop(k, None)
        os.environ.update(env)
        device.hash_fixed(alg, msgs, out=out)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(steps):
            device.hash_fixed(alg, msgs, out=out)
        e.record()
        torch.cuda.synchronize()
        if ref is None:
            ref = out.clone()
        assert torch.equal(out, ref), name
        times.setdefault(name, []).append(s.elapsed_time(e) / steps)
for name, ts in times.items():
    ms = statistics.median(ts)
    print(json.dumps({"alg": alg, "n": n, "L": L, "arm": name, "ms_median": round(ms, 4), "ms_min": round(min(ts), 4),
                      "GBps": round(n * L / ms / 1e6, 1)}), flush=True)
