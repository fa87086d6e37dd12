"""A/B of tuning knobs on fixed-width batches measured the way the configs[4]
sweep measures them: a CUDA graph of 10 passes over 10 identical copies (every
pass reads HBM), the L2 flushed before each replay, interleaved rounds; digests
of every arm cross-checked against the first arm's.

usage: AB_ARMS='{"base": {}, "nopdl": {"HB_PDL": "0"}}' \
       AB_POINTS='md5:65536:1024,sha1:65536:256' python tools/ab_mid.py
(use HETOC_B200_LIB=libhetoc_b200_ab.so for the A/B-only knobs)
"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_09333_b200 import _native, device  # noqa: E402

DLEN = {"md5": 16, "sha1": 20, "sm3": 32}
arms = json.loads(os.environ.get("AB_ARMS", '{"base": {}}'))
points = [p.split(":") for p in os.environ.get("AB_POINTS", "md5:65536:1024").split(",")]
rounds = int(os.environ.get("AB_ROUNDS", 3))
keys = sorted({k for env in arms.values() for k in env})
flush = torch.empty(2 * 126 * 10**6, dtype=torch.uint8, device="cuda:0")


def set_arm(env):
    for k in keys:
        os.environ.pop(k, None)
    os.environ.update(env)
    _native.reload_tuning()


for alg, n, L in points:
    n, L = int(n), int(L)
    buf = torch.empty(n * L, dtype=torch.uint8, device="cuda:0")
    device.fill_random(buf, 7)
    copies = [buf.view(n, L)] + [buf.view(n, L).clone() for _ in range(9)]
    out = torch.empty((n, DLEN[alg]), dtype=torch.uint8, device="cuda:0")
    graphs, names = {}, {}
    for name, env in arms.items():
        set_arm(env)
        graphs[name] = device.FixedHashGraph(alg, copies, out)
        device.hash_fixed(alg, copies[0], out=out)
        names[name] = _native.last_kernel_name().split("(")[0]
    ref, times = None, {}
    for _ in range(rounds):
        for name, g in graphs.items():
            g.replay()
            torch.cuda.synchronize()
            if ref is None:
                ref = out.clone()
            assert torch.equal(out, ref), name
            ts = []
            for _ in range(5):
                flush.fill_(1)
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                g.replay()
                e.record()
                torch.cuda.synchronize()
                ts.append(s.elapsed_time(e) / 10)
            times.setdefault(name, []).extend(ts)
    for name, ts in times.items():
        ms = statistics.median(ts)
        print(json.dumps({"alg": alg, "n": n, "L": L, "arm": name, "us_median": round(ms * 1e3, 2),
                          "us_min": round(min(ts) * 1e3, 2), "GBps": round(n * L / ms / 1e6, 1),
                          "kernel": names[name]}), flush=True)
    del buf, copies, graphs
    torch.cuda.empty_cache()
set_arm({})
