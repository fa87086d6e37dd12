"""Interleaved A/B of fixed-width arms measured the way bench.py times its
headline: per round and arm, an idle cool-down (AB_COOL s, so every arm starts
from the same power state), W warm-up launches, then K timed launches
bracketed by CUDA events, with HB_FLAG_INPUT_READY as the bench passes it;
NVML SM clock sampled during the timed launches.  Digests cross-checked.

usage: AB_ARMS='{"dflt": {}, "old": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "1"}}' \\
       HETOC_B200_LIB=libhetoc_b200_ab.so python tools/ab_headline.py md5 [n] [L]
"""
import json
import os
import statistics
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_09333_b200 import _native, device  # noqa: E402

alg = sys.argv[1] if len(sys.argv) > 1 else "md5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 24
L = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
arms = json.loads(os.environ.get("AB_ARMS", '{"dflt": {}}'))
rounds = int(os.environ.get("AB_ROUNDS", 4))
warm, steps = int(os.environ.get("AB_WARMUP", 5)), int(os.environ.get("AB_STEPS", 20))
cool = float(os.environ.get("AB_COOL", 3))
flags = 0 if os.environ.get("AB_FLAGS") == "none" else _native.HB_FLAG_INPUT_READY
keys = sorted({k for env in arms.values() for k in env})

import pynvml  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples = []
stop = threading.Event()


def sampler():
    while not stop.wait(0.01):
        try:
            samples.append((time.perf_counter(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
        except Exception:
            pass


threading.Thread(target=sampler, daemon=True).start()


def set_arm(env):
    for k in keys:
        os.environ.pop(k, None)
    os.environ.update(env)
    _native.reload_tuning()


buf = torch.empty(n * L, dtype=torch.uint8, device="cuda:0")
device.fill_random(buf, 2)
msgs = buf.view(n, L)
out = torch.empty((n, {"md5": 16, "sha1": 20, "sm3": 32}[alg]), dtype=torch.uint8, device="cuda:0")
ref = None
res = {a: {"ms": [], "mhz": []} for a in arms}
names = {}
for _ in range(rounds):
    for name, env in arms.items():
        set_arm(env)
        torch.cuda.synchronize()
        time.sleep(cool)
        for _ in range(warm):
            device.hash_fixed(alg, msgs, out=out, flags=flags)
        torch.cuda.synchronize()
        names[name] = _native.last_kernel_name().split("(")[0]
        if ref is None:
            ref = out.clone()
        assert torch.equal(out, ref), name
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        s.record()
        for _ in range(steps):
            device.hash_fixed(alg, msgs, out=out, flags=flags)
        e.record()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        res[name]["ms"].append(s.elapsed_time(e) / steps)
        win = [x[1] for x in samples if t0 <= x[0] <= t1]
        if win:
            res[name]["mhz"].append(statistics.median(win))
stop.set()
set_arm({})
for name, r in res.items():
    ms = statistics.median(r["ms"])
    print(json.dumps({"alg": alg, "n": n, "L": L, "arm": name, "ms_median": round(ms, 4), "ms_min": round(min(r["ms"]), 4),
                      "ms_all": [round(x, 4) for x in r["ms"]], "GBps": round(n * L / ms / 1e6, 1),
                      "sm_mhz": r["mhz"], "kernel": names[name]}), flush=True)
