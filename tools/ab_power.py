"""Sustained-load A/B of fixed-width kernel arms (configs[1] shape by default):
each arm runs STEPS back-to-back launches per round (long enough for the
board to settle at its power limit), interleaved rounds, with NVML SM clock
and power sampled during every arm; digests cross-checked between arms.
Prints the board's power limits first.

usage: AB_ARMS='{"base": {}, "v0": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "0"}}' \\
       HETOC_B200_LIB=libhetoc_b200_ab.so python tools/ab_power.py md5 [n] [L]
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
arms = json.loads(os.environ.get("AB_ARMS", '{"base": {}}'))
rounds = int(os.environ.get("AB_ROUNDS", 3))
steps = int(os.environ.get("AB_STEPS", 60))
keys = sorted({k for env in arms.values() for k in env})

import pynvml  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
lim = {}
for name, fn in (("limit_w", pynvml.nvmlDeviceGetPowerManagementLimit),
                 ("default_limit_w", pynvml.nvmlDeviceGetPowerManagementDefaultLimit),
                 ("enforced_limit_w", pynvml.nvmlDeviceGetEnforcedPowerLimit)):
    try:
        lim[name] = fn(h) / 1000.0
    except Exception as e:  # noqa: BLE001
        lim[name] = str(e)
try:
    lo, hi = pynvml.nvmlDeviceGetPowerManagementLimitConstraints(h)
    lim["constraints_w"] = [lo / 1000.0, hi / 1000.0]
except Exception:
    pass
print(json.dumps({"power": lim}), flush=True)

samples = []
stop = threading.Event()


def sampler():
    while not stop.wait(0.02):
        try:
            samples.append((time.perf_counter(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
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
res = {a: {"ms": [], "mhz": [], "w": []} for a in arms}
names = {}
for _ in range(rounds):
    for name, env in arms.items():
        set_arm(env)
        device.hash_fixed(alg, msgs, out=out)
        torch.cuda.synchronize()
        names[name] = _native.last_kernel_name().split("(")[0]
        if ref is None:
            ref = out.clone()
        assert torch.equal(out, ref), name
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        s.record()
        for _ in range(steps):
            device.hash_fixed(alg, msgs, out=out)
        e.record()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        res[name]["ms"].append(s.elapsed_time(e) / steps)
        win = [x for x in samples if t0 + 0.3 * (t1 - t0) <= x[0] <= t1]  # settled part of the arm
        if win:
            res[name]["mhz"].append(statistics.median(x[1] for x in win))
            res[name]["w"].append(statistics.median(x[2] for x in win))
stop.set()
set_arm({})
for name, r in res.items():
    ms = statistics.median(r["ms"])
    print(json.dumps({"alg": alg, "n": n, "L": L, "arm": name, "ms_median": round(ms, 4), "ms_min": round(min(r["ms"]), 4),
                      "GBps": round(n * L / ms / 1e6, 1), "sm_mhz": statistics.median(r["mhz"]) if r["mhz"] else None,
                      "power_w": round(statistics.median(r["w"]), 1) if r["w"] else None, "kernel": names[name]}),
          flush=True)
