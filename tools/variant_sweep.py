"""A/B the TMA tile configurations x pipe-balancing variants of k_fixed_tma on
the GPU (kernel-only).

For each algorithm: 2^24 x 1 KiB messages resident in HBM; every (cfg,
variant) combination is timed with CUDA events in ROUNDS interleaved rounds
(so clock drift hits all equally); digests of every combination must equal the
first one's bit for bit.  nvidia-smi clocks are sampled throughout.  Prints one
JSON line per (alg, cfg, variant) with the median and min ms.

env: SWEEP_CFGS (default "1x3,1x2,ws2,ws3"), SWEEP_VARS ("01"), SWEEP_ROUNDS (3)
"""
import json
import os
import statistics
import subprocess
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_09333_b200 import device  # noqa: E402

n = int(os.environ.get("SWEEP_N", 1 << 24))
L = int(os.environ.get("SWEEP_L", 1024))
steps = int(os.environ.get("SWEEP_STEPS", 10))
rounds = int(os.environ.get("SWEEP_ROUNDS", 3))
cfgs = os.environ.get("SWEEP_CFGS", "1x3,1x2,ws2,ws3").split(",")
vars_ = list(os.environ.get("SWEEP_VARS", "01"))
buf = torch.empty(n * L, dtype=torch.uint8, device="cuda:0")
device.fill_random(buf, 2)
msgs = buf.view(n, L)
blocks = n * ((L + 8) // 64 + 1)
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                        "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
for alg in sys.argv[1:] or ["md5", "sha1", "sm3"]:
    ref = None
    times = {}
    for _ in range(rounds):
        for cfg in cfgs:
            for v in vars_:
                os.environ["HB_VARIANT"] = v
                os.environ["HB_TMA_CFG"] = cfg
                out = torch.empty((n, {"md5": 16, "sha1": 20, "sm3": 32}[alg]), dtype=torch.uint8, device="cuda:0")
                for _ in range(2):
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
                assert torch.equal(out, ref), (alg, cfg, v)
                times.setdefault((cfg, v), []).append(s.elapsed_time(e) / steps)
    for (cfg, v), ts in times.items():
        ms = statistics.median(ts)
        print(json.dumps({"alg": alg, "cfg": cfg, "variant": int(v), "ms_median": round(ms, 4),
                          "ms_min": round(min(ts), 4), "GBps": round(n * L / ms / 1e6, 1),
                          "ns_per_block_per_sm": round(ms * 1e6 * 148 / blocks, 4)}), flush=True)
smi.terminate()
clk = [ln.split(",") for ln in smi.stdout.read().strip().splitlines()]
sm = [float(c[0]) for c in clk if len(c) >= 3]
print(json.dumps({"clock_mhz_median": statistics.median(sm) if sm else None, "clock_mhz_min": min(sm) if sm else None,
                  "power_w_max": max(float(c[1]) for c in clk if len(c) >= 3) if sm else None,
                  "reasons": sorted({c[2].strip() for c in clk if len(c) >= 3})}), flush=True)
