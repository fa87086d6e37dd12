"""Kernel time vs batch size at a fixed message length, in warps per SM
sub-partition (148 SMs x 4 SMSPs = 592 schedulers): where a batch stops being
bound by one message's dependent chain and starts being bound by throughput,
and what the 3.46-warps-per-scheduler shape of a 65,536-message batch costs.
Each point: CUDA graph of 10 passes over 10 copies, L2 flushed before each
replay ("cold", every pass reads HBM) and not flushed ("hot").

usage: SCAN='md5:1024,sha1:64' python tools/ab_scan.py
"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_09333_b200 import _native, device  # noqa: E402

DLEN = {"md5": 16, "sha1": 20, "sm3": 32}
WARPS = [float(x) for x in os.environ.get("SCAN_WARPS", "1,2,3,3.46,4,5,6,8,12,16").split(",")]
flush = torch.empty(2 * 126 * 10**6, dtype=torch.uint8, device="cuda:0")
for item in os.environ.get("SCAN", "md5:1024").split(","):
    alg, L = item.split(":")
    L = int(L)
    for wps in WARPS:
        n = int(round(wps * 592 * 32))
        buf = torch.empty(n * L, dtype=torch.uint8, device="cuda:0")
        device.fill_random(buf, 3)
        copies = [buf.view(n, L)] + [buf.view(n, L).clone() for _ in range(9)]
        out = torch.empty((n, DLEN[alg]), dtype=torch.uint8, device="cuda:0")
        g = device.FixedHashGraph(alg, copies, out)
        kern = _native.last_kernel_name().split("(")[0]
        res = {}
        for mode in ("cold", "hot"):
            ts = []
            for _ in range(7):
                if mode == "cold":
                    flush.fill_(1)
                else:
                    g.replay()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                g.replay()
                e.record()
                torch.cuda.synchronize()
                ts.append(s.elapsed_time(e) / 10 * 1e3)
            res[mode] = round(statistics.median(ts), 2)
        print(json.dumps({"alg": alg, "L": L, "warps_per_smsp": wps, "n": n, "us_cold": res["cold"],
                          "us_hot": res["hot"], "GBps_cold": round(n * L / res["cold"] / 1e3, 1), "kernel": kern}),
              flush=True)
        del buf, copies, g
        torch.cuda.empty_cache()
