"""A/B the pipe-balancing variants of k_fixed_tma on the GPU (kernel-only).

For each algorithm: 2^24 x 1 KiB messages resident in HBM, HB_VARIANT=0..3,
CUDA-event timing on the launching stream; every variant's digests must equal
variant 0's bit for bit.  Prints one JSON line per (alg, variant).
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_09333_b200 import device  # noqa: E402

n = int(os.environ.get("SWEEP_N", 1 << 24))
L = int(os.environ.get("SWEEP_L", 1024))
steps = 20
buf = torch.empty(n * L, dtype=torch.uint8, device="cuda:0")
device.fill_random(buf, 2)
msgs = buf.view(n, L)
blocks = n * ((L + 8) // 64 + 1)
combos = [(c, v) for c in os.environ.get("SWEEP_CFGS", "1x3,ws2,ws3").split(",") for v in os.environ.get("SWEEP_VARS", "01").split(",")[0]]
for alg in sys.argv[1:] or ["md5", "sha1", "sm3"]:
    ref = None
    for cfg, v in combos:
        os.environ["HB_VARIANT"] = v
        os.environ["HB_TMA_CFG"] = cfg
        out = device.hash_fixed(alg, msgs)
        for _ in range(3):
            device.hash_fixed(alg, msgs, out=out)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(steps):
            device.hash_fixed(alg, msgs, out=out)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / steps
        if ref is None:
            ref = out.clone()
        same = bool(torch.equal(out, ref))
        print(json.dumps({"alg": alg, "cfg": cfg, "variant": int(v), "ms": round(ms, 4), "GBps": round(n * L / ms / 1e6, 1),
                          "ns_per_block_per_sm": round(ms * 1e6 * 148 / blocks, 4), "same_as_v0": same}), flush=True)
