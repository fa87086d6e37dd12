"""A/B of the in-kernel decimal workload (paper: 10^9 x 9 digits) across round
variants ($HB_CONST_VARIANT) and kernels ($HB_DEC_RUN: runs of ten vs one
message per thread), kernel-only, digests cross-checked.  Arms: $AB_ARMS."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_09333_b200 import _native, device  # noqa: E402

n = int(os.environ.get("AB_N", 10**9))
for alg in sys.argv[1:] or ["md5", "sha1", "sm3"]:
    out = torch.empty((n, {"md5": 16, "sha1": 20, "sm3": 32}[alg]), dtype=torch.uint8, device="cuda:0")
    ref, times = None, {}
    for _ in range(3):
        for arm in os.environ.get("AB_ARMS", "v1_fma_digits,v3_fma_digits,v1_run,v3_run").split(","):
            os.environ["HB_CONST_VARIANT"] = arm[1:].split("_")[0]
            os.environ["HB_FMA_DIGITS"] = "1" if "fma" in arm or "run" in arm else "0"
            os.environ["HB_DEC_RUN"] = "1" if "run" in arm else "0"
            _native.reload_tuning()  # the library parses $HB_* once
            device.hash_decimal(alg, 0, n, 9, out=out)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(3):
                device.hash_decimal(alg, 0, n, 9, out=out)
            e.record()
            torch.cuda.synchronize()
            h = out[:: 997].clone()
            if ref is None:
                ref = h
            assert torch.equal(h, ref), (alg, arm)
            times.setdefault(arm, []).append(s.elapsed_time(e) / 3)
    for arm, ts in times.items():
        ms = statistics.median(ts)
        print(json.dumps({"alg": alg, "arm": arm, "ms": round(ms, 3), "Mhash_s": round(n / ms / 1e3, 1)}), flush=True)
    del out
    torch.cuda.empty_cache()
