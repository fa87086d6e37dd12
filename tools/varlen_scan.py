"""Per-block cost of the varlen kernel against message length: batches of
equal-length messages (an odd length L puts consecutive messages at every
byte alignment), ~4 GiB each, sort + hash timed with
CUDA events.  A per-message overhead (the perm -> offsets -> data load chain
at a thread's start, the 1-2 finishing blocks) shows up as a rising cost per
64-byte block at short lengths.

usage: python tools/varlen_scan.py md5 [L ...]     (HB_* env selects arms)
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_09333_b200 import _native, device  # noqa: E402

DLEN = {"md5": 16, "sha1": 20, "sm3": 32}
alg = sys.argv[1] if len(sys.argv) > 1 else "md5"
lens = [int(x) for x in sys.argv[2:]] or [63, 191, 511, 1023, 2047, 4095, 16383]
for L in lens:
    n = min((4 << 30) // L, 1 << 24)
    off = np.arange(n + 1, dtype=np.int64) * L  # equal lengths; an odd L cycles through every alignment
    data = torch.empty(n * L, dtype=torch.uint8, device="cuda:0")
    device.fill_random(data, 3)
    d_off = torch.from_numpy(off).cuda()
    out = torch.empty((n, DLEN[alg]), dtype=torch.uint8, device="cuda:0")
    scratch = torch.empty(int(_native.lib().hb_varlen_scratch_bytes(n)), dtype=torch.uint8, device="cuda:0")
    f = lambda: device.hash_varlen(alg, data, d_off, out=out, scratch=scratch, offset_base=0)  # noqa: E731
    f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        f()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    blocks = n * ((L + 8) // 64 + 1)
    print(json.dumps({"alg": alg, "L": L, "n": n, "ms": round(ms, 4), "GBps": round(n * L / ms / 1e6, 1),
                      "ns_per_block_per_sm": round(ms * 1e6 * 148 / blocks, 3),
                      "kernel": _native.last_kernel_name().split("(")[0]}), flush=True)
    del data, d_off, out, scratch
    torch.cuda.empty_cache()
