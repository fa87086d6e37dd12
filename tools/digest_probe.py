"""Per-call latency of the single-message path: crypto.digest (hb_digest_small
up to 4 KiB), the bare hb_digest_small call, and for comparison the staged
paths it replaced (batch_digest_varlen with a caller-owned output, the bare
varlen and one-row fixed-width calls).  Median of 400 calls, us.

usage: python tools/digest_probe.py [alg] [len ...]
"""
import json
import os
import sys
import time
import ctypes

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_09333_b200 import _native  # noqa: E402
from paper_2407_09333_b200.crypto import DIGEST_LEN, batch_digest_varlen, digest  # noqa: E402

alg = sys.argv[1] if len(sys.argv) > 1 else "md5"
lens = [int(x) for x in sys.argv[2:]] or [55, 1024, 4096]
a = _native.ALG_ID[alg]
lib = _native.lib()


def med(f, k=400):
    for _ in range(20):
        f()
    ts = []
    for _ in range(k):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    return round(ts[k // 2] * 1e6, 2)


garr, ng = _native.gpu_array(None)
for L in lens:
    msg = bytes((i * 7 + 1) & 255 for i in range(L))
    m = np.frombuffer(msg, np.uint8).copy()
    off = np.array([0, L], np.uint64)
    out = np.empty((1, DIGEST_LEN[alg]), np.uint8)
    sbuf = ctypes.create_string_buffer(32)
    res = {"alg": alg, "len": L,
           "digest": med(lambda: digest(alg, msg)),
           "ctypes_digest_small": med(lambda: lib.hb_digest_small(a, msg, L, sbuf, -1)),
           "batch_digest_varlen": med(lambda: batch_digest_varlen(alg, m, off, out=out)),
           "ctypes_varlen": med(lambda: lib.hb_hash_varlen(a, m.ctypes.data, off.ctypes.data, 1, out.ctypes.data,
                                                            garr, ng, 0, None))}
    if L:
        res["ctypes_fixed_1row"] = med(lambda: lib.hb_hash_fixed(a, m.ctypes.data, 1, L, out.ctypes.data, garr, ng, 0,
                                                                  None))
    assert digest(alg, msg).data == batch_digest_varlen(alg, m, off)[0].tobytes()
    print(json.dumps(res), flush=True)
