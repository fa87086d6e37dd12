"""End-to-end throughput of the public API on PAGEABLE host buffers (a plain
numpy array in, a fresh numpy array out) vs page-locked ones, same bytes.
usage: python tools/e2e_pageable.py [alg] [n] [L]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import hostref  # noqa: E402
from paper_2407_09333_b200.crypto import batch_digest  # noqa: E402

alg = sys.argv[1] if len(sys.argv) > 1 else "md5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 22
L = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
data = hostref.random_bytes(n * L, 2).reshape(n, L)  # pageable
batch_digest(alg, data)  # warm
res = {}
for name in ("pageable_in_fresh_out", "pageable_in_reused_out"):
    out = np.empty((n, {"md5": 16, "sha1": 20, "sm3": 32}[alg]), np.uint8)
    out.fill(0)
    t0 = time.perf_counter()
    for _ in range(3):
        r = batch_digest(alg, data) if name.startswith("pageable_in_fresh") else batch_digest(alg, data, out=out)
    dt = (time.perf_counter() - t0) / 3
    res[name] = round(n * L / dt / 1e9, 2)
# cudaHostRegister path: pin the caller's pageable buffer in place (inside the
# timed region, as a caller would per batch), hash with direct DMA, unregister
import torch  # noqa: E402

cudart = torch.cuda.cudart()
out = np.empty((n, {"md5": 16, "sha1": 20, "sm3": 32}[alg]), np.uint8)
t0 = time.perf_counter()
for _ in range(3):
    cudart.cudaHostRegister(data.ctypes.data, data.nbytes, 0)
    cudart.cudaHostRegister(out.ctypes.data, out.nbytes, 0)
    batch_digest(alg, data, out=out)
    cudart.cudaHostUnregister(out.ctypes.data)
    cudart.cudaHostUnregister(data.ctypes.data)
dt = (time.perf_counter() - t0) / 3
res["host_register_per_call"] = round(n * L / dt / 1e9, 2)
cudart.cudaHostRegister(data.ctypes.data, data.nbytes, 0)
cudart.cudaHostRegister(out.ctypes.data, out.nbytes, 0)
t0 = time.perf_counter()
for _ in range(3):
    batch_digest(alg, data, out=out)
dt = (time.perf_counter() - t0) / 3
res["host_registered_once"] = round(n * L / dt / 1e9, 2)
print(json.dumps({"alg": alg, "n": n, "L": L, "GBps": res, "host_threads": os.cpu_count()}))
