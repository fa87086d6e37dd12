"""Per-call latency of the public API on small pinned batches (SHA-1, 64-byte
messages): wall time per call, with and without the engine's stage timings."""
import time, numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
from paper_2407_09333_b200.crypto import batch_digest
from paper_2407_09333_b200 import _native
def pinned(shape):
    return torch.empty(shape, dtype=torch.uint8, pin_memory=True).numpy()
for n, L in ((1, 64), (1024, 64), (65536, 64)):
    src = pinned((n, L)); src[:] = 7
    out = pinned((n, 20))
    for _ in range(20): batch_digest("sha1", src, out=out)
    ts = []
    for _ in range(200):
        t0 = time.perf_counter(); batch_digest("sha1", src, out=out, timing={}); ts.append(time.perf_counter() - t0)
    t = {}
    batch_digest("sha1", src, out=out, timing=t)
    ts.sort()
    print(n, L, "median us", round(ts[100]*1e6, 1), "p10", round(ts[20]*1e6, 1), {k: round(v, 4) if isinstance(v, float) else v for k, v in t.items()})
# the same calls without timing (the API default): the engine records no per-stage events
for n, L in ((1, 64), (1024, 64), (65536, 64)):
    src = pinned((n, L)); src[:] = 7
    out = pinned((n, 20))
    for _ in range(20): batch_digest("sha1", src, out=out)
    ts = []
    for _ in range(200):
        t0 = time.perf_counter(); batch_digest("sha1", src, out=out); ts.append(time.perf_counter() - t0)
    ts.sort()
    print(n, L, "untimed: median us", round(ts[100]*1e6, 1), "p10", round(ts[20]*1e6, 1))
