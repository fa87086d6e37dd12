"""Per-chunk timeline of the engine's H2D -> kernel -> D2H ring (the nsys
view of an end-to-end call; nsys is not installed in this image).

One timed `crypto.batch_digest` call on a pinned host array (and one
`batch_digest_varlen`) with `timing=`; prints the engine's stage unions, the
per-chunk CUDA-event spans from `hb_last_timeline` and an ASCII Gantt chart
(one row per chunk: `h` H2D, `K` kernel, `d` D2H), so the copy/compute
overlap of the chunk ring can be read off directly.

usage: python tools/e2e_timeline.py [n_msgs] [msg_len]   (default 2^22 x 1024 B)
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import hostref  # noqa: E402  (hashlib checker)
from paper_2407_09333_b200 import _native  # noqa: E402
from paper_2407_09333_b200.crypto import batch_digest, batch_digest_varlen  # noqa: E402


def pinned(nbytes):
    import ctypes

    p = _native.lib().hb_alloc_pinned(nbytes)
    if not p:
        raise MemoryError("hb_alloc_pinned")
    return np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_uint8)), shape=(nbytes,))


def gantt(spans, width=100, rows=24):
    t_end = max(s["t1_ms"] for s in spans)
    chunks = sorted({s["chunk"] for s in spans})
    mark = {"h2d": "h", "kernel": "K", "d2h": "d"}
    lines = [f"0 ms {'-' * (width - 12)} {t_end:.1f} ms"]
    for c in chunks[:rows]:
        line = [" "] * width
        for s in spans:
            if s["chunk"] != c:
                continue
            a = int(s["t0_ms"] / t_end * (width - 1))
            b = max(a, int(s["t1_ms"] / t_end * (width - 1)))
            for x in range(a, b + 1):
                line[x] = mark.get(s["stage"], "?")
        lines.append(f"{c:3d} " + "".join(line))
    if len(chunks) > rows:
        lines.append(f"... {len(chunks) - rows} more chunks")
    return "\n".join(lines)


def report(name, t, spans):
    print(f"## {name}")
    print(json.dumps(t))
    by = {}
    for s in spans:
        by.setdefault(s["stage"], []).append(s["t1_ms"] - s["t0_ms"])
    for k, v in by.items():
        print(f"{k}: {len(v)} spans, mean {np.mean(v):.3f} ms, sum {np.sum(v):.1f} ms")
    print(gantt(spans))
    print()


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
    L = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
    data = pinned(n * L).reshape(n, L)
    data[:] = hostref.random_bytes(n * L, 9).reshape(n, L)
    out = pinned(n * 16).reshape(n, 16)
    batch_digest("md5", data, gpus=[0], out=out)  # warm-up: ring allocation, attributes
    t = {}
    batch_digest("md5", data, gpus=[0], out=out, timing=t)
    spans = _native.last_timeline()
    rows = np.array([0, n // 2, n - 1])
    assert np.array_equal(out[rows], hostref.digests("md5", data[rows]))
    report(f"batch_digest md5 {n} x {L} B (pinned in/out)", t, spans)

    nv = n // 2
    lens = np.random.default_rng(4).integers(1, 4097, nv).astype(np.uint64)
    off = np.zeros(nv + 1, np.uint64)
    off[1:] = np.cumsum(lens)
    vdata = pinned(int(off[-1]))
    vdata[:] = hostref.random_bytes(int(off[-1]), 4)
    batch_digest_varlen("md5", vdata, off, gpus=[0])
    t = {}
    batch_digest_varlen("md5", vdata, off, gpus=[0], timing=t)
    report(f"batch_digest_varlen md5 {nv} x U(1, 4096) B (pinned in)", t, _native.last_timeline())


if __name__ == "__main__":
    main()
