"""Measure every BASELINE.json config on one B200 (kernel-only, device-resident
inputs; CUDA events on the launching stream) and write JSON lines.

  C1  SHA-1, 65,536 x 64 B                      (configs[0])
  C2  MD5, 2^24 x 1 KiB                         (configs[1])
  C3  SM3, 2^24 x 1 KiB                         (configs[2], 1-GPU point)
  C4  varlen, 2^22 msgs uniform 1 B-4 KiB, all 3 algorithms (configs[3], 1-GPU point)
  C5  message-size sweep 16 B-64 KiB x batch count, all 3 algorithms (configs[4], 1-GPU)

Every point's digests are checked against hashlib (tools/hostref.py) on a sample of rows.
usage: python tools/bench_configs.py [out.jsonl] [--quick]
"""

import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import hostref  # noqa: E402  (hashlib checker)
from paper_2407_09333_b200 import _native, device  # noqa: E402

DLEN = {"sha1": 20, "md5": 16, "sm3": 32}
READY = _native.HB_FLAG_INPUT_READY
import bench  # noqa: E402  (the same defensive MEASURED_PEAKS.json reader)

PEAK = bench.load_peaks()[0]["hbm_gbs"]
# minimal ALU-pipe ops per 64-byte block and the 64 lanes/clk/SM ALU rate
ALU_OPS = {"md5": 128, "sha1": 448, "sm3": 1084}
# Dependent-chain latency of one compression with nothing to overlap it (one
# warp per SM; tools/compress_bench.cu, profiles/compress_bench_r1b.txt): a
# message's blocks are compressed in sequence, so no batch finishes faster than
# (blocks per message) x this -- the binding bound when there are fewer
# messages than the GPU has lanes to overlap.
CHAIN_CYCLES = bench.CHAIN_CYCLES  # one set of measured constants (bench.py)
SMS = 148


def timed(fn, steps, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / steps


_FLUSH = []


def l2_flush():
    """Write a buffer of 2 x L2 so the next timed launch reads its batch from HBM."""
    if not _FLUSH:
        _FLUSH.append(torch.empty(bench.L2_DEFEAT_BYTES, dtype=torch.uint8, device="cuda:0"))
    _FLUSH[0].fill_(1)


def timed_cold(fn, reps, passes, warmup=2):
    """Mean time per pass of `fn` (which runs `passes` passes), each call
    preceded by an L2 flush outside its event pair: the batch is read from HBM
    at every timed repetition, as bench.py's rotation does for small batches."""
    for _ in range(warmup):
        fn()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for s, e in evs:
        l2_flush()
        s.record()
        fn()
        e.record()
    torch.cuda.synchronize()
    return sum(s.elapsed_time(e) for s, e in evs) / (reps * passes)


def clock_mhz():
    try:
        import subprocess

        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits", "-i", "0"],
                             capture_output=True, text=True).stdout.strip()
        return float(out.splitlines()[0])
    except Exception:
        return 1965.0


def roof(alg, n_blocks, bytes_hbm, ms, f_mhz, max_blocks_per_msg=0, overlapped=False):
    """overlapped: consecutive flagged passes run side by side (bench.pdl_overlap),
    so one batch's dependent chain does not bound the per-pass time."""
    t = {"hbm": bytes_hbm / (PEAK * 1e9),
         "alu": n_blocks * ALU_OPS[alg] / (64 * SMS * f_mhz * 1e6),
         "chain": max_blocks_per_msg * CHAIN_CYCLES[alg] / (f_mhz * 1e6)}
    cand = {k: v for k, v in t.items() if not (overlapped and k == "chain")}
    bound = max(cand, key=cand.get)
    return {"bound": bound, "t_roof_ms": round(t[bound] * 1e3, 4), "frac": round(t[bound] / (ms * 1e-3), 4),
            "t_ms": {k: round(v * 1e3, 4) for k, v in t.items()}, "chain_applies": not overlapped}


def fixed_point(alg, n, L, seed, steps, out, tag):
    buf = torch.empty(n * L, dtype=torch.uint8, device="cuda:0")
    device.fill_random(buf, seed)
    msgs = buf.view(n, L)
    dig = torch.empty((n, DLEN[alg]), dtype=torch.uint8, device="cuda:0")
    copies = None
    if n * L <= (64 << 20):
        # launch-bound sizes: CUDA-graph replays of 10 passes over 10 identical
        # copies, L2 flushed before each replay, so every pass reads HBM
        # (HB_FLAG_INPUT_READY, as bench.py passes it: the inputs are written
        # before the timed region, never by the preceding kernel)
        copies = [msgs] + [msgs.clone() for _ in range(9)]
        g = device.FixedHashGraph(alg, copies, dig, flags=READY)
        ms = timed_cold(g.replay, max(3, steps // 10), 10)
    elif n * L < bench.L2_DEFEAT_BYTES:  # fits (partly) in L2: flush between launches
        ms = timed_cold(lambda: device.hash_fixed(alg, msgs, out=dig, flags=READY), max(3, steps), 1)
    else:  # larger than 2 x L2: back-to-back launches already read HBM
        ms = timed(lambda: device.hash_fixed(alg, msgs, out=dig, flags=READY), steps)
    del copies
    rows = np.unique(np.concatenate([np.random.default_rng(seed).integers(0, n, 256), [0, n - 1]]))
    sample = msgs[torch.from_numpy(rows).cuda()].cpu().numpy()
    ok = bool(np.array_equal(dig.cpu().numpy()[rows], hostref.digests(alg, sample)))
    blocks = n * ((L + 8) // 64 + 1)
    f = clock_mhz()
    l2 = ("10-copy graph replay, L2 flushed before each" if n * L <= (64 << 20) else
          "L2 flushed before each launch" if n * L < bench.L2_DEFEAT_BYTES else "inputs > 2 x L2, back-to-back")
    rec = {"config": tag, "alg": alg, "n": n, "msg_len": L, "l2": l2, "ms": round(ms, 4),
           "GBps": round(n * L / ms / 1e6, 2), "Mhash_s": round(n / ms / 1e3, 2),
           # passes overlap only when launched back to back (graph replays, or launches with no
           # L2-flush kernel in between)
           "roofline": roof(alg, blocks, n * (L + DLEN[alg]), ms, f, (L + 8) // 64 + 1,
                            bench.pdl_overlap("fixed", n, (L + 8) // 64 + 1) and
                            (n * L <= (64 << 20) or n * L >= bench.L2_DEFEAT_BYTES)), "sm_mhz": f,
           "bit_exact_sample": ok}
    print(json.dumps(rec), flush=True)
    out.write(json.dumps(rec) + "\n")
    del buf, dig


def varlen_point(alg, n, maxlen, seed, steps, out, flags=0):
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, maxlen + 1, n).astype(np.int64)
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum(lens)
    total = int(off[-1])
    data = torch.empty(total + 16, dtype=torch.uint8, device="cuda:0")
    device.fill_random(data, seed)
    d_off = torch.from_numpy(off).cuda()
    dig = torch.empty((n, DLEN[alg]), dtype=torch.uint8, device="cuda:0")
    scratch = torch.empty(int(_native.lib().hb_varlen_scratch_bytes(n)), dtype=torch.uint8, device="cuda:0")
    ms = timed(lambda: device.hash_varlen(alg, data, d_off, out=dig, scratch=scratch, flags=flags, offset_base=0), steps)
    k = 512
    h = data[: int(off[k])].cpu().numpy()
    ok = bool(np.array_equal(dig[:k].cpu().numpy(), hostref.digests_varlen(alg, h, off[: k + 1])))
    blocks = int(((lens + 8) // 64 + 1).sum())
    f = clock_mhz()
    tagf = {0: "", _native.HB_FLAG_NO_SORT: " (no sort)", _native.HB_FLAG_VARLEN_WORDS: " (32-bit loads)",
            _native.HB_FLAG_VARLEN_COOP_OFF: " (per-thread 128-bit loads)",
            _native.HB_FLAG_VARLEN_COOP: " (warp-cooperative cp.async)"}[flags]
    rec = {"config": "C4 varlen" + tagf, "alg": alg, "n": n, "len": f"uniform 1-{maxlen}",
           "bytes": total, "ms": round(ms, 4), "GBps": round(total / ms / 1e6, 2), "Mhash_s": round(n / ms / 1e3, 2),
           "roofline": roof(alg, blocks, total + 8 * (n + 1) + n * DLEN[alg], ms, f, (maxlen + 8) // 64 + 1),
           "sm_mhz": f,
           "bit_exact_sample": ok}
    print(json.dumps(rec), flush=True)
    out.write(json.dumps(rec) + "\n")
    del data, d_off, dig, scratch


def sweep(out):
    """configs[4]: message size 16 B .. 64 KiB (13 powers of two) x batch count
    2^12, 2^14, ..., 2^22 and the largest power of two with n*L <= 16 GiB (cap 2^24)."""
    for k in range(13):
        L = 16 << k
        nmax = min(1 << 24, (16 << 30) // L)
        for n in sorted({x for x in (1 << 12, 1 << 14, 1 << 16, 1 << 18, 1 << 20, 1 << 22, nmax) if x <= nmax}):
            for alg in ("sha1", "md5", "sm3"):
                fixed_point(alg, n, L, 5000 + k, 5 if n * L > (1 << 30) else 30, out, "C5")
                torch.cuda.empty_cache()


def main():
    path = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else "gpurun_out/configs.jsonl"
    quick = "--quick" in sys.argv
    if "--sweep-only" in sys.argv:
        with open(path, "w") as out:
            sweep(out)
        return
    os.makedirs(os.path.dirname(path) or ".", exist_ok=True)
    t0 = time.time()
    with open(path, "w") as out:
        fixed_point("sha1", 65536, 64, 1, 200, out, "C1")
        fixed_point("md5", 1 << 24, 1024, 2, 20, out, "C2")
        fixed_point("sm3", 1 << 24, 1024, 3, 10, out, "C3")
        fixed_point("sha1", 1 << 24, 1024, 2, 10, out, "C5 point")
        for alg in ("sha1", "md5", "sm3"):
            varlen_point(alg, 1 << 22, 4096, 4, 5, out)
        varlen_point("md5", 1 << 22, 4096, 4, 5, out, flags=_native.HB_FLAG_NO_SORT)
        for alg in ("sha1", "md5", "sm3"):
            varlen_point(alg, 1 << 22, 4096, 4, 5, out, flags=_native.HB_FLAG_VARLEN_COOP_OFF)
            varlen_point(alg, 1 << 22, 4096, 4, 5, out, flags=_native.HB_FLAG_VARLEN_COOP)
        if not quick:
            sweep(out)
    print(f"# done in {time.time() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    main()
