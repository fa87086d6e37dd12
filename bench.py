#!/usr/bin/env python
"""Benchmark of the B200 batched-hash engine (the BASELINE.json north-star path).

Default workload = BASELINE.json configs[1]: MD5 over 2^24 random 1 KiB
messages per GPU (weak scaling under torchrun: rank r hashes global messages
[r*2^24, (r+1)*2^24)).  Prints ONE JSON line (rank 0):

  value        kernel-only GB/s of message bytes, inputs resident in HBM, CUDA
               events on the launching stream, max over ranks, summed over ranks
  e2e          the same metric through the public API (crypto.batch_digest on a
               pinned host array -> hb_hash_fixed): H2D + kernel + D2H per step
  roofline     dominant kernel (k_fixed_tma<MD5>) vs the measured HBM copy peak
  cpu_baseline the CPU oracle (C port of the reference algorithm) on a bounded
               sample of the same bytes, all host threads; its digests are also
               compared bit-for-bit with the GPU's for that sample

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload md5_1k|sha1_1k|sm3_1k|sha1_64|varlen|decimal|sweep]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SHA-1/MD5/SM3 hashed GB/s and Mhash/s at 1/2/4/8 B200 vs CPU reference"
DLEN = {"sha1": 20, "md5": 16, "sm3": 32}
# Minimal ALU-pipe operations per 64-byte block (LOP3 boolean functions, SHF
# rotates, LEA.HI rotate+add, PRMT byte swaps -- the work with no full-rate
# FMA-pipe equivalent; every addition can be issued as IMAD/VIADD instead).
# The ALU pipe retires 64 lanes/clk/SM on sm_100 (tools/pipe_bench.cu,
# profiles/pipe_bench_r1.txt).  DESIGN.md §4 derives these counts.
ALU_OPS_PER_BLOCK = {"md5": 128, "sha1": 448, "sm3": 1084}

WORKLOADS = {
    # name: (alg, n per GPU, msg_len, seed, BASELINE config)
    "md5_1k": ("md5", 1 << 24, 1024, 2, "configs[1]: MD5 over 2^24 random 1 KiB messages per B200"),
    "sha1_1k": ("sha1", 1 << 24, 1024, 2, "SHA-1 over 2^24 random 1 KiB messages per B200 (configs[4] point)"),
    "sm3_1k": ("sm3", 1 << 24, 1024, 3, "configs[2]: SM3 over 2^24 random 1 KiB messages per B200"),
    "sha1_64": ("sha1", 65536, 64, 1, "configs[0]: SHA-1 over 65,536 random 64-byte messages"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ----------------------------------------------------------------- clocks --
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 50 ms while active."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines: list[str] = []
        self.active = False
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            if self.active:
                self.lines.append(line.strip())

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx.append(float(p[2]))
            except ValueError:
                continue
            for name, v in zip(names, p[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------ distributed --
def dist_setup(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def reduce_max(x: float, world: int, local: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured (MEASURED_PEAKS.json)"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md)"


def load_ncu_traffic(alg: str, n: int, L: int):
    """dram bytes per launch of the dominant kernel from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    k = d.get(f"{alg}_{n}x{L}")
    return k.get("dram_bytes") if k else None


# ------------------------------------------------------------ CPU oracle --
def cpu_oracle_run(alg: str, rows, threads: int):
    import oracle

    t0 = time.perf_counter()
    out = oracle.batch_fixed(alg, rows, threads=threads)
    return out, time.perf_counter() - t0


def cpu_sample_rows(alg: str, L: int, n: int, threads: int, target_s: float):
    """Pick a sample size giving ~target_s seconds of wall time on `threads` threads."""
    import oracle

    probe = oracle.fill_random(min(n, 2048) * L, 123).reshape(-1, L)
    _, t = cpu_oracle_run(alg, probe, 1)
    per_row = max(t / probe.shape[0], 1e-9)
    rows = int(target_s * threads / per_row)
    rows = max(threads * 16, min(n, rows))
    return rows


# ---------------------------------------------------------------- our arm --
def run_ours(args):
    import numpy as np
    import torch

    from paper_2407_09333_b200 import _native, device
    from paper_2407_09333_b200.crypto import batch_digest

    world, rank, local = dist_setup(args)
    alg, n, L, seed, cfg_desc = WORKLOADS[args.workload]
    if args.n:
        n = args.n
    dlen = DLEN[alg]
    stream = torch.cuda.current_stream(local)
    sampler = ClockSampler(local)
    sampler.start()

    # ---- inputs resident in HBM: global messages [rank*n, (rank+1)*n)
    buf = torch.empty(n * L, dtype=torch.uint8, device=f"cuda:{local}")
    device.fill_random(buf, seed, byte_offset=rank * n * L)
    msgs = buf.view(n, L)
    out = torch.empty((n, dlen), dtype=torch.uint8, device=f"cuda:{local}")
    torch.cuda.synchronize()

    def step():
        device.hash_fixed(alg, msgs, out=out)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    l0 = _native.launch_count()
    sampler.active = True
    t_wall0 = time.perf_counter()
    for s, e in evs:
        s.record(stream)
        step()
        e.record(stream)
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall0
    sampler.active = False
    launches = _native.launch_count() - l0
    barrier(world)
    per_step = [s.elapsed_time(e) for s, e in evs]
    ms_local = sum(per_step) / len(per_step)
    ms = reduce_max(ms_local, world, local)
    total_bytes = world * n * L
    value = total_bytes / (ms * 1e-3) / 1e9
    mhash = world * n / (ms * 1e-3) / 1e6
    log(f"[rank {rank}] kernel-only {alg} {n}x{L}: {ms_local:.3f} ms/step (min {min(per_step):.3f}, "
        f"max {max(per_step):.3f}); wall {t_wall * 1e3 / args.steps:.3f} ms/step")

    # ---- end to end through the public API: pinned host input -> hb_hash_fixed
    e2e = None
    lib = _native.lib()
    hp = lib.hb_alloc_pinned(n * L) if not args.no_e2e else None
    if hp:
        import ctypes

        host = np.ctypeslib.as_array(ctypes.cast(hp, ctypes.POINTER(ctypes.c_uint8)), shape=(n * L,)).reshape(n, L)
        host_t = torch.from_numpy(host.reshape(-1))
        host_t.copy_(buf, non_blocking=False)  # same bytes as the device-resident run
        e2e_steps = args.e2e_steps or min(args.steps, 10)
        tim = {}
        for _ in range(max(1, min(args.warmup, 2))):
            batch_digest(alg, host, gpus=[local])
        barrier(world)
        torch.cuda.synchronize()
        sampler.active = True
        l1 = _native.launch_count()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            res = batch_digest(alg, host, gpus=[local], timing=tim)
        t1 = time.perf_counter()
        sampler.active = False
        e2e_launches = _native.launch_count() - l1
        barrier(world)
        e2e_ms = reduce_max((t1 - t0) * 1e3 / e2e_steps, world, local)
        ok = bool(np.array_equal(res, out.cpu().numpy()))
        e2e = {"value": round(total_bytes / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": world * n * L, "d2h_bytes_per_step": world * n * dlen,
               "ms_per_step": round(e2e_ms, 3), "mhash_per_s": round(world * n / (e2e_ms * 1e-3) / 1e6, 2),
               "api": "paper_2407_09333_b200.crypto.batch_digest(pinned host array) -> hb_hash_fixed",
               "steps": e2e_steps, "engine_timing_last_step": {k: (round(v, 3) if isinstance(v, float) else v)
                                                               for k, v in tim.items()},
               "gpu_launches": e2e_launches, "matches_device_run": ok}
        log(f"[rank {rank}] e2e {e2e_ms:.1f} ms/step, engine {tim}")
        del host_t, host
        lib.hb_free_pinned(hp)
    sampler.stop()

    # ---- CPU baseline + bit-exact sample check (rank 0, N=1 only)
    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        rows = cpu_sample_rows(alg, L, n, threads, args.cpu_seconds)
        sample = buf[: rows * L].cpu().numpy().reshape(rows, L)
        ref, t = cpu_oracle_run(alg, sample, threads)
        parity = {"rows_checked": rows, "bit_exact": bool(np.array_equal(ref, out[:rows].cpu().numpy()))}
        cpu = {"value": round(rows * L / t / 1e9, 4), "unit": "GB/s", "cores": threads, "kind": "port",
               "sample": f"first {rows} of the {n} x {L} B messages (same bytes), oracle/hetoc_oracle.c "
                         f"batch_fixed on {threads} threads, {t:.2f} s",
               "mhash_per_s": round(rows / t / 1e6, 4)}

    # ---- roofline of the dominant kernel (k_fixed_tma<alg>)
    peaks, peak_src = load_peaks()
    alg_bytes = n * (L + dlen)  # per launch: message bytes read + digests written
    achieved = alg_bytes / (ms_local * 1e-3) / 1e9
    blocks = n * ((L + 8) // 64 + 1)
    clk = sampler.summary()
    f_max = peaks.get("sm_max_mhz", 1965.0)
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    alu_peak = sms * 64 * f_max * 1e6  # ALU-pipe lane-ops/s at max clock
    alu_ach = blocks * ALU_OPS_PER_BLOCK[alg] / (ms_local * 1e-3)
    t_hbm = alg_bytes / (peaks["hbm_gbs"] * 1e9)
    t_alu = blocks * ALU_OPS_PER_BLOCK[alg] / alu_peak
    alu = {"achieved": round(alu_ach / 1e12, 3), "peak": round(alu_peak / 1e12, 3), "unit": "Tops/s",
           "frac": round(alu_ach / alu_peak, 4), "alu_ops_per_block": ALU_OPS_PER_BLOCK[alg],
           "blocks_per_launch": blocks, "clock_mhz": f_max}
    if t_hbm >= t_alu:
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": round(achieved / peaks["hbm_gbs"], 4)}
    else:  # integer (ALU-pipe) bound: report against the ALU-pipe roofline, HBM alongside
        roof = {"bound": "alu", "achieved": alu["achieved"], "peak": alu["peak"], "unit": "Tops/s",
                "frac": alu["frac"], "hbm_achieved_gbs": round(achieved, 1), "hbm_peak_gbs": peaks["hbm_gbs"]}
    roof.update({"traffic": load_ncu_traffic(alg, n, L), "kernel": f"k_fixed_tma_ws<{alg}>",
                 "bytes_per_launch": alg_bytes, "peak_source": peak_src,
                 "t_roof_ms": round(max(t_hbm, t_alu) * 1e3, 4), "alu_pipe": alu})
    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
                "data": f"synthetic: counter-based splitmix64 bytes (seed {seed}), generated on device",
                "config": {"workload": f"{alg} {n} x {L} B fixed-width per GPU ({cfg_desc})", "alg": alg,
                           "msgs_per_gpu": n, "msg_len": L, "global_batch_msgs": world * n,
                           "parallelism": f"message-range shards over {world} GPU(s), no collective",
                           "l2": "inputs are %.1f GiB per GPU >> 126 MB L2; no flush needed" % (n * L / 2**30)},
                "mhash_per_s": round(mhash, 2), "clocks": clk, "e2e": e2e, "gpu_launches": launches,
                "roofline": roof, "cpu_baseline": cpu, "parity": parity}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


# --------------------------------------------------------- reference arm --
def run_reference(args):
    """The reference algorithm's CPU implementation (oracle port of hetoc.crypto;
    the reference itself is pure Python/numpy and is not installed on the box)
    on all host threads, each step a bounded sample of the same workload."""
    import numpy as np

    import oracle

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    alg, n, L, seed, cfg_desc = WORKLOADS[args.workload]
    if args.n:
        n = args.n
    threads = os.cpu_count() or 1
    rows = cpu_sample_rows(alg, L, n, threads, args.ref_step_seconds)
    data = oracle.fill_random(rows * L, seed).reshape(rows, L)
    for _ in range(args.warmup):
        cpu_oracle_run(alg, data[: max(threads, rows // 8)], threads)
    times = []
    for _ in range(args.steps):
        _, t = cpu_oracle_run(alg, data, threads)
        times.append(t)
    t = sum(times) / len(times)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    value = rows * L / t / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": f"synthetic: counter-based splitmix64 bytes (seed {seed})",
            "config": {"workload": f"{alg} {n} x {L} B fixed-width per GPU ({cfg_desc})", "alg": alg,
                       "msgs_per_gpu": n, "msg_len": L},
            "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": threads, "kind": "port",
                             "sample": f"{rows} of the {n} x {L} B messages per step, oracle/hetoc_oracle.c "
                                       f"(C restatement of hetoc.crypto) on {threads} threads"},
            "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "mhash_per_s": round(rows / t / 1e6, 4)}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="md5_1k")
    ap.add_argument("--n", type=int, default=0, help="override messages per GPU")
    ap.add_argument("--e2e-steps", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=3.0)
    ap.add_argument("--ref-step-seconds", type=float, default=1.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        log("note: timing rules want >= 3 warm-up steps")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
