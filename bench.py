#!/usr/bin/env python
"""Benchmark of the B200 batched-hash engine (the BASELINE.json north-star path).

Default workload = BASELINE.json configs[1]: MD5 over 2^24 random 1 KiB
messages per GPU (weak scaling: rank r hashes global messages
[r*2^24, (r+1)*2^24)).  Prints ONE JSON line (rank 0):

  value        kernel-only GB/s of message bytes, inputs resident in HBM: one
               CUDA-event pair on the launching stream around K back-to-back
               steps, max over ranks; bytes summed over ranks
  e2e          the same metric through the public API (crypto.batch_digest on
               a pinned host array): H2D + kernels + D2H every step;
               e2e_pageable: the reference call shape (pageable numpy in, fresh
               array out)
  roofline     the kernel that ran (its name from the library), against the
               HBM copy peak or the ALU-pipe peak (+ the dependent-chain bound)
  cpu_baseline the CPU oracle (C port of the reference algorithm) on the same
               bytes, all host threads; its digests are compared with the GPU's
  configs      every other BASELINE config measured the same way in the same
               run: C1 (SHA-1 65,536 x 64 B), C3 (SM3 2^24 x 1 KiB split over
               the GPUs), C4 (varlen U(1, 4 KiB) x 3 algorithms) and a reduced
               C5 grid (16 B / 1 KiB / 64 KiB x three batch counts x 3
               algorithms), each with kernel-only and e2e rates, roofline,
               clocks and full-batch parity (N=1; a row sample per rank at N>1)

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--configs all|none] [--gather none|p2p] [--dry-run]
                  [--workload md5_1k|sha1_1k|sm3_1k|sha1_64|varlen_{md5,sha1,sm3}|paper_{sha1,md5,sm3}]

--gpus N > 1 without WORLD_SIZE in the environment relaunches this script
under torch.distributed.run with N ranks (one process per GPU); it fails
loudly when fewer than N GPUs are visible (unless $HB_BENCH_BACKEND=gloo, the
CPU test hook that lets ranks share GPUs).
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

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
# SURVEY.md §8(d)'s roofline, reported alongside: fused integer instructions
# per block (its Appendix B) at an issue peak of 128 lanes/clk/SM.  It is
# looser than the ALU-pipe bound above for SHA-1 and SM3 -- their 448 / 1,084
# boolean/rotate ops can only issue at 64 lanes/clk/SM -- so it reads lower.
SURVEY_C_ALG = {"md5": 324, "sha1": 613, "sm3": 1412}
# Dependent-chain latency of one compression (cycles, one warp per SM: 4,736
# messages of 64 KiB, profiles/r2/ab_chain_r2d.txt and ab_mid_r2p.txt; the
# smallest measurement).  MD5 is the round-variant-6 tile the dispatch runs
# below 2^16 messages (544.6 us for 1,025 blocks at 1,965 MHz, the best of the final passes; variant 3:
# 1,132, variant 1: 1,462-1,509).  A batch with too few messages to overlap
# cannot finish before (blocks per message) x this.
CHAIN_CYCLES = {"md5": 1044, "sha1": 1116, "sm3": 2514}
_BACKEND = os.environ.get("HB_BENCH_BACKEND", "nccl")


def alu_ops_decimal(alg, width):
    """ALU-pipe ops of one single-block decimal message (the paper workload)
    under the same cost model as ALU_OPS_PER_BLOCK, with constant folding:
    only the digit words vary between messages, the padding words (0x80,
    zeros, the length) are compile-time constants, so a boolean function or
    rotate whose inputs are all constant costs nothing.  An XOR of t
    non-constant terms (plus one folded constant) is ceil((t-1)/2) LOP3s;
    byte swaps are free (the digit bytes can be placed in either order).
    Gives 127 / 404 / 1,010 for MD5 / SHA-1 / SM3 at width 9 (the same model
    with every word non-constant: 127 / 427 / 1,057 -- the first rounds see
    the constant IV either way).  DESIGN.md §4."""
    if width + 9 > 64:
        raise ValueError("one-block messages only")
    V = None  # a per-message (non-constant) value; ints are constants
    n_var_words = (width + 3) // 4  # digit bytes, plus the 0x80 byte when it shares a word
    words = [V if i < n_var_words else 0 for i in range(16)]
    cost = 0

    def xor(*terms):  # one XOR group: LOP3 takes three inputs (or an immediate)
        nonlocal cost
        nv = sum(t is V for t in terms)
        if nv == 0:
            return 0
        cost += -(-(nv - 1) // 2)
        return V

    def rot(x):
        nonlocal cost
        if x is V:
            cost += 1
        return x if x is not V else V

    def lop(*xs):  # any other 3-input boolean function
        nonlocal cost
        if any(x is V for x in xs):
            cost += 1
            return V
        return 0

    def add(*xs):
        return V if any(x is V for x in xs) else 0

    if alg == "md5":
        a = b = c = d = 0
        for i in range(64):
            f = lop(b, c, d)
            g = i if i < 16 else (5 * i + 1) % 16 if i < 32 else (3 * i + 5) % 16 if i < 48 else (7 * i) % 16
            u = add(a, f, words[g])
            a, d, c, b = d, c, b, add(b, rot(u))
    elif alg == "sha1":
        w = list(words)
        a = b = c = d = e = 0
        for t in range(80):
            if t >= 16:
                w[t & 15] = rot(xor(w[(t - 3) & 15], w[(t - 8) & 15], w[(t - 14) & 15], w[t & 15]))
            f = xor(b, c, d) if 20 <= t < 40 or t >= 60 else lop(b, c, d)
            a, b, c, d, e = add(rot(a), f, e, w[t & 15]), a, rot(b), c, d
    elif alg == "sm3":
        w = list(words) + [0] * 52
        for j in range(16, 68):
            x = xor(w[j - 16], w[j - 9], rot(w[j - 3]))
            w[j] = xor(x, rot(x), rot(x), rot(w[j - 13]), w[j - 6]) if x is V else xor(rot(w[j - 13]), w[j - 6])
        A = B = C = D = E = F = G = H = 0
        for j in range(64):
            a12 = rot(A)
            ss1 = rot(add(a12, E))
            ss2 = xor(ss1, a12)
            ff = xor(A, B, C) if j < 16 else lop(A, B, C)
            gg = xor(E, F, G) if j < 16 else lop(E, F, G)
            tt1 = add(ff, D, ss2, xor(w[j], w[j + 4]))
            tt2 = add(gg, H, ss1, w[j])
            D, C, B, A = C, rot(B), A, tt1
            H, G, F = G, rot(F), E
            E = xor(tt2, rot(tt2), rot(tt2))
    else:
        raise ValueError(alg)
    return cost


# ----------------------------------------------------------------- clocks --
class ClockSampler:
    """SM clock, max clock, power and clock-event (throttle) reasons of one GPU,
    polled through NVML every 10 ms on a background thread (nvidia-smi -lms
    as the fallback); begin()/end() bracket a timed region, and end() also
    takes one synchronous sample so even a sub-10 ms region has a record."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples: list[tuple] = []  # (t, sm_mhz, max_mhz, power_w, reasons bitmask)
        self.stop_ev = threading.Event()
        self.thread = None
        self.nvml = None
        self.handle = None
        self.source = "none"

    def _query(self):
        n = self.nvml
        h = self.handle
        sm = n.nvmlDeviceGetClockInfo(h, n.NVML_CLOCK_SM)
        mx = n.nvmlDeviceGetMaxClockInfo(h, n.NVML_CLOCK_SM)
        try:
            pw = n.nvmlDeviceGetPowerUsage(h) / 1000.0
        except Exception:
            pw = None
        try:
            rs = n.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            rs = n.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        return (time.perf_counter(), float(sm), float(mx), pw, int(rs))

    def start(self):
        try:
            import pynvml
            import torch

            pynvml.nvmlInit()
            uuid = str(torch.cuda.get_device_properties(self.gpu).uuid).lower().removeprefix("gpu-")
            for i in range(pynvml.nvmlDeviceGetCount()):
                h = pynvml.nvmlDeviceGetHandleByIndex(i)
                u = pynvml.nvmlDeviceGetUUID(h)
                u = (u.decode() if isinstance(u, bytes) else u).lower().removeprefix("gpu-")
                if u == uuid:
                    self.handle = h
            if self.handle is None:
                self.handle = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.nvml = pynvml
            self._query()
            self.source = "NVML, 10 ms"
        except Exception:
            self.nvml = None
            self.source = "unavailable"
            return
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def _run(self):
        while not self.stop_ev.wait(0.01):
            try:
                self.samples.append(self._query())
            except Exception:
                pass

    def begin(self):
        return time.perf_counter()

    def end(self, t0):
        if self.nvml is not None:
            try:
                self.samples.append(self._query())
            except Exception:
                pass
        return self.summary([s for s in self.samples if s[0] >= t0])

    def stop(self):
        self.stop_ev.set()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self, samples):
        if not samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "source": self.source}
        reasons = sorted({name for s in samples for name, bit in self.REASONS.items() if s[4] & bit})
        pw = [s[3] for s in samples if s[3] is not None]
        return {"sm_mhz": statistics.median(s[1] for s in samples), "sm_min_mhz": min(s[1] for s in samples),
                "sm_max_mhz": max(s[2] for s in samples), "power_w_max": round(max(pw), 1) if pw else None,
                "reasons": reasons, "reason_masks": sorted({hex(s[4]) for s in samples}),
                "samples": len(samples), "source": self.source}



WORKLOADS = {
    # name: (alg | "varlen:"alg | "decimal:"alg | "strong:"alg, n per GPU, msg_len | max varlen length, seed, BASELINE config)
    "md5_1k": ("md5", 1 << 24, 1024, 2, "configs[1]: MD5 over 2^24 random 1 KiB messages per B200"),
    "sha1_1k": ("sha1", 1 << 24, 1024, 2, "SHA-1 over 2^24 random 1 KiB messages per B200 (configs[4] point)"),
    "sm3_1k": ("strong:sm3", 1 << 24, 1024, 3,
               "configs[2]: SM3 over 2^24 random 1 KiB messages sharded by message range across the GPUs"),
    "sha1_64": ("sha1", 65536, 64, 1, "configs[0]: SHA-1 over 65,536 random 64-byte messages"),
    "varlen_md5": ("varlen:md5", 1 << 22, 4096, 4, "configs[3]: mixed variable-length batch, uniform 1 B-4 KiB"),
    "varlen_sha1": ("varlen:sha1", 1 << 22, 4096, 4, "configs[3]: mixed variable-length batch, uniform 1 B-4 KiB"),
    "varlen_sm3": ("varlen:sm3", 1 << 22, 4096, 4, "configs[3]: mixed variable-length batch, uniform 1 B-4 KiB"),
    "paper_sha1": ("decimal:sha1", 10**9, 9, 0, "paper workload: 10^9 x 9-digit messages, PAPER.md:206"),
    "paper_md5": ("decimal:md5", 10**9, 9, 0, "paper workload: 10^9 x 9-digit messages, PAPER.md:206"),
    "paper_sm3": ("decimal:sm3", 10**9, 9, 0, "paper workload: 10^9 x 9-digit messages, PAPER.md:206"),
}

# The reduced configs[4] grid of the suite: message size -> batch counts per
# GPU (at most 16 GiB of messages per GPU), x the three algorithms.
C5_GRID = {16: (1 << 16, 1 << 20, 1 << 24), 1024: (1 << 16, 1 << 20, 1 << 24), 65536: (1 << 12, 1 << 16, 1 << 18)}
C5_SEED = 5000


def suite_specs():
    """(entry name, WORKLOADS-style spec) of every BASELINE config besides the headline."""
    out = [("C1_sha1_64", WORKLOADS["sha1_64"]), ("C3_sm3_1k", WORKLOADS["sm3_1k"])]
    for alg in ("md5", "sha1", "sm3"):
        out.append((f"C4_varlen_{alg}", WORKLOADS[f"varlen_{alg}"]))
    k = 0
    for alg in ("md5", "sha1", "sm3"):
        for L, counts in C5_GRID.items():
            for n in counts:
                out.append((f"C5_{alg}_{L}x{n}",
                            (alg, n, L, C5_SEED + k, f"configs[4] point: {alg} {n} x {L} B per GPU")))
                k += 1
    return out


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------ distributed --
HOST = {"affinity": "unbound (one process, N=1)"}


def dist_setup():
    """Process group (NCCL, one GPU per rank; gloo with ranks sharing GPUs as
    the CPU test hook) and this rank's host side bound to its GPU's NUMA node."""
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if _BACKEND == "gloo":
            local = local % max(1, torch.cuda.device_count())
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            t0 = time.perf_counter()
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            log(f"[rank {rank}] NCCL communicator on cuda:{local} initialised in "
                f"{(time.perf_counter() - t0) * 1e3:.0f} ms (world {world})")
        from paper_2407_09333_b200.device import bind_host_to_gpu

        cores = bind_host_to_gpu(local)
        HOST["affinity"] = f"{len(cores)} GPU-local cores (NVML)" if cores else "unbound (NVML gave no mask)"
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def rank_record(rank, local):
    import torch

    p = torch.cuda.get_device_properties(local)
    return {"rank": rank, "local_rank": local, "cuda_device": local, "gpu": p.name,
            "pci_bus_id": f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}",
            "uuid": str(p.uuid), "pid": os.getpid(), "host": socket.gethostname(),
            "cpu_affinity": len(os.sched_getaffinity(0)), "host_affinity": HOST["affinity"]}


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def _reduce(x: float, world: int, local: int, op) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cpu" if _BACKEND == "gloo" else f"cuda:{local}")
    dist.all_reduce(t, op=op)
    return float(t.item())


def reduce_max(x, world, local):
    import torch.distributed as dist

    return _reduce(x, world, local, dist.ReduceOp.MAX if world > 1 else None)


def reduce_min(x, world, local):
    import torch.distributed as dist

    return _reduce(x, world, local, dist.ReduceOp.MIN if world > 1 else None)


def reduce_sum(x, world, local):
    import torch.distributed as dist

    return _reduce(x, world, local, dist.ReduceOp.SUM if world > 1 else None)


def gather_objects(obj, world):
    if world == 1:
        return [obj]
    import torch.distributed as dist

    out = [None] * world
    dist.all_gather_object(out, obj)
    return out


# ------------------------------------------------------------- peaks/ncu --
def load_peaks():
    """Roofline denominators: the driver-measured HBM copy bandwidth from
    MEASURED_PEAKS.json ("of measured"), else B200_PROFILING.md's fallback
    ("of fallback").  Only a positive numeric `hbm_gbs` is taken from the file;
    anything else in it is ignored rather than trusted."""
    peaks = {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if not os.path.exists(p):
        return peaks, "fallback (B200_PROFILING.md)"
    try:
        with open(p) as f:
            d = json.load(f)
        hbm = d.get("hbm_gbs") if isinstance(d, dict) else None
        if isinstance(hbm, (int, float)) and hbm > 0:
            peaks["hbm_gbs"] = float(hbm)
            mhz = d.get("sm_max_mhz")
            if isinstance(mhz, (int, float)) and mhz > 0:
                peaks["sm_max_mhz"] = float(mhz)
            return peaks, "measured (MEASURED_PEAKS.json)"
    except (OSError, ValueError):
        pass
    return peaks, "fallback (B200_PROFILING.md; MEASURED_PEAKS.json unreadable or without hbm_gbs)"


# bench workloads whose shape is a suite entry: the suite's ncu record is the one
# tools/ncu_configs.py refreshes with every capture
NCU_ALIASES = {"sha1_64": "C1_sha1_64", "sm3_1k": "C3_sm3_1k", "sha1_1k": "C5_sha1_1024x16777216",
               "varlen_md5": "C4_varlen_md5", "varlen_sha1": "C4_varlen_sha1", "varlen_sm3": "C4_varlen_sm3"}


def _kernel_key(name):
    """'void hb::k_x<1, false, -1>(...)' and 'void k_x<1, 0, (int)-1>(...)' -> 'k_x<1,0,-1>'."""
    base = (name or "").replace("(int)", "").split("(")[0].replace("void ", "").replace("hb::", "")
    head, _, args = base.partition("<")
    vals = [a.strip().replace("false", "0").replace("true", "1") for a in args.rstrip(">").split(",")]
    return head.strip() + "<" + ",".join(vals) + ">"


def load_ncu(name: str, kernel: str = None):
    """The committed ncu --set full record of this config's dominant kernel
    (profiles/ncu_summary.json, tools/ncu_configs.py): dram bytes per launch.
    A record of a different kernel than the one that ran is not used."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        summ = json.load(f)
    rec = summ.get(NCU_ALIASES.get(name, name)) or summ.get(name)
    if rec and kernel and _kernel_key(rec.get("kernel")) != _kernel_key(kernel):
        return None
    return rec


def library_info():
    """The engine library this run loaded: path, size, A/B build flag and the
    number of kernels in its sm_100a cubins (cuobjdump, when present)."""
    from paper_2407_09333_b200 import _native

    path = _native.LIB_PATH
    info = {"so": os.path.relpath(path, ROOT), "bytes": os.path.getsize(path), "ab_build": _native.built_with_ab()}
    try:
        sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True, timeout=60).stdout
        info["kernels"] = sass.count("Function :")
        info["arch"] = sorted({l.split("=")[-1].strip() for l in sass.splitlines() if "arch = " in l})
    except Exception:
        info["kernels"] = None
    return info


def cpu_info():
    """lscpu model / sockets x cores / threads and the SHA-NI flag."""
    info = {"os_cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0))}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = {}
        for ln in out.splitlines():
            if ":" in ln:
                k, v = ln.split(":", 1)
                kv[k.strip()] = v.strip()
        info.update({"model": kv.get("Model name"), "sockets": kv.get("Socket(s)"),
                     "cores_per_socket": kv.get("Core(s) per socket"), "threads_per_core": kv.get("Thread(s) per core"),
                     "numa_nodes": kv.get("NUMA node(s)")})
        flags = kv.get("Flags", "").split()
        info["sha_ni"] = "sha_ni" in flags
    except Exception as e:  # lscpu missing: keep what os gives
        info["lscpu"] = f"unavailable ({e})"
    return info


# ---------------------------------------------------------- host buffers --
class PinnedPool:
    """One page-locked host buffer per role, grown to the largest config and
    reused (cudaHostAlloc of 16 GiB takes seconds; every config would pay it)."""

    def __init__(self):
        self.bufs = {}

    def get(self, role: str, nbytes: int) -> np.ndarray:
        import ctypes

        from paper_2407_09333_b200 import _native

        lib = _native.lib()
        cur = self.bufs.get(role)
        if cur is None or cur[1] < nbytes:
            if cur is not None:
                lib.hb_free_pinned(cur[0])
            size = max(nbytes, 1)
            p = lib.hb_alloc_pinned(size)
            if not p:
                raise MemoryError(f"hb_alloc_pinned({size}) failed: {_native.last_error()}")
            self.bufs[role] = (p, size)
            cur = self.bufs[role]
        arr = np.ctypeslib.as_array(ctypes.cast(cur[0], ctypes.POINTER(ctypes.c_uint8)), shape=(cur[1],))
        return arr[:nbytes]

    def close(self):
        from paper_2407_09333_b200 import _native

        for p, _ in self.bufs.values():
            _native.lib().hb_free_pinned(p)
        self.bufs.clear()


GRAPH_STEPS = 10
L2_DEFEAT_BYTES = 2 * 126 * 10**6  # twice the B200's 126 MB L2
PROFILE_ONLY = False  # tools/ncu_configs.py: no rotated copies, no graphs (one launch per config)
INPUT_READY = 0x40  # HB_FLAG_INPUT_READY (include/hetoc_b200.h): inputs resident, not written by the previous kernel


# -------------------------------------------------------------- workloads --
class FixedWorkload:
    """n messages of L bytes per GPU, (n, L) row-major (configs[0..2], [4])."""

    kind = "fixed"

    def __init__(self, name, alg, n, L, seed, desc, rank, local, world=1, strong=False):
        import torch

        from paper_2407_09333_b200 import device
        from paper_2407_09333_b200.passes import partition_range

        self.name, self.alg, self.L, self.seed, self.desc, self.local = name, alg, L, seed, desc, local
        self.scaling = "strong" if strong else "weak"
        if strong:  # configs[2]: the SAME n messages split over the GPUs by message range
            lo, hi = partition_range(0, n, [1.0 / world] * world)[rank]
            self.total_msgs = n
        else:  # n messages per GPU: rank r hashes global messages [r*n, (r+1)*n)
            lo, hi = rank * n, (rank + 1) * n
            self.total_msgs = world * n
        n = hi - lo
        self.n, self.lo = n, lo
        self.dlen = DLEN[alg]
        self.buf = torch.empty(max(1, n * L), dtype=torch.uint8, device=f"cuda:{local}")
        device.fill_random(self.buf[: n * L], seed, byte_offset=lo * L)
        self.msgs = self.buf[: n * L].view(n, L)
        self.out = torch.empty((n, self.dlen), dtype=torch.uint8, device=f"cuda:{local}")
        self.msg_bytes = n * L
        self.total_bytes = self.total_msgs * L
        self.alg_bytes = n * (L + self.dlen)  # message bytes read once + digests written once
        self.blocks_per_msg = (L + 8) // 64 + 1
        self.blocks = n * self.blocks_per_msg
        self.h2d_bytes, self.d2h_bytes = n * L, n * self.dlen
        # A step of a small batch is a few microseconds of GPU work, less than a
        # launch from Python: those steps run as CUDA-graph replays of
        # GRAPH_STEPS back-to-back passes (each pass hashes the whole batch).
        # A batch smaller than 2x L2 would be re-read from L2 by back-to-back
        # steps: it is rotated over enough identical copies (a multiple of
        # GRAPH_STEPS, >= 2 x 126 MB in total) that every step reads a copy
        # last touched >= 63 steps earlier, i.e. from HBM.
        self.copies = [self.msgs]
        if n * L and n * L < L2_DEFEAT_BYTES and not PROFILE_ONLY:
            r = -(-L2_DEFEAT_BYTES // (n * L))
            r = -(-r // GRAPH_STEPS) * GRAPH_STEPS
            self.copies += [self.msgs.clone() for _ in range(r - 1)]
        self.turn = 0
        self.graphs, self.graph1s = [], []
        if n * L <= (64 << 20) and not PROFILE_ONLY:
            # GRAPH_STEPS consecutive copies per replayed graph, one single-pass graph per copy for remainders
            for j in range(0, len(self.copies), GRAPH_STEPS):
                group = self.copies[j:j + GRAPH_STEPS]
                reps = GRAPH_STEPS // len(group) if len(group) < GRAPH_STEPS else 1
                self.graphs.append(device.FixedHashGraph(alg, group, self.out, flags=INPUT_READY, repeats=reps))
            self.graph1s = [device.FixedHashGraph(alg, c, self.out, flags=INPUT_READY) for c in self.copies]

    def step(self):
        from paper_2407_09333_b200 import device

        i = self.turn % len(self.copies)
        self.turn += 1
        if self.graph1s:
            self.graph1s[i].replay()
        else:
            device.hash_fixed(self.alg, self.copies[i], out=self.out, flags=INPUT_READY)

    def run_steps(self, k):
        if self.graphs:
            # start on a graph boundary (skipping ahead only lengthens every copy's
            # idle time), whole GRAPH_STEPS-pass graphs, then single passes
            self.turn = -(-self.turn // GRAPH_STEPS) * GRAPH_STEPS
            while k >= GRAPH_STEPS:
                self.graphs[(self.turn % len(self.copies)) // GRAPH_STEPS].replay()
                self.turn += GRAPH_STEPS
                k -= GRAPH_STEPS
        for _ in range(k):
            self.step()

    def launches_per_step(self):
        return self.graph1s[0].kernels_per_replay if self.graph1s else None

    def probe_kernel(self):
        """One direct launch (outside any graph): the name of the kernel the dispatch picks."""
        from paper_2407_09333_b200 import _native, device

        device.hash_fixed(self.alg, self.msgs, out=self.out)
        return _native.last_kernel_name()

    def free_extra(self):
        self.graphs, self.graph1s, self.copies = [], [], [self.msgs]

    def stage_host(self, pool):
        """The same bytes in page-locked host memory (the e2e input and the oracle's)."""
        import torch

        host = pool.get("in", self.n * self.L)
        if self.n * self.L:
            torch.from_numpy(host).copy_(self.buf[: self.n * self.L])
        self.host = host.reshape(self.n, self.L)

    def e2e_step(self, out_host):
        from paper_2407_09333_b200.crypto import batch_digest

        return batch_digest(self.alg, self.host, gpus=[self.local], out=out_host)

    def e2e_pageable_step(self):
        from paper_2407_09333_b200.crypto import batch_digest

        return batch_digest(self.alg, self.pageable, gpus=[self.local])

    api = "paper_2407_09333_b200.crypto.batch_digest(pinned host array, out=pinned) -> hb_hash_fixed"

    def parity(self, full, threads):
        """Oracle digests of the staged bytes vs the device run: every row when
        `full`, else 65,536 random rows plus the first and last."""
        import oracle

        dev = self.out.cpu().numpy()
        t0 = time.perf_counter()
        if full or self.n <= 65536:
            ref = oracle.batch_fixed(self.alg, self.host, threads=threads)
            rows = self.n
            ok = bool(np.array_equal(ref, dev))
        else:
            idx = np.unique(np.concatenate([np.random.default_rng(self.seed).integers(0, self.n, 65536),
                                            [0, self.n - 1]]))
            ref = oracle.batch_fixed(self.alg, np.ascontiguousarray(self.host[idx]), threads=threads)
            rows = len(idx)
            ok = bool(np.array_equal(ref, dev[idx]))
        return rows, ok, time.perf_counter() - t0, self.n * self.L if (full or self.n <= 65536) else rows * self.L

    def config(self, world):
        what = (f"{self.alg} {self.total_msgs} x {self.L} B fixed-width, split over the GPUs" if self.scaling == "strong"
                else f"{self.alg} {self.n} x {self.L} B fixed-width per GPU")
        return {"workload": f"{what} ({self.desc})", "alg": self.alg,
                "msgs_per_gpu": self.n, "msg_len": self.L, "global_batch_msgs": self.total_msgs,
                "launch_flags": "HB_FLAG_INPUT_READY: the inputs are written before the timed region and never by "
                                "the preceding kernel, so each launch starts loading them while the previous one "
                                "drains (programmatic dependent launch)",
                "parallelism": f"message-range shards over {world} GPU(s), no collective",
                "l2": ("inputs are %.2f GiB per GPU > 2 x 126 MB L2; no flush needed" % (self.n * self.L / 2**30)
                       if len(self.copies) == 1 else
                       "%.2f MiB batch rotated over %d identical copies (%.0f MB > 2 x 126 MB L2): each step "
                       "reads a copy untouched for %d steps, from HBM" % (self.n * self.L / 2**20, len(self.copies),
                                                                            len(self.copies) * self.n * self.L / 1e6,
                                                                            len(self.copies) - 1))}


class VarlenWorkload:
    """configs[3]: n messages per GPU, lengths uniform 1..maxlen B, offsets
    layout (data bytes + u64 offsets[n+1])."""

    kind = "varlen"
    scaling = "weak"

    def __init__(self, name, alg, n, maxlen, seed, desc, rank, local, world=1):
        import torch

        from paper_2407_09333_b200 import _native, device

        self.name, self.alg, self.n, self.maxlen, self.seed, self.desc = name, alg, n, maxlen, seed, desc
        self.local = local
        self.total_msgs = world * n
        self.dlen = DLEN[alg]
        lens = np.random.default_rng(seed + 1000 * rank).integers(1, maxlen + 1, n).astype(np.uint64)
        self.off = np.zeros(n + 1, np.uint64)
        self.off[1:] = np.cumsum(lens)
        total = int(self.off[-1])
        self.total = total
        self.buf = torch.empty(total, dtype=torch.uint8, device=f"cuda:{local}")
        device.fill_random(self.buf, seed, byte_offset=8 * ((rank * total + 7) // 8))
        self.d_off = torch.from_numpy(self.off.view(np.int64)).to(f"cuda:{local}")
        self.out = torch.empty((n, self.dlen), dtype=torch.uint8, device=f"cuda:{local}")
        self.scratch = torch.empty(int(_native.lib().hb_varlen_scratch_bytes(n)), dtype=torch.uint8,
                                   device=f"cuda:{local}")
        self.msg_bytes = total
        self.total_bytes = int(reduce_sum(float(total), world, local)) if world > 1 else total
        self.alg_bytes = total + 8 * (n + 1) + n * self.dlen
        self.blocks_per_msg = (maxlen + 8) // 64 + 1
        self.blocks = int(((lens + 8) // 64 + 1).sum())
        self.h2d_bytes, self.d2h_bytes = total + 8 * (n + 1), n * self.dlen
        self.copies = [self.buf]

    def launches_per_step(self):
        return None

    def run_steps(self, k):
        for _ in range(k):
            self.step()

    def step(self):
        from paper_2407_09333_b200 import device

        # HB_FLAG_INPUT_READY: data and offsets are written before the timed region, never by
        # the preceding kernel (MD5: the length sort may start while the previous step drains)
        device.hash_varlen(self.alg, self.buf, self.d_off, out=self.out, scratch=self.scratch, offset_base=0,
                           flags=INPUT_READY)

    def probe_kernel(self):
        from paper_2407_09333_b200 import _native

        self.step()
        return _native.last_kernel_name()

    def free_extra(self):
        pass

    def stage_host(self, pool):
        import torch

        host = pool.get("in", self.total)
        torch.from_numpy(host).copy_(self.buf)
        self.host = host

    def e2e_step(self, out_host):
        from paper_2407_09333_b200.crypto import batch_digest_varlen

        return batch_digest_varlen(self.alg, self.host, self.off, gpus=[self.local], out=out_host)

    api = ("paper_2407_09333_b200.crypto.batch_digest_varlen(pinned host data, offsets, out=pinned) "
           "-> hb_hash_varlen")

    def parity(self, full, threads):
        import oracle

        dev = self.out.cpu().numpy()
        t0 = time.perf_counter()
        if full:
            ref = oracle.batch_varlen(self.alg, self.host, self.off, threads=threads)
            return self.n, bool(np.array_equal(ref, dev)), time.perf_counter() - t0, self.total
        k = min(self.n, 65536)  # a contiguous run of messages (rank-local offsets)
        ref = oracle.batch_varlen(self.alg, self.host, self.off[: k + 1], threads=threads)
        return k, bool(np.array_equal(ref, dev[:k])), time.perf_counter() - t0, int(self.off[k])

    def config(self, world):
        return {"workload": f"{self.alg} {self.n} messages of uniform 1-{self.maxlen} B per GPU, offsets layout "
                            f"({self.desc})", "alg": self.alg, "msgs_per_gpu": self.n,
                "msg_len": f"uniform 1-{self.maxlen}", "bytes_per_gpu": self.total,
                "global_batch_msgs": world * self.n,
                "parallelism": f"message-range shards over {world} GPU(s), no collective",
                "l2": "inputs are %.1f GiB per GPU >> 126 MB L2; no flush needed" % (self.total / 2**30),
                "step": "length sort (k_sort_window / k_sort_hist..scatter) + hash kernel, both timed",
                "launch_flags": "HB_FLAG_INPUT_READY: data and offsets are written before the timed region and "
                                "never by the preceding kernel (MD5's windowed sort may start while the previous "
                                "step's hash kernel drains)"}


class DecimalWorkload:
    """The paper's workload: 10^9
    messages of 9 ASCII digits, message i = zero-padded decimal of i
    (``gen_messages``).  The bytes are generated in registers inside the hash
    kernel; only digests touch HBM.  Total work is fixed, so N GPUs split the
    index range with ``partition_range`` (strong scaling)."""

    kind = "decimal"
    scaling = "strong"

    def __init__(self, name, alg, n, width, seed, desc, rank, local, world=1):
        import torch

        from paper_2407_09333_b200.passes import partition_range

        self.name, self.alg, self.width, self.seed, self.desc, self.local = name, alg, width, seed, desc, local
        self.total = self.total_msgs = n
        self.start, end = partition_range(0, n, [1.0 / world] * world)[rank]
        self.n = end - self.start
        self.dlen = DLEN[alg]
        self.out = torch.empty((self.n, self.dlen), dtype=torch.uint8, device=f"cuda:{local}")
        self.msg_bytes = self.n * width
        self.total_bytes = n * width
        self.alg_bytes = self.n * self.dlen  # message bytes never leave registers
        self.blocks_per_msg = (width + 8) // 64 + 1
        self.blocks = self.n * self.blocks_per_msg
        # ALU-pipe ops per block with the padding words constant-folded
        self.alu_ops_per_block = alu_ops_decimal(alg, width) if width + 9 <= 64 else ALU_OPS_PER_BLOCK[alg]
        self.h2d_bytes, self.d2h_bytes = 0, self.n * self.dlen
        self.copies = []

    def step(self):
        from paper_2407_09333_b200 import device

        device.hash_decimal(self.alg, self.start, self.n, self.width, device=self.local, out=self.out)

    def launches_per_step(self):
        return None

    def run_steps(self, k):
        for _ in range(k):
            self.step()

    def probe_kernel(self):
        from paper_2407_09333_b200 import _native

        self.step()
        return _native.last_kernel_name()

    def free_extra(self):
        pass

    def stage_host(self, pool):
        self.host = None  # nothing to stage: the API call takes only the index range

    def e2e_step(self, out_host):
        from paper_2407_09333_b200.crypto import hash_decimal

        return hash_decimal(self.alg, self.start, self.n, self.width, gpus=[self.local], out=out_host)

    api = "paper_2407_09333_b200.crypto.hash_decimal(start, count, 9, out=pinned) -> hb_hash_decimal"

    def parity(self, full, threads):
        import oracle

        dev = self.out.cpu().numpy()
        k = self.n if full else min(self.n, 1 << 22)
        t0 = time.perf_counter()
        ref = oracle.batch_fixed(self.alg, oracle.gen_decimal(self.start, k, self.width), threads=threads)
        return k, bool(np.array_equal(ref, dev[:k])), time.perf_counter() - t0, k * self.width

    def config(self, world):
        return {"workload": f"{self.alg} over {self.total} messages of {self.width} decimal digits, generated "
                            f"in-kernel ({self.desc})", "alg": self.alg, "msgs_total": self.total,
                "msgs_per_gpu": self.n, "msg_len": self.width, "global_batch_msgs": self.total,
                "parallelism": f"partition_range index split over {world} GPU(s), no collective",
                "l2": "no input in memory; digests %.1f GB per GPU >> 126 MB L2" % (self.n * self.dlen / 1e9)}


def make_workload(name, spec, rank, local, n_override=0, world=1):
    alg = spec[0].split(":")[-1]
    n = n_override or spec[1]
    if spec[0].startswith("decimal:"):
        return DecimalWorkload(name, alg, n, spec[2], spec[3], spec[4], rank, local, world)
    if spec[0].startswith("varlen:"):
        return VarlenWorkload(name, alg, n, spec[2], spec[3], spec[4], rank, local, world)
    return FixedWorkload(name, alg, n, spec[2], spec[3], spec[4], rank, local, world,
                         strong=spec[0].startswith("strong:"))


def copy_peak(buf_bytes: int, local: int, d2h: bool = False) -> float:
    """Pinned host <-> device copy bandwidth (GB/s) on this GPU's link, same size class."""
    import torch

    nbytes = max(1 << 20, min(buf_bytes, 1 << 30))
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{local}")
    src, dst = (d, h) if d2h else (h, d)
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3):
        dst.copy_(src, non_blocking=True)
    e.record()
    torch.cuda.synchronize()
    return 3 * nbytes / (s.elapsed_time(e) * 1e-3) / 1e9


# ------------------------------------------------------------- measuring --
class Ctx:
    def __init__(self, args, world, rank, local, sampler, pool):
        self.args, self.world, self.rank, self.local = args, world, rank, local
        self.sampler, self.pool = sampler, pool
        self.peaks, self.peak_src = load_peaks()
        import torch

        self.sms = torch.cuda.get_device_properties(local).multi_processor_count
        self.threads = len(os.sched_getaffinity(0)) or (os.cpu_count() or 1)
        self.bw = {}

    def link_peak(self, nbytes, d2h):
        key = "d2h" if d2h else "h2d"
        if key not in self.bw:
            self.bw[key] = copy_peak(nbytes, self.local, d2h=d2h)
        return self.bw[key]


def time_kernel(w, ctx, steps, warmup, min_region_ms=0.0, ramp_ms=0.0):
    """K back-to-back steps between one CUDA-event pair on the launching
    stream, after W warm-up steps, barrier + synchronize on both sides; clocks
    sampled during the region; re-measured once on hardware/thermal throttling.
    min_region_ms > 0 (suite entries): K is raised until the region lasts that
    long (estimated from the warm-up), so every entry has a clock record."""
    import torch

    from paper_2407_09333_b200 import _native

    world, rank, local = ctx.world, ctx.rank, ctx.local
    stream = torch.cuda.current_stream(local)
    t_ramp = time.perf_counter()
    while (time.perf_counter() - t_ramp) * 1e3 < ramp_ms:  # untimed: let the SM clock settle before the warm-up
        w.step()
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(warmup):
        w.step()
    e1.record(stream)
    torch.cuda.synchronize()
    if min_region_ms > 0:
        est = reduce_max(e0.elapsed_time(e1) / max(1, warmup), world, local)
        need = int(min_region_ms / max(est, 1e-4)) + 1
        if need > steps:
            steps = -(-need // GRAPH_STEPS) * GRAPH_STEPS if w.launches_per_step() else need
    barrier(world)
    torch.cuda.synchronize()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    remeasured = False
    for attempt in range(2):
        mark = ctx.sampler.begin()
        l0 = _native.launch_count()
        t_wall0 = time.perf_counter()
        t_start.record(stream)
        w.run_steps(steps)
        t_end.record(stream)
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall0
        clk = ctx.sampler.end(mark)
        launches = _native.launch_count() - l0
        # a region that saw hardware / thermal throttling is measured once more
        # (sw_power_cap is the normal state of a long integer kernel: kept, noted)
        bad = set(clk["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
        if attempt == 1 or not reduce_max(1.0 if bad else 0.0, world, local):
            break
        log(f"[rank {rank}] {w.name}: throttling during the timed region ({sorted(bad)}): re-measuring once")
        remeasured = True
        barrier(world)
        torch.cuda.synchronize()
    if remeasured:
        clk["remeasured"] = True
    if w.launches_per_step() is not None:  # CUDA-graph replays are not seen by the launch counter
        launches = w.launches_per_step() * steps
    ms_local = t_start.elapsed_time(t_end) / steps
    ms = reduce_max(ms_local, world, local)
    return ms_local, ms, launches, clk, t_wall * 1e3 / steps, steps


def pdl_overlap(kind, n, blocks_per_msg):
    """Whether consecutive flagged fixed-width steps overlap on the GPU
    (HB_FLAG_INPUT_READY + programmatic dependent launch; the engine uses PDL
    for rows of <= 128 B and for TMA grids of short messages or of at least one
    CTA per SM).  A stream of such steps is not bound by one batch's
    dependent chain -- several batches' chains run side by side -- so the
    chain bound does not enter its roofline."""
    return kind == "fixed" and (blocks_per_msg <= 17 or n >= 148 * 128)


def roofline(w, ctx, ms_local, kernel, name):
    peaks = ctx.peaks
    f_max = peaks.get("sm_max_mhz", 1965.0)
    alu_peak = ctx.sms * 64 * f_max * 1e6  # ALU-pipe lane-ops/s at max clock
    ops = getattr(w, "alu_ops_per_block", ALU_OPS_PER_BLOCK[w.alg])
    t = ms_local * 1e-3
    achieved = w.alg_bytes / t / 1e9
    t_hbm = w.alg_bytes / (peaks["hbm_gbs"] * 1e9)
    t_alu = w.blocks * ops / alu_peak
    # a batch too small to overlap its messages' dependent chains is bound by one
    # chain -- unless consecutive steps overlap (pdl_overlap), then only HBM / ALU bind
    t_chain = w.blocks_per_msg * CHAIN_CYCLES[w.alg] / (f_max * 1e6)
    chain_applies = not pdl_overlap(w.kind, getattr(w, "n", 0), w.blocks_per_msg)
    t_chain_b = t_chain if chain_applies else 0.0
    alu = {"achieved": round(w.blocks * ops / t / 1e12, 3), "peak": round(alu_peak / 1e12, 3), "unit": "Tops/s",
           "frac": round(t_alu / t, 4), "alu_ops_per_block": ops, "blocks_per_launch": w.blocks,
           "clock_mhz": f_max}
    bound = max((("hbm", t_hbm), ("alu", t_alu), ("chain", t_chain_b)), key=lambda x: x[1])[0]
    if bound == "hbm" or (bound == "chain" and t_hbm >= t_alu):
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": round(achieved / peaks["hbm_gbs"], 4)}
    else:  # integer (ALU-pipe) bound: report against the ALU-pipe roofline, HBM alongside
        roof = {"bound": "alu", "achieved": alu["achieved"], "peak": alu["peak"], "unit": "Tops/s",
                "frac": alu["frac"], "hbm_achieved_gbs": round(achieved, 1), "hbm_peak_gbs": peaks["hbm_gbs"]}
    t_roof = max(t_hbm, t_alu, t_chain_b)
    roof["max_bound"] = {"bound": bound, "t_ms": {"hbm": round(t_hbm * 1e3, 5), "alu": round(t_alu * 1e3, 5),
                                                  "chain": round(t_chain * 1e3, 5)},
                         "chain_applies": chain_applies, "frac": round(t_roof / t, 4)}
    if w.kind != "decimal":  # the survey's per-block counts assume arbitrary message words
        t_int = w.blocks * SURVEY_C_ALG[w.alg] / (ctx.sms * 128 * f_max * 1e6)
        roof["survey_issue_model"] = {
            "c_alg": SURVEY_C_ALG[w.alg], "issue_peak_tops": round(ctx.sms * 128 * f_max * 1e6 / 1e12, 3),
            "t_roof_ms": round(max(t_int, t_hbm) * 1e3, 4), "frac": round(max(t_int, t_hbm) / t, 4)}
    ncu = load_ncu(name, kernel)
    roof.update({"traffic": ncu.get("dram_bytes") if ncu else None,
                 "traffic_over_algorithmic": round(ncu["dram_bytes"] / w.alg_bytes, 4) if ncu else None,
                 "ncu_kernel": ncu.get("kernel") if ncu else None, "kernel": kernel,
                 "bytes_per_launch": w.alg_bytes, "peak_source": ctx.peak_src, "t_roof_ms": round(t_roof * 1e3, 5),
                 "alu_pipe": alu})
    return roof


def time_e2e(w, ctx, steps, warmup=1):
    """The same metric through the public API on page-locked host buffers,
    host->device copies and the digests' device->host copy inside every step."""
    import torch

    from paper_2407_09333_b200 import _native

    world, local = ctx.world, ctx.local
    out_host = ctx.pool.get("out", w.n * w.dlen).reshape(w.n, w.dlen)
    for _ in range(warmup):
        w.e2e_step(out_host)
    barrier(world)
    torch.cuda.synchronize()
    mark = ctx.sampler.begin()
    l1 = _native.launch_count()
    t0 = time.perf_counter()
    for _ in range(steps):
        res = w.e2e_step(out_host)
    t1 = time.perf_counter()
    clk = ctx.sampler.end(mark)
    launches = _native.launch_count() - l1
    barrier(world)
    e2e_ms = reduce_max((t1 - t0) * 1e3 / steps, world, local)
    ok = bool(np.array_equal(res, w.out.cpu().numpy())) if w.n <= (1 << 25) else None
    # one more call with timing= for the engine's stage breakdown (not part of the timed steps)
    tim = {}
    if w.kind == "fixed":
        from paper_2407_09333_b200.crypto import batch_digest

        batch_digest(w.alg, w.host, gpus=[local], out=out_host, timing=tim)
    elif w.kind == "varlen":
        from paper_2407_09333_b200.crypto import batch_digest_varlen

        batch_digest_varlen(w.alg, w.host, w.off, gpus=[local], out=out_host, timing=tim)
    else:
        from paper_2407_09333_b200.crypto import hash_decimal

        hash_decimal(w.alg, w.start, w.n, w.width, gpus=[local], out=out_host, timing=tim)
    d2h_dom = w.h2d_bytes < w.d2h_bytes
    bw = ctx.link_peak(max(w.h2d_bytes, w.d2h_bytes), d2h_dom)
    h2d_tot = int(reduce_sum(float(w.h2d_bytes), world, local))
    d2h_tot = int(reduce_sum(float(w.d2h_bytes), world, local))
    link_gbs = max(w.h2d_bytes, w.d2h_bytes) / (e2e_ms * 1e-3) / 1e9
    return {"value": round(w.total_bytes / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
            "h2d_bytes_per_step": h2d_tot, "d2h_bytes_per_step": d2h_tot,
            "ms_per_step": round(e2e_ms, 4), "mhash_per_s": round(w.total_msgs / (e2e_ms * 1e-3) / 1e6, 2),
            "api": w.api, "steps": steps,
            "roofline": {"bound": "pcie_d2h" if d2h_dom else "pcie_h2d", "achieved": round(link_gbs, 2),
                         "peak": round(bw, 2), "unit": "GB/s per GPU", "frac": round(link_gbs / bw, 4),
                         "peak_source": "pinned %s copy of up to 1 GiB on the same GPU, this run"
                                        % ("device->host" if d2h_dom else "host->device")},
            "engine_timing": {k: (round(v, 3) if isinstance(v, float) else v) for k, v in tim.items()},
            "clocks": clk, "gpu_launches": launches, "matches_device_run": ok}


def time_e2e_pageable(w, ctx, steps=2):
    """The reference call shape: a pageable numpy array in, a fresh digest
    array out (batch.py:274-290); the engine stages through its pinned ring."""
    import torch

    from paper_2407_09333_b200.crypto import batch_digest

    w.pageable = np.empty_like(w.host)
    np.copyto(w.pageable, w.host)
    batch_digest(w.alg, w.pageable, gpus=[ctx.local])
    barrier(ctx.world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        res = batch_digest(w.alg, w.pageable, gpus=[ctx.local])
    ms = reduce_max((time.perf_counter() - t0) * 1e3 / steps, ctx.world, ctx.local)
    ok = bool(np.array_equal(res, w.out.cpu().numpy()))
    w.pageable = None
    return {"value": round(w.total_bytes / (ms * 1e-3) / 1e9, 3), "unit": "GB/s", "ms_per_step": round(ms, 3),
            "steps": steps, "api": "paper_2407_09333_b200.crypto.batch_digest(pageable numpy array) -> new array",
            "matches_device_run": ok}


def measure(name, w, ctx, steps, warmup, e2e_steps, full_parity):
    """One config: kernel-only rate, roofline of the kernel that ran, e2e rate
    through the public API, clocks, parity against the CPU oracle."""
    import torch

    args = ctx.args
    ms_local, ms, launches, clk, wall_ms, steps = time_kernel(w, ctx, steps, warmup, min_region_ms=60.0)
    kernel = w.probe_kernel()
    torch.cuda.synchronize()
    value = w.total_bytes / (ms * 1e-3) / 1e9
    ent = {"value": round(value, 3), "unit": "GB/s", "ms_per_step": round(ms, 5),
           "mhash_per_s": round(w.total_msgs / (ms * 1e-3) / 1e6, 2), "steps": steps, "warmup": warmup,
           "scaling": w.scaling, "config": w.config(ctx.world), "clocks": clk, "gpu_launches": launches,
           "launch": f"CUDA-graph replays of {GRAPH_STEPS} back-to-back steps" if w.launches_per_step() else
                     "direct launch per step",
           "roofline": roofline(w, ctx, ms_local, kernel, name)}
    log(f"[rank {ctx.rank}] {name}: {ms_local:.5f} ms/step ({value:.1f} GB/s), wall {wall_ms:.4f} ms/step, "
        f"{launches} launches, kernel {kernel.split('(')[0]}")
    w.free_extra()
    w.stage_host(ctx.pool)
    if not args.no_e2e:
        ent["e2e"] = time_e2e(w, ctx, e2e_steps)
        log(f"[rank {ctx.rank}] {name} e2e {ent['e2e']['ms_per_step']:.3f} ms/step ({ent['e2e']['value']} GB/s)")
    rows, ok, t_cpu, nbytes = w.parity(full_parity, ctx.threads)
    rows_all = int(reduce_sum(float(rows), ctx.world, ctx.local))
    ok_all = bool(reduce_min(1.0 if ok else 0.0, ctx.world, ctx.local))
    ent["parity"] = {"rows_checked": rows_all, "rows_total": w.total_msgs, "bit_exact": ok_all,
                     "oracle": "oracle/hetoc_oracle.c (C restatement of hetoc.crypto)",
                     "scope": "every row" if full_parity else "65,536 random rows per rank (+ first/last)"}
    ent["_cpu"] = (rows, nbytes, t_cpu)
    log(f"[rank {ctx.rank}] {name} parity {rows}/{w.n} rows bit_exact={ok} ({t_cpu:.1f} s on {ctx.threads} threads)")
    return ent


def measure_latency(ctx):
    """Per-call latency of the drop-in API on tiny inputs (the reference's
    scalar digest and a 4 KiB _fast_digest-sized batch_digest)."""
    from paper_2407_09333_b200.crypto import batch_digest, digest

    out = {}
    msg = b"abc"
    small = np.frombuffer(os.urandom(4096), np.uint8).reshape(64, 64).copy()
    for _ in range(20):
        digest("sha1", msg)
        batch_digest("sha1", small)
    for key, fn in (("digest_us", lambda: digest("sha1", msg)),
                    ("batch_digest_4KiB_us", lambda: batch_digest("sha1", small))):
        ts = []
        for _ in range(200):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        out[key] = round(statistics.median(ts) * 1e6, 1)
    out["note"] = "median of 200 calls, default device set (small calls run on one GPU), pageable input"
    return out


# ---------------------------------------------------------------- our arm --
def run_ours(args):
    import torch

    from paper_2407_09333_b200 import _native

    world, rank, local = dist_setup()
    ranks = gather_objects(rank_record(rank, local), world)
    sampler = ClockSampler(local)
    sampler.start()
    pool = PinnedPool()
    ctx = Ctx(args, world, rank, local, sampler, pool)
    spec = WORKLOADS[args.workload]
    w = make_workload(args.workload, spec, rank, local, args.msgs, world)
    gather = None
    if args.gather == "p2p" and world > 1 and w.kind == "fixed":
        # fused device-side gather: each rank's kernel stores its digests into rank 0's buffer (CUDA IPC / NVLink)
        from paper_2407_09333_b200.distributed import P2PDigestGather

        gather = P2PDigestGather(w.alg, w.msgs, w.total_msgs)
        w.graphs, w.graph1s, w.copies = [], [], [w.msgs]
        w.step = gather.launch
    torch.cuda.synchronize()
    ms_local, ms, launches, clk, wall_ms, _ = time_kernel(w, ctx, args.steps, args.warmup)
    # The same kernel under sustained load: after ~1 s of back-to-back steps the
    # board sits at its 1,000 W limit and an issue-bound kernel runs at a lower
    # SM clock (tools/ab_power.py).  Reported beside the headline, not instead.
    sustained = None
    if w.kind in ("fixed", "varlen") and gather is None:
        s_local, s_ms, _, s_clk, _, s_steps = time_kernel(w, ctx, max(60, args.steps), 0, ramp_ms=1000.0)
        s_val = w.total_bytes / (s_ms * 1e-3) / 1e9
        sustained = {"value": round(s_val, 2), "unit": "GB/s", "ms_per_step": round(s_ms, 4), "steps": s_steps,
                     "after_ms_of_load": 1000, "clocks": s_clk,
                     "note": "K back-to-back steps after 1 s of untimed load: the board at its power limit"}
    if gather is not None:  # the gather wrote into rank 0's buffer; refill the local digests for the checks below
        from paper_2407_09333_b200 import device as _device

        _device.hash_fixed(w.alg, w.msgs, out=w.out)
        torch.cuda.synchronize()
    kernel = w.probe_kernel()
    value = w.total_bytes / (ms * 1e-3) / 1e9
    log(f"[rank {rank}] headline {w.name}: {ms_local:.4f} ms/step, wall {wall_ms:.3f} ms/step, {launches} launches")
    roof = roofline(w, ctx, ms_local, kernel, args.workload)
    if sustained is not None and roof and roof.get("peak"):
        sustained["roofline_frac"] = round(roof["achieved"] * ms_local / sustained["ms_per_step"] / roof["peak"], 4)
    w.free_extra()
    w.stage_host(pool)
    e2e = e2e_pageable = None
    if not args.no_e2e:
        e2e = time_e2e(w, ctx, args.e2e_steps or min(args.steps, 3 if w.kind == "decimal" else 10))
        if w.kind == "fixed":
            e2e_pageable = time_e2e_pageable(w, ctx)
        log(f"[rank {rank}] e2e {e2e['ms_per_step']:.1f} ms/step; pageable "
            f"{e2e_pageable['ms_per_step'] if e2e_pageable else '-'} ms/step")
    full = world == 1 and not args.sample_parity
    rows, ok, t_cpu, nbytes = w.parity(full, ctx.threads)
    rows_all = int(reduce_sum(float(rows), world, local))
    ok_all = bool(reduce_min(1.0 if ok else 0.0, world, local))
    parity = {"rows_checked": rows_all, "rows_total": w.total_msgs, "bit_exact": ok_all,
              "scope": "every row" if full else "65,536 random rows per rank (+ first/last)"}
    cpu = None
    if rank == 0 and world == 1:
        cpu = {"value": round(nbytes / t_cpu / 1e9, 4), "unit": "GB/s", "cores": ctx.threads, "kind": "port",
               "sample": f"{'all' if full else rows} of the {w.n} messages (same bytes), oracle/hetoc_oracle.c on "
                         f"{ctx.threads} threads, {t_cpu:.2f} s", "mhash_per_s": round(rows / t_cpu / 1e6, 4),
               "host_cpu": cpu_info()}
    latency = measure_latency(ctx) if rank == 0 and not args.no_e2e else None
    head = {"config": w.config(world), "scaling": w.scaling, "total_msgs": w.total_msgs, "kind": w.kind,
            "seed": w.seed}
    del w
    torch.cuda.empty_cache()

    configs = {}
    if args.configs == "all":
        t_suite = time.perf_counter()
        for name, sspec in suite_specs():
            if world == 1 and name in ("C5_md5_1024x16777216",):  # == the headline at N=1
                configs[name] = {"same_as": "headline (configs[1])"}
                continue
            if world == 1 and name == "C5_sm3_1024x16777216":  # == C3 at N=1
                configs[name] = {"same_as": "C3_sm3_1k"}
                continue
            sw = make_workload(name, sspec, rank, local, 0, world)
            steps = max(3, min(args.steps, 20))
            configs[name] = measure(name, sw, ctx, steps, max(3, min(args.warmup, 5)),
                                    args.suite_e2e_steps, world == 1 and not args.sample_parity)
            cpu_rows, cpu_bytes, cpu_t = configs[name].pop("_cpu")
            if rank == 0 and world == 1:
                configs[name]["cpu_oracle"] = {"value": round(cpu_bytes / cpu_t / 1e9, 4), "unit": "GB/s",
                                               "cores": ctx.threads, "seconds": round(cpu_t, 2)}
            del sw
            torch.cuda.empty_cache()
        log(f"[rank {rank}] suite of {len(configs)} configs in {time.perf_counter() - t_suite:.1f} s")
    sampler.stop()
    pool.close()
    if rank == 0:
        if roof and clk and "sw_power_cap" in (clk.get("reasons") or []) and clk.get("sm_mhz"):
            # The board reached its power limit (1,000 W on this pool, tools/ab_power.py): the
            # SM clock fell below its maximum, so an issue-bound kernel runs slower than the
            # same kernel at full clock.  Reported, not corrected.
            roof["power_note"] = (f"sw_power_cap during the timed region: SM clock median {clk['sm_mhz']:.0f} MHz "
                                  f"of {clk.get('sm_max_mhz') or 1965:.0f}; the ALU-pipe and chain bounds above "
                                  "assume the maximum clock")
        line = {"metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
                "higher_is_better": True, "scaling": head["scaling"], "vs_baseline": None, "dtype": "u32",
                "data": ("paper workload: decimal messages generated in-kernel" if head["kind"] == "decimal" else
                         f"synthetic: counter-based splitmix64 bytes (seed {head['seed']}), generated on device"),
                "config": dict(head["config"], gather="fused P2P into rank 0 (CUDA IPC)" if gather is not None
                               else "none", host_affinity=HOST["affinity"]),
                "mhash_per_s": round(head["total_msgs"] / (ms * 1e-3) / 1e6, 2), "clocks": clk,
                "e2e": e2e, "e2e_pageable": e2e_pageable, "latency": latency, "sustained": sustained,
                "gpu_launches": launches, "roofline": roof, "cpu_baseline": cpu, "parity": parity,
                "ranks": ranks, "library": library_info(), "configs": configs}
        print(json.dumps(line), flush=True)
    if gather is not None:
        gather.close()
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


# --------------------------------------------------------- reference arm --
def numpy_reference(alg, data, budget_s):
    """The reference's own batch_digest (hetoc.crypto, numpy) as installed in
    baseline/_ref, when present: 1 core as-is, and a process pool over the
    np.linspace split of batch.py:305 on every host core -- a stated baseline
    beside the C port (SURVEY §8(d) CPU reference timing 1-2)."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "hetoc")):
        return {"unavailable": "baseline/_ref not installed on this box"}
    code = r'''
import json, os, sys, time
import numpy as np
from multiprocessing import Pool
sys.path.insert(0, sys.argv[1])
from hetoc.crypto import batch_digest
alg, n, L, seed, budget = sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]), float(sys.argv[6])
rng = np.random.default_rng(seed)
data = rng.integers(0, 256, (n, L), dtype=np.uint8)
t0 = time.perf_counter(); batch_digest(alg, data[:4096]); t1 = time.perf_counter()
per_row = (t1 - t0) / 4096
rows1 = int(max(4096, min(n, budget / 2 / per_row)))
t0 = time.perf_counter(); batch_digest(alg, data[:rows1]); one = time.perf_counter() - t0
cores = len(os.sched_getaffinity(0))
rowsp = int(max(cores * 4096, min(n, budget / 2 / per_row * cores)))
def part(b):
    return batch_digest(alg, data[b[0]:b[1]])
bounds = np.linspace(0, rowsp, cores + 1, dtype=np.int64)
with Pool(cores) as p:
    p.map(part, [(0, 1)] * cores)
    t0 = time.perf_counter(); p.map(part, list(zip(bounds[:-1], bounds[1:]))); pool = time.perf_counter() - t0
res = {"one_core": {"value": rows1 * L / one / 1e9, "rows": rows1, "seconds": one},
       "pool": {"value": rowsp * L / pool / 1e9, "rows": rowsp, "seconds": pool, "cores": cores}}
# hash_batch as-is over the same rows with threads = cores (thread pool over
# the np.linspace split, list[Digest] built), SURVEY §8(d) CPU timing 1
from hetoc.crypto import MessageBatch, hash_batch
mb = MessageBatch(rowsp, L, data[:rowsp].tobytes())
t0 = time.perf_counter(); hash_batch(alg, mb, threads=cores); hb = time.perf_counter() - t0
res["hash_batch_threads"] = {"value": rowsp * L / hb / 1e9, "rows": rowsp, "seconds": hb, "threads": cores}
# the SHA-1 accel path (hashlib / SHA-NI, batch.py:266-271) on SHA-1 rows of the same shape, timing 3
t0 = time.perf_counter(); batch_digest("sha1", data[:4096], accel=True); per = (time.perf_counter() - t0) / 4096
rowsa = int(max(4096, min(n, budget / 6 / per)))
t0 = time.perf_counter(); batch_digest("sha1", data[:rowsa], accel=True); a1 = time.perf_counter() - t0
mba = MessageBatch(rowsa, L, data[:rowsa].tobytes())
t0 = time.perf_counter(); hash_batch("sha1", mba, threads=cores, accel=True); at = time.perf_counter() - t0
res["sha1_accel"] = {"one_core": rowsa * L / a1 / 1e9, "hash_batch_threads": rowsa * L / at / 1e9, "rows": rowsa}
print(json.dumps(res))
'''
    try:
        n, L = data
        out = subprocess.run([sys.executable, "-c", code, ref_dir, alg, str(n), str(L), "7", str(budget_s)],
                             capture_output=True, text=True, timeout=budget_s * 4 + 120)
        r = json.loads(out.stdout.strip().splitlines()[-1])
        return {"one_core_gbs": round(r["one_core"]["value"], 4), "pool_gbs": round(r["pool"]["value"], 4),
                "pool_cores": r["pool"]["cores"],
                "hash_batch_threads_gbs": round(r["hash_batch_threads"]["value"], 4),
                "sha1_accel_gbs": {"one_core": round(r["sha1_accel"]["one_core"], 4),
                                   "hash_batch_threads": round(r["sha1_accel"]["hash_batch_threads"], 4),
                                   "rows": r["sha1_accel"]["rows"],
                                   "api": "hetoc.crypto.batch_digest / hash_batch(..., accel=True), SHA-1 rows "
                                          "of the same shape (hashlib, SHA-NI on this host)"},
                "sample": f"{r['one_core']['rows']} rows on 1 core, {r['pool']['rows']} rows over a process pool "
                          f"(np.linspace split, batch.py:305) of {L} B random messages",
                "api": "hetoc.crypto.batch_digest (baseline/_ref, unmodified reference)"}
    except Exception as e:
        return {"unavailable": f"reference run failed: {type(e).__name__}: {str(e)[:200]}"}


def run_reference(args):
    """The reference algorithm's CPU implementation on all host threads: the
    oracle port of hetoc.crypto (the reference is pure Python/numpy, 10-50x
    slower than the port), each step the FULL batch of the headline config
    when the whole --steps K --warmup W run fits --ref-budget-seconds, else a
    bounded sample; the numpy reference itself is timed beside it when
    baseline/_ref exists."""
    import oracle

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    spec = WORKLOADS[args.workload]
    alg = spec[0].split(":")[-1]
    n = args.msgs or spec[1]
    seed, cfg_desc = spec[3], spec[4]
    threads = len(os.sched_getaffinity(0)) or (os.cpu_count() or 1)
    total_steps = max(1, args.steps + args.warmup)
    step_budget = args.ref_budget_seconds / total_steps
    strong = spec[0].startswith(("strong:", "decimal:"))
    # the same per-GPU work as our arm at N GPUs: weak configs n per GPU (one GPU's share here), strong the whole batch / N
    n_cpu = n if not strong else -(-n // world)
    if spec[0].startswith("decimal:"):
        width = spec[2]
        per = cpu_rate_probe(lambda k: oracle.batch_fixed(alg, oracle.gen_decimal(0, k, width), threads=1), 1 << 14)
        rows = min(n_cpu, max(threads * 16, int(step_budget * threads / per)))
        data = oracle.gen_decimal(0, rows, width)
        run = lambda: oracle.batch_fixed(alg, data, threads=threads)  # noqa: E731
        nbytes = rows * width
        config = {"workload": f"{alg} over {n} messages of {width} decimal digits ({cfg_desc})", "alg": alg,
                  "msgs_total": n, "msg_len": width}
        np_ref = None
    elif spec[0].startswith("varlen:"):
        maxlen = spec[2]
        lens = np.random.default_rng(seed).integers(1, maxlen + 1, n).astype(np.uint64)
        off = np.zeros(n + 1, np.uint64)
        off[1:] = np.cumsum(lens)
        probe_k = min(n, 2048)
        probe = oracle.fill_random(int(off[probe_k]), seed)
        per = cpu_rate_probe(lambda k: oracle.batch_varlen(alg, probe, off[: k + 1], threads=1), probe_k)
        rows = min(n, max(threads * 16, int(step_budget * threads / per)))
        data = oracle.fill_random(int(off[rows]), seed)
        run = lambda: oracle.batch_varlen(alg, data, off[: rows + 1], threads=threads)  # noqa: E731
        nbytes = int(off[rows])
        config = {"workload": f"{alg} {n} messages of uniform 1-{maxlen} B per GPU, offsets layout ({cfg_desc})",
                  "alg": alg, "msgs_per_gpu": n, "msg_len": f"uniform 1-{maxlen}"}
        np_ref = None
    else:
        L = spec[2]
        probe = oracle.fill_random(2048 * L, 123).reshape(2048, L)
        per = cpu_rate_probe(lambda k: oracle.batch_fixed(alg, probe[:k], threads=1), 2048)
        rows = min(n_cpu, max(threads * 16, int(step_budget * threads / per * 0.9)))
        data = oracle.fill_random(rows * L, seed).reshape(rows, L)
        run = lambda: oracle.batch_fixed(alg, data, threads=threads)  # noqa: E731
        nbytes = rows * L
        what = (f"{alg} {n} x {L} B fixed-width, split over the GPUs" if strong
                else f"{alg} {n} x {L} B fixed-width per GPU")
        config = {"workload": f"{what} ({cfg_desc})", "alg": alg, "msgs_per_gpu": n_cpu, "msg_len": L}
        np_ref = numpy_reference(alg, (min(n, 1 << 20), L), args.numpy_ref_seconds) if not args.no_numpy_ref else None
    same = rows == n_cpu
    for _ in range(args.warmup):
        run()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    value = nbytes / t / 1e9
    sample = (f"the full batch ({rows} messages = one GPU's share at N={world}) per step" if same else
              f"{rows} of the {n_cpu} messages per step (bounded: --ref-budget-seconds {args.ref_budget_seconds})")
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3), "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "u32",
            "data": "paper workload: decimal messages (gen_messages)" if spec[0].startswith("decimal:") else
                    f"synthetic: counter-based splitmix64 bytes (seed {seed})", "config": config,
            "same_config": same,
            "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": threads, "kind": "port",
                             "sample": f"{sample}, oracle/hetoc_oracle.c (C restatement of hetoc.crypto) "
                                       f"on {threads} threads", "host_cpu": cpu_info()},
            "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "mhash_per_s": round(rows / t / 1e6, 4), "reference_numpy": np_ref}
    print(json.dumps(line), flush=True)


def cpu_rate_probe(fn, k):
    """Seconds per message of fn on one thread (k messages)."""
    fn(min(k, 64))
    t0 = time.perf_counter()
    fn(k)
    return max((time.perf_counter() - t0) / k, 1e-9)


# -------------------------------------------------------------- launching --
def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def self_launch(args):
    """--gpus N is authoritative: without WORLD_SIZE, N > 1 relaunches this
    script under torch.distributed.run (one rank per GPU); returns the exit
    code, or None when this process is already the right one."""
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is not None:
        if int(env_world) != args.gpus:
            log(f"error: --gpus {args.gpus} but WORLD_SIZE={env_world}")
            return 2
        return None
    if args.gpus <= 1:
        return None
    if _BACKEND != "gloo" and not args.dry_run and args.impl == "ours":
        try:
            import torch

            visible = torch.cuda.device_count()
        except Exception:
            visible = 0
        if visible < args.gpus:
            log(f"error: --gpus {args.gpus} needs {args.gpus} visible CUDA devices, found {visible} "
                "(set HB_BENCH_BACKEND=gloo to share GPUs between ranks for testing)")
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    log(f"launching {args.gpus} ranks: {' '.join(cmd)}")
    return subprocess.call(cmd)


def run_dry(args):
    """--dry-run: the launch path only (process group, per-rank records), no
    GPU work -- the CPU test of the --gpus N launch."""
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo")
    recs = gather_objects({"rank": rank, "local_rank": int(os.environ.get("LOCAL_RANK", "0")), "pid": os.getpid()},
                          world)
    if rank == 0:
        print(json.dumps({"dry_run": True, "impl": args.impl, "n_gpus": world, "ranks": recs}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="md5_1k")
    ap.add_argument("--configs", choices=["all", "none"], default="all",
                    help="measure every other BASELINE config in the same run (default workload only)")
    ap.add_argument("--msgs", type=int, default=0, help="override the message count (per GPU; total for strong-scaling workloads)")
    ap.add_argument("--e2e-steps", type=int, default=0)
    ap.add_argument("--suite-e2e-steps", type=int, default=3)
    ap.add_argument("--sample-parity", action="store_true", help="row sample instead of every row at N=1")
    ap.add_argument("--ref-budget-seconds", type=float, default=150.0,
                    help="--impl reference: upper bound on the whole run's CPU time")
    ap.add_argument("--numpy-ref-seconds", type=float, default=20.0)
    ap.add_argument("--no-numpy-ref", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--gather", choices=["none", "p2p"], default="none",
                    help="N>1: fused device-side digest gather into rank 0 (hash kernels store over NVLink)")
    ap.add_argument("--dry-run", action="store_true")
    args = ap.parse_args()
    rc = self_launch(args)
    if rc is not None:
        sys.exit(rc)
    if args.dry_run:
        run_dry(args)
        return
    if args.warmup < 3 and args.impl == "ours":
        log("note: timing rules want >= 3 warm-up steps")
    if args.workload != "md5_1k" or args.msgs:
        args.configs = "none"
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
