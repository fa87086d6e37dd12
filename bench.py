#!/usr/bin/env python
"""Benchmark of the B200 batched-hash engine (the BASELINE.json north-star path).

Default workload = BASELINE.json configs[1]: MD5 over 2^24 random 1 KiB
messages per GPU (weak scaling under torchrun: rank r hashes global messages
[r*2^24, (r+1)*2^24)).  Prints ONE JSON line (rank 0):

  value        kernel-only GB/s of message bytes, inputs resident in HBM: one
               CUDA-event pair on the launching stream around K back-to-back
               steps, max over ranks; bytes summed over ranks
  e2e          the same metric through the public API (crypto.batch_digest /
               batch_digest_varlen / hash_decimal on pinned host arrays):
               H2D + kernels + D2H every step; its roofline is the pinned-copy
               bandwidth measured in the same run
  roofline     the dominant kernel vs the HBM copy peak or the ALU-pipe peak
  cpu_baseline the CPU oracle (C port of the reference algorithm) on a bounded
               sample of the same bytes, all host threads; its digests are also
               compared bit-for-bit with the GPU's for that sample

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--gather none|p2p]
                  [--workload md5_1k|sha1_1k|sm3_1k|sha1_64|varlen_{md5,sha1,sm3}|paper_{sha1,md5,sm3}]
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

WORKLOADS = {
    # name: (alg | "varlen:"alg, n per GPU, msg_len | max varlen length, seed, BASELINE config)
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
# $HB_BENCH_BACKEND=gloo (test hook): run the N>1 path with ranks sharing the
# visible GPUs round-robin -- NCCL needs one GPU per rank, gloo does not -- so
# the multi-rank bench (sharding, max-over-ranks timing, the fused P2P gather)
# can be exercised on a one-GPU box.  Production runs use NCCL, one GPU per rank.
_BACKEND = os.environ.get("HB_BENCH_BACKEND", "nccl")


HOST_AFFINITY = ["unbound (one process, N=1)"]


def dist_setup(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if _BACKEND == "gloo":
            local = local % torch.cuda.device_count()
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        # host side next to this rank's GPU (pinned e2e buffers are allocated later)
        from paper_2407_09333_b200.device import bind_host_to_gpu

        cores = bind_host_to_gpu(local)
        HOST_AFFINITY[0] = f"{len(cores)} GPU-local cores (NVML)" if cores else "unbound (NVML gave no mask)"
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

    t = torch.tensor([x], dtype=torch.float64, device="cpu" if _BACKEND == "gloo" else f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


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


def load_ncu_traffic(workload: str):
    """dram bytes per launch of the dominant kernel from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    k = d.get(workload)
    return k.get("dram_bytes") if k else None


# ------------------------------------------------------------ CPU oracle --
def cpu_sample_rows(alg: str, L: int, n: int, threads: int, target_s: float):
    """Pick a sample size giving ~target_s seconds of wall time on `threads` threads."""
    import oracle

    probe = oracle.fill_random(min(n, 2048) * L, 123).reshape(-1, L)
    t0 = time.perf_counter()
    oracle.batch_fixed(alg, probe, threads=1)
    t = time.perf_counter() - t0
    per_row = max(t / probe.shape[0], 1e-9)
    rows = int(target_s * threads / per_row)
    rows = max(threads * 16, min(n, rows))
    return rows


# -------------------------------------------------------------- workloads --
class FixedWorkload:
    """n messages of L bytes per GPU, (n, L) row-major (configs[0..2], [4])."""

    kind = "fixed"

    def __init__(self, name, alg, n, L, seed, desc, rank, local, world=1, strong=False):
        import torch

        from paper_2407_09333_b200 import device
        from paper_2407_09333_b200.passes import partition_range

        self.name, self.alg, self.L, self.seed, self.desc = name, alg, L, seed, desc
        self.scaling = "strong" if strong else "weak"
        if strong:  # configs[2]: the SAME 2^24 messages split over the GPUs by message range
            lo, hi = partition_range(0, n, [1.0 / world] * world)[rank]
            self.total_msgs = n
        else:  # n messages per GPU: rank r hashes global messages [r*n, (r+1)*n)
            lo, hi = rank * n, (rank + 1) * n
            self.total_msgs = world * n
        n = hi - lo
        self.n, self.lo = n, lo
        self.dlen = DLEN[alg]
        self.buf = torch.empty(n * L, dtype=torch.uint8, device=f"cuda:{local}")
        device.fill_random(self.buf, seed, byte_offset=lo * L)
        self.msgs = self.buf.view(n, L)
        self.out = torch.empty((n, self.dlen), dtype=torch.uint8, device=f"cuda:{local}")
        self.msg_bytes = n * L
        self.alg_bytes = n * (L + self.dlen)  # message bytes read once + digests written once
        self.blocks = n * ((L + 8) // 64 + 1)
        self.h2d_bytes, self.d2h_bytes = n * L, n * self.dlen
        # Small batches (a few microseconds of GPU work, configs[0]) are launched
        # as a CUDA-graph replay so the host call overhead does not idle the GPU.
        # A step of a small batch is a few microseconds of GPU work, less than a
        # launch from Python: those steps run as CUDA-graph replays of
        # GRAPH_STEPS back-to-back passes (each pass hashes the whole batch).
        # A batch smaller than 2x L2 would be re-read from L2 by back-to-back
        # steps: it is rotated over enough identical copies (a multiple of
        # GRAPH_STEPS, >= 2 x 126 MB in total) that every step reads a copy
        # last touched >= 63 steps earlier, i.e. from HBM.
        self.copies = [self.msgs]
        if n * L and n * L < L2_DEFEAT_BYTES:
            r = -(-L2_DEFEAT_BYTES // (n * L))
            r = -(-r // GRAPH_STEPS) * GRAPH_STEPS
            self.copies += [self.msgs.clone() for _ in range(r - 1)]
        self.turn = 0
        self.graphs, self.graph1s = [], []
        if n * L <= (64 << 20):
            # GRAPH_STEPS consecutive copies per replayed graph, one single-pass graph per copy for remainders
            for j in range(0, len(self.copies), GRAPH_STEPS):
                group = self.copies[j:j + GRAPH_STEPS]
                reps = GRAPH_STEPS // len(group) if len(group) < GRAPH_STEPS else 1
                self.graphs.append(device.FixedHashGraph(alg, group, self.out, repeats=reps))
            self.graph1s = [device.FixedHashGraph(alg, c, self.out) for c in self.copies]
        self.graph = self.graphs[0] if self.graphs else None  # kept for callers that test for graph mode

    def step(self):
        from paper_2407_09333_b200 import device

        i = self.turn % len(self.copies)
        self.turn += 1
        if self.graph1s:
            self.graph1s[i].replay()
        else:
            device.hash_fixed(self.alg, self.copies[i], out=self.out)

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
        else:
            for _ in range(k):
                self.step()

    def launches_per_step(self):
        return self.graph1s[0].kernels_per_replay if self.graph1s else None

    def host_inputs(self, lib):
        import ctypes

        import numpy as np

        hp = lib.hb_alloc_pinned(self.n * self.L)
        if not hp:
            return None
        host = np.ctypeslib.as_array(ctypes.cast(hp, ctypes.POINTER(ctypes.c_uint8)),
                                     shape=(self.n * self.L,)).reshape(self.n, self.L)
        import torch

        torch.from_numpy(host.reshape(-1)).copy_(self.buf)  # same bytes as the device-resident run
        self._host = host
        return hp

    def e2e_step(self, local, tim):
        from paper_2407_09333_b200.crypto import batch_digest

        return batch_digest(self.alg, self._host, gpus=[local], timing=tim, out=self._out_host)

    def config(self, world):
        what = (f"{self.alg} {self.total_msgs} x {self.L} B fixed-width, split over the GPUs" if self.scaling == "strong"
                else f"{self.alg} {self.n} x {self.L} B fixed-width per GPU")
        return {"workload": f"{what} ({self.desc})", "alg": self.alg,
                "msgs_per_gpu": self.n, "msg_len": self.L, "global_batch_msgs": self.total_msgs,
                "parallelism": f"message-range shards over {world} GPU(s), no collective",
                "l2": ("inputs are %.1f GiB per GPU >> 126 MB L2; no flush needed" % (self.n * self.L / 2**30)
                       if len(self.copies) == 1 else
                       "%.1f MiB batch rotated over %d identical copies (%.0f MB > 2 x 126 MB L2): each step "
                       "reads a copy untouched for %d steps, from HBM" % (self.n * self.L / 2**20, len(self.copies),
                                                                            len(self.copies) * self.n * self.L / 1e6,
                                                                            len(self.copies) - 1))}

    def kernel_name(self):
        return "k_fixed_tma_ws<%s>" % self.alg

    def cpu_sample(self, threads, target_s):
        import oracle

        rows = cpu_sample_rows(self.alg, self.L, self.n, threads, target_s)
        sample = self.buf[: rows * self.L].cpu().numpy().reshape(rows, self.L)
        t0 = time.perf_counter()
        ref = oracle.batch_fixed(self.alg, sample, threads=threads)
        t = time.perf_counter() - t0
        ok = bool(np.array_equal(ref, self.out[:rows].cpu().numpy()))
        return rows, rows * self.L, t, ok, f"first {rows} of the {self.n} x {self.L} B messages (same bytes)"


GRAPH_STEPS = 10
L2_DEFEAT_BYTES = 2 * 126 * 10**6  # twice the B200's 126 MB L2


class VarlenWorkload:
    """configs[3]: n messages per GPU, lengths uniform 1..maxlen B, offsets
    layout (data bytes + u64 offsets[n+1])."""

    kind = "varlen"

    def __init__(self, name, alg, n, maxlen, seed, desc, rank, local, world=1):
        import numpy as np
        import torch

        from paper_2407_09333_b200 import _native, device

        self.name, self.alg, self.n, self.maxlen, self.seed, self.desc = name, alg, n, maxlen, seed, desc
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
        self.alg_bytes = total + 8 * (n + 1) + n * self.dlen
        self.blocks = int(((lens + 8) // 64 + 1).sum())
        self.h2d_bytes, self.d2h_bytes = total + 8 * (n + 1), n * self.dlen

    def launches_per_step(self):
        return None

    def run_steps(self, k):
        for _ in range(k):
            self.step()

    def step(self):
        from paper_2407_09333_b200 import device

        device.hash_varlen(self.alg, self.buf, self.d_off, out=self.out, scratch=self.scratch, offset_base=0)

    def host_inputs(self, lib):
        import ctypes

        import numpy as np
        import torch

        hp = lib.hb_alloc_pinned(self.total)
        if not hp:
            return None
        self._host = np.ctypeslib.as_array(ctypes.cast(hp, ctypes.POINTER(ctypes.c_uint8)), shape=(self.total,))
        torch.from_numpy(self._host).copy_(self.buf)
        return hp

    def e2e_step(self, local, tim):
        from paper_2407_09333_b200.crypto import batch_digest_varlen

        return batch_digest_varlen(self.alg, self._host, self.off, gpus=[local], timing=tim, out=self._out_host)

    def config(self, world):
        return {"workload": f"{self.alg} {self.n} messages of uniform 1-{self.maxlen} B per GPU, offsets layout "
                            f"({self.desc})", "alg": self.alg, "msgs_per_gpu": self.n,
                "msg_len": f"uniform 1-{self.maxlen}", "bytes_per_gpu": self.total,
                "global_batch_msgs": world * self.n,
                "parallelism": f"message-range shards over {world} GPU(s), no collective",
                "l2": "inputs are %.1f GiB per GPU >> 126 MB L2; no flush needed" % (self.total / 2**30)}

    def kernel_name(self):
        return "k_varlen16<%s>" % self.alg

    def cpu_sample(self, threads, target_s):
        import oracle

        k = min(self.n, max(threads * 16, int(self.n * min(1.0, target_s / 8.0))))
        data = self.buf[: int(self.off[k])].cpu().numpy()
        t0 = time.perf_counter()
        ref = oracle.batch_varlen(self.alg, data, self.off[: k + 1], threads=threads)
        t = time.perf_counter() - t0
        ok = bool(np.array_equal(ref, self.out[:k].cpu().numpy()))
        return k, int(self.off[k]), t, ok, f"first {k} of the {self.n} messages (same bytes)"


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
        self.alg_bytes = self.n * self.dlen  # message bytes never leave registers
        self.blocks = self.n * ((width + 8) // 64 + 1)
        # ALU-pipe ops per block with the padding words constant-folded
        self.alu_ops_per_block = alu_ops_decimal(alg, width) if width + 9 <= 64 else ALU_OPS_PER_BLOCK[alg]
        self.h2d_bytes, self.d2h_bytes = 0, self.n * self.dlen

    def step(self):
        from paper_2407_09333_b200 import device

        device.hash_decimal(self.alg, self.start, self.n, self.width, device=self.local, out=self.out)

    def launches_per_step(self):
        return None

    def run_steps(self, k):
        for _ in range(k):
            self.step()

    def host_inputs(self, lib):
        return -1  # nothing to stage: the API call takes only the index range

    def e2e_step(self, local, tim):
        from paper_2407_09333_b200.crypto import hash_decimal

        return hash_decimal(self.alg, self.start, self.n, self.width, gpus=[local], timing=tim, out=self._out_host)

    def config(self, world):
        return {"workload": f"{self.alg} over {self.total} messages of {self.width} decimal digits, generated "
                            f"in-kernel ({self.desc})", "alg": self.alg, "msgs_total": self.total,
                "msgs_per_gpu": self.n, "msg_len": self.width, "global_batch_msgs": self.total,
                "parallelism": f"partition_range index split over {world} GPU(s), no collective",
                "l2": "no input in memory; digests %.1f GB per GPU >> 126 MB L2" % (self.n * self.dlen / 1e9)}

    def kernel_name(self):
        return "k_decimal<%s, %d>" % (self.alg, self.width)

    def cpu_sample(self, threads, target_s):
        import oracle

        from paper_2407_09333_b200.crypto import gen_messages

        k = min(self.n, cpu_sample_rows(self.alg, self.width, self.n, threads, target_s))
        rows = gen_messages(self.start, k, self.width).as_array()
        t0 = time.perf_counter()
        ref = oracle.batch_fixed(self.alg, rows, threads=threads)
        t = time.perf_counter() - t0
        ok = bool(np.array_equal(ref, self.out[:k].cpu().numpy()))
        return k, k * self.width, t, ok, f"first {k} of the {self.n} decimal messages (same bytes)"


def make_workload(name, rank, local, n_override=0, world=1):
    spec = WORKLOADS[name]
    alg = spec[0].split(":")[-1]
    n = n_override or spec[1]
    if spec[0].startswith("decimal:"):
        return DecimalWorkload(name, alg, n, spec[2], spec[3], spec[4], rank, local, world)
    if spec[0].startswith("varlen:"):
        return VarlenWorkload(name, alg, n, spec[2], spec[3], spec[4], rank, local, world)
    return FixedWorkload(name, alg, n, spec[2], spec[3], spec[4], rank, local, world,
                         strong=spec[0].startswith("strong:"))


def h2d_peak(buf_bytes: int, local: int, d2h: bool = False) -> float:
    """Pinned host <-> device copy bandwidth (GB/s) on this GPU's link, same size class."""
    import torch

    nbytes = min(buf_bytes, 1 << 30)
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


# ---------------------------------------------------------------- our arm --
def run_ours(args):
    import numpy as np  # noqa: F401
    import torch

    from paper_2407_09333_b200 import _native

    world, rank, local = dist_setup(args)
    w = make_workload(args.workload, rank, local, args.msgs, world)
    alg = w.alg
    gather = None
    if args.gather == "p2p" and world > 1 and w.kind == "fixed":
        # fused device-side gather: each rank's kernel stores its digests into rank 0's buffer (CUDA IPC / NVLink)
        from paper_2407_09333_b200.distributed import P2PDigestGather

        gather = P2PDigestGather(alg, w.msgs, w.total_msgs)
        w.graph, w.graphs, w.graph1s, w.copies = None, [], [], [w.msgs]
        w.step = gather.launch
    stream = torch.cuda.current_stream(local)
    sampler = ClockSampler(local)
    sampler.start()
    torch.cuda.synchronize()

    for _ in range(args.warmup):
        w.step()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    # One event pair brackets the K back-to-back steps (whole-job throughput:
    # per-step event pairs would add a launch latency, ~9 us on this box, to
    # every small step); a few per-step pairs after it give the spread.
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    remeasured = False
    for attempt in range(2):
        sampler.lines.clear()
        l0 = _native.launch_count()
        sampler.active = True
        t_wall0 = time.perf_counter()
        t_start.record(stream)
        w.run_steps(args.steps)
        t_end.record(stream)
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall0
        sampler.active = False
        launches = _native.launch_count() - l0
        # a region that saw hardware / thermal throttling is measured once more
        # (sw_power_cap is the normal state of a long integer kernel: kept, noted)
        bad = set(sampler.summary()["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
        if attempt == 1 or not reduce_max(1.0 if bad else 0.0, world, local):
            break
        log(f"[rank {rank}] throttling during the timed region ({sorted(bad)}): re-measuring once")
        remeasured = True
        barrier(world)
        torch.cuda.synchronize()
    if gather is not None:  # the gather wrote into rank 0's buffer; refill the local digests for the checks below
        from paper_2407_09333_b200 import device as _device

        _device.hash_fixed(alg, w.msgs, out=w.out)
        torch.cuda.synchronize()
    if w.launches_per_step() is not None:  # CUDA-graph replays are not seen by the launch counter
        launches = w.launches_per_step() * args.steps
    barrier(world)
    ms_local = t_start.elapsed_time(t_end) / args.steps
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(3)]
    for s, e in evs:  # spread of single steps (not part of the timed value)
        s.record(stream)
        w.step()
        e.record(stream)
    torch.cuda.synchronize()
    per_step = [s.elapsed_time(e) for s, e in evs]
    ms = reduce_max(ms_local, world, local)
    total_msgs = w.total_msgs  # messages hashed by all ranks in one step
    total_bytes = w.msg_bytes * world if w.kind == "varlen" else total_msgs * (w.L if w.kind == "fixed" else w.width)
    value = total_bytes / (ms * 1e-3) / 1e9
    mhash = total_msgs / (ms * 1e-3) / 1e6
    log(f"[rank {rank}] kernel-only {w.name}: {ms_local:.4f} ms/step over {args.steps} back-to-back steps "
        f"(single steps {min(per_step):.4f}-{max(per_step):.4f}); wall {t_wall * 1e3 / args.steps:.3f} ms/step; "
        f"{launches} launches")

    # ---- end to end through the public API: pinned host input -> hb_hash_fixed / hb_hash_varlen
    e2e = None
    lib = _native.lib()
    hp = w.host_inputs(lib) if not args.no_e2e else None
    hpo = lib.hb_alloc_pinned(w.n * w.dlen) if hp else None
    if hp and hpo:
        import ctypes

        # digests land in one page-locked array reused across steps (the API's out= argument)
        w._out_host = np.ctypeslib.as_array(ctypes.cast(hpo, ctypes.POINTER(ctypes.c_uint8)),
                                            shape=(w.n * w.dlen,)).reshape(w.n, w.dlen)
        e2e_steps = args.e2e_steps or min(args.steps, 3 if w.kind == "decimal" else 10)
        tim = {}
        for _ in range(max(1, min(args.warmup, 2))):
            w.e2e_step(local, tim)
        barrier(world)
        torch.cuda.synchronize()
        sampler.active = True
        l1 = _native.launch_count()
        t0 = time.perf_counter()
        for k in range(e2e_steps):  # engine stage timings from the last step only (the API's default is untimed)
            res = w.e2e_step(local, tim if k == e2e_steps - 1 else None)
        t1 = time.perf_counter()
        sampler.active = False
        e2e_launches = _native.launch_count() - l1
        barrier(world)
        e2e_ms = reduce_max((t1 - t0) * 1e3 / e2e_steps, world, local)
        if res.shape[0] <= (1 << 24):
            ok = bool(np.array_equal(res, w.out.cpu().numpy()))
        else:  # very large outputs (paper workload: 10^9 digests): compare a row sample
            import torch

            idx = np.unique(np.random.default_rng(0).integers(0, res.shape[0], 1 << 16))
            ok = bool(np.array_equal(res[idx], w.out[torch.from_numpy(idx).to(w.out.device)].cpu().numpy()))
        bw = h2d_peak(max(w.h2d_bytes, w.d2h_bytes), local, d2h=w.h2d_bytes < w.d2h_bytes)
        e2e_gbs = total_bytes / (e2e_ms * 1e-3) / 1e9
        # per-step bytes over all ranks (fixed/decimal: exact from the global message count)
        if w.kind == "varlen":
            h2d_tot, d2h_tot = world * w.h2d_bytes, world * w.d2h_bytes
        else:
            h2d_tot = w.total_msgs * w.L if w.kind == "fixed" else 0
            d2h_tot = w.total_msgs * w.dlen
        h2d_gbs = max(h2d_tot, d2h_tot) / (e2e_ms * 1e-3) / 1e9
        e2e = {"value": round(e2e_gbs, 3), "unit": "GB/s",
               "h2d_bytes_per_step": h2d_tot, "d2h_bytes_per_step": d2h_tot,
               "ms_per_step": round(e2e_ms, 3), "mhash_per_s": round(total_msgs / (e2e_ms * 1e-3) / 1e6, 2),
               "api": ("paper_2407_09333_b200.crypto.batch_digest(pinned host array, out=pinned) -> hb_hash_fixed"
                       if w.kind == "fixed" else
                       "paper_2407_09333_b200.crypto.batch_digest_varlen(pinned host data, offsets, out=pinned) "
                       "-> hb_hash_varlen" if w.kind == "varlen" else
                       "paper_2407_09333_b200.crypto.hash_decimal(start, count, 9, out=pinned) -> hb_hash_decimal"),
               "steps": e2e_steps,
               "roofline": {"bound": "pcie_h2d" if w.h2d_bytes >= w.d2h_bytes else "pcie_d2h",
                            "achieved": round(h2d_gbs / world, 2), "peak": round(bw, 2),
                            "unit": "GB/s per GPU", "frac": round(h2d_gbs / world / bw, 4),
                            "peak_source": "pinned %s copy of 1 GiB on the same GPU, this run"
                                           % ("host->device" if w.h2d_bytes >= w.d2h_bytes else "device->host")},
               "engine_timing_last_step": {k: (round(v, 3) if isinstance(v, float) else v) for k, v in tim.items()},
               "gpu_launches": e2e_launches, "matches_device_run": ok}
        log(f"[rank {rank}] e2e {e2e_ms:.1f} ms/step, H2D peak {bw:.1f} GB/s, engine {tim}")
        w._host = None
        w._out_host = res = None
        if hp != -1:
            lib.hb_free_pinned(hp)
        lib.hb_free_pinned(hpo)
    sampler.stop()

    # ---- CPU baseline + bit-exact sample check (rank 0, N=1 only)
    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        rows, nbytes, t, ok, what = w.cpu_sample(threads, args.cpu_seconds)
        parity = {"rows_checked": rows, "bit_exact": ok}
        fn = "batch_fixed" if w.kind == "fixed" else "batch_varlen"
        cpu = {"value": round(nbytes / t / 1e9, 4), "unit": "GB/s", "cores": threads, "kind": "port",
               "sample": f"{what}, oracle/hetoc_oracle.c {fn} on {threads} threads, {t:.2f} s",
               "mhash_per_s": round(rows / t / 1e6, 4)}

    # ---- roofline of the dominant kernel
    peaks, peak_src = load_peaks()
    achieved = w.alg_bytes / (ms_local * 1e-3) / 1e9
    clk = sampler.summary()
    if remeasured:
        clk["remeasured"] = True
    f_max = peaks.get("sm_max_mhz", 1965.0)
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    alu_peak = sms * 64 * f_max * 1e6  # ALU-pipe lane-ops/s at max clock
    ops = getattr(w, "alu_ops_per_block", ALU_OPS_PER_BLOCK[alg])
    alu_ach = w.blocks * ops / (ms_local * 1e-3)
    t_hbm = w.alg_bytes / (peaks["hbm_gbs"] * 1e9)
    t_alu = w.blocks * ops / alu_peak
    alu = {"achieved": round(alu_ach / 1e12, 3), "peak": round(alu_peak / 1e12, 3), "unit": "Tops/s",
           "frac": round(alu_ach / alu_peak, 4), "alu_ops_per_block": ops,
           "blocks_per_launch": w.blocks, "clock_mhz": f_max}
    if t_hbm >= t_alu:
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": round(achieved / peaks["hbm_gbs"], 4)}
    else:  # integer (ALU-pipe) bound: report against the ALU-pipe roofline, HBM alongside
        roof = {"bound": "alu", "achieved": alu["achieved"], "peak": alu["peak"], "unit": "Tops/s",
                "frac": alu["frac"], "hbm_achieved_gbs": round(achieved, 1), "hbm_peak_gbs": peaks["hbm_gbs"]}
    if w.kind != "decimal":  # the survey's per-block counts assume arbitrary message words
        t_int = w.blocks * SURVEY_C_ALG[alg] / (sms * 128 * f_max * 1e6)
        roof["survey_issue_model"] = {
            "c_alg": SURVEY_C_ALG[alg], "issue_peak_tops": round(sms * 128 * f_max * 1e6 / 1e12, 3),
            "t_roof_ms": round(max(t_int, t_hbm) * 1e3, 4),
            "frac": round(max(t_int, t_hbm) / (ms_local * 1e-3), 4)}
    roof.update({"traffic": load_ncu_traffic(w.name), "kernel": w.kernel_name(),
                 "bytes_per_launch": w.alg_bytes, "peak_source": peak_src,
                 "t_roof_ms": round(max(t_hbm, t_alu) * 1e3, 4), "alu_pipe": alu})
    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
                "higher_is_better": True, "scaling": getattr(w, "scaling", "weak"), "vs_baseline": None,
                "dtype": "u32",
                "data": ("paper workload: decimal messages generated in-kernel" if w.kind == "decimal" else
                         f"synthetic: counter-based splitmix64 bytes (seed {w.seed}), generated on device"),
                "config": dict(w.config(world), launch=f"CUDA-graph replays of {GRAPH_STEPS} back-to-back steps"
                               if w.launches_per_step() else "direct launch per step",
                               gather="fused P2P into rank 0 (CUDA IPC)" if gather is not None else "none",
                               host_affinity=HOST_AFFINITY[0]),
                "mhash_per_s": round(mhash, 2), "clocks": clk, "e2e": e2e,
                "gpu_launches": launches, "roofline": roof, "cpu_baseline": cpu, "parity": parity}
        print(json.dumps(line), flush=True)
    if gather is not None:
        gather.close()
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


# --------------------------------------------------------- reference arm --
def run_reference(args):
    """The reference algorithm's CPU implementation (oracle port of hetoc.crypto;
    the reference itself is pure Python/numpy and is not installed on the box)
    on all host threads, each step a bounded sample of the same workload."""
    # each step a bounded sample: --ref-step-seconds, shrunk so the whole
    # --steps K --warmup W run stays within --ref-budget-seconds
    step_s = min(args.ref_step_seconds, max(0.05, args.ref_budget_seconds / max(1, args.steps + args.warmup)))
    import oracle

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    spec = WORKLOADS[args.workload]
    alg = spec[0].split(":")[-1]
    n = args.msgs or spec[1]
    seed, cfg_desc = spec[3], spec[4]
    threads = os.cpu_count() or 1
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if spec[0].startswith("decimal:"):
        from paper_2407_09333_b200.crypto import gen_messages

        width = spec[2]
        rows = cpu_sample_rows(alg, width, n, threads, step_s)
        data = gen_messages(0, rows, width).as_array()
        run = lambda: oracle.batch_fixed(alg, data, threads=threads)  # noqa: E731
        nbytes = rows * width
        sample = f"messages 0..{rows - 1} of the {n} decimal messages per step"
        config = {"workload": f"{alg} over {n} messages of {width} decimal digits, generated in-kernel ({cfg_desc})",
                  "alg": alg, "msgs_total": n, "msgs_per_gpu": n // world, "msg_len": width}
    elif spec[0].startswith("varlen:"):
        maxlen = spec[2]
        lens = np.random.default_rng(seed).integers(1, maxlen + 1, n).astype(np.uint64)
        probe_k = min(n, 2048)
        off = np.zeros(n + 1, np.uint64)
        off[1:] = np.cumsum(lens)
        probe = oracle.fill_random(int(off[probe_k]), seed)
        t0 = time.perf_counter()
        oracle.batch_varlen(alg, probe, off[: probe_k + 1], threads=1)
        per_msg = max((time.perf_counter() - t0) / probe_k, 1e-9)
        k = max(threads * 16, min(n, int(step_s * threads / per_msg)))
        data = oracle.fill_random(int(off[k]), seed)
        run = lambda: oracle.batch_varlen(alg, data, off[: k + 1], threads=threads)  # noqa: E731
        nbytes, rows = int(off[k]), k
        sample = f"first {k} of the {n} messages (uniform 1-{maxlen} B) per step"
        config = {"workload": f"{alg} {n} messages of uniform 1-{maxlen} B per GPU, offsets layout ({cfg_desc})",
                  "alg": alg, "msgs_per_gpu": n, "msg_len": f"uniform 1-{maxlen}"}
    else:
        L = spec[2]
        rows = cpu_sample_rows(alg, L, n, threads, step_s)
        data = oracle.fill_random(rows * L, seed).reshape(rows, L)
        run = lambda: oracle.batch_fixed(alg, data, threads=threads)  # noqa: E731
        nbytes = rows * L
        sample = f"{rows} of the {n} x {L} B messages per step"
        strong = spec[0].startswith("strong:")
        what = (f"{alg} {n} x {L} B fixed-width, split over the GPUs" if strong
                else f"{alg} {n} x {L} B fixed-width per GPU")
        config = {"workload": f"{what} ({cfg_desc})", "alg": alg, "msgs_per_gpu": n // world if strong else n,
                  "msg_len": L}
    for _ in range(args.warmup):
        run()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    value = nbytes / t / 1e9
    dec = spec[0].startswith("decimal:") or spec[0].startswith("strong:")
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3), "higher_is_better": True,
            "scaling": "strong" if dec else "weak", "vs_baseline": None, "dtype": "u32",
            "data": "paper workload: decimal messages (gen_messages)" if spec[0].startswith("decimal:") else
                    f"synthetic: counter-based splitmix64 bytes (seed {seed})", "config": config,
            "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": threads, "kind": "port",
                             "sample": f"{sample}, oracle/hetoc_oracle.c (C restatement of hetoc.crypto) "
                                       f"on {threads} threads"},
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
    ap.add_argument("--msgs", type=int, default=0, help="override the message count (per GPU; total for strong-scaling workloads)")
    ap.add_argument("--e2e-steps", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=3.0)
    ap.add_argument("--ref-step-seconds", type=float, default=1.0)
    ap.add_argument("--ref-budget-seconds", type=float, default=150.0,
                    help="--impl reference: upper bound on the whole run's CPU time")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--gather", choices=["none", "p2p"], default="none",
                    help="N>1: fused device-side digest gather into rank 0 (hash kernels store over NVLink)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        log("note: timing rules want >= 3 warm-up steps")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
