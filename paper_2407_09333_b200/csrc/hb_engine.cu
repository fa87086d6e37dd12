// hb_engine.cu -- host-side engine and C ABI of the batched-hash engine.
//
// This is the B200 realisation of the reference's *hyper* data management and
// task splitting for crypto.hash_batch:
//   * message-range split across GPUs   = partition_range (passes/partition.py:17-31)
//                                          as applied by lower_loop (passes/lower_hyper_for.py:207-254)
//   * per-device staging                = _emit_dev_launch (passes/lower_hyper_for.py:279-368):
//       hyper.alloc(slice) -> hyper.memcpy(src_off = s*stride) -> dev.launch[0,n) offset s
//       -> hyper.memcpy(dst_off = s*dlen) -> hyper.dealloc
//   * capacity sub-batching             = _run_group (runtime/executor.py:603-699),
//       here a ring of kSlots chunk buffers per GPU whose H2D / kernel / D2H run
//       on separate streams so copies overlap compute.
// One host thread per GPU drives its shard; all CUDA work of a shard is
// asynchronous on that GPU's slot streams.
#include <cuda.h>
#include <cuda_runtime.h>
#include <ctype.h>
#include <cxxabi.h>
#include <pthread.h>
#include <sched.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <deque>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/hetoc_b200.h"
#include "hb_internal.h"

namespace hb {
uint64_t launches_total();

// ------------------------------------------------------------ error state --
static thread_local std::string g_err;

static int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define HB_CK(expr)                                                                                        \
    do {                                                                                                   \
        cudaError_t e_ = (expr);                                                                           \
        if (e_ != cudaSuccess) {                                                                           \
            cudaGetLastError(); /* clear a non-sticky error so the next launch check does not report it */ \
            const char* extra_ = (e_ == cudaErrorNotSupported || e_ == cudaErrorInvalidValue) ? tma_error() : ""; \
            return fail(e_ == cudaErrorMemoryAllocation ? HB_ERR_NOMEM : HB_ERR_CUDA, "%s failed: %s %s (%s:%d)", \
                        #expr, cudaGetErrorString(e_), extra_, __FILE__, __LINE__);                        \
        }                                                                                                  \
    } while (0)

static int digest_len(int alg) {
    switch (alg) {
    case HB_SHA1: return 20;
    case HB_MD5: return 16;
    case HB_SM3: return 32;
    default: return -1;
    }
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int d) {
        cudaGetDevice(&prev);
        if (prev != d) cudaSetDevice(d);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

static int device_count() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

// ---------------------------------------------------------------- tuning --
// Chunk budget for a shard of `staged` input bytes and `out` digest bytes.
// When the digests are big enough for their copy-out to matter (short
// messages: >= pipe_min_out, 4 MiB), the shard is cut into at least
// pipe_chunks (4) chunks of >= min_chunk_bytes (8 MiB), so chunk k's
// kernel + D2H overlap chunk k+1's H2D across the slot ring instead of running
// back to back.  Smaller shards, or long messages with few digest bytes, stay
// one chunk: every extra chunk costs ~10-20 us of copy/launch latency
// (profiles/ab_pipe_r1.txt: +7..17 % e2e at 16-64 MB of 64-byte messages,
// -3..-40 % if 4 MB batches or 1 KiB messages were split).  `cap` is the
// GPU's chunk limit from its HBM budget (GpuCtx::chunk_cap).
static uint64_t pipelined_budget(uint64_t staged, uint64_t out, uint64_t cap) {
    const Tuning& T = tuning();
    const uint64_t chunk = std::min(T.chunk_bytes, cap);
    if (out < T.pipe_min_out) return chunk;
    return std::min(chunk, std::max(T.min_chunk_bytes, (staged + T.pipe_chunks - 1) / T.pipe_chunks));
}
static int memcpy_threads(int n_gpus) {
    if (tuning().memcpy_threads) return (int)tuning().memcpy_threads;
    unsigned hw = std::thread::hardware_concurrency();
    int per = (int)(hw ? hw : 8) / std::max(1, n_gpus);
    return std::max(1, std::min(8, per));
}

// Host memcpy split across threads (pageable <-> pinned staging).
static void parallel_memcpy(void* dst, const void* src, uint64_t bytes, int nthreads) {
    if (bytes < (8ull << 20) || nthreads <= 1) {
        memcpy(dst, src, bytes);
        return;
    }
    std::vector<std::thread> ts;
    const uint64_t per = ((bytes / nthreads) + 4095) & ~4095ull;
    for (int k = 0; k < nthreads; ++k) {
        const uint64_t lo = per * k;
        if (lo >= bytes) break;
        const uint64_t len = std::min(per, bytes - lo);
        ts.emplace_back([=] { memcpy((uint8_t*)dst + lo, (const uint8_t*)src + lo, len); });
    }
    for (auto& t : ts) t.join();
}

static bool is_pinned(const void* p, uint64_t bytes) {
    if (!p || !bytes) return false;
    const void* probes[2] = {p, (const uint8_t*)p + bytes - 1};
    for (const void* q : probes) {
        cudaPointerAttributes a;
        if (cudaPointerGetAttributes(&a, q) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        if (a.type != cudaMemoryTypeHost) return false;
    }
    return true;
}

// ------------------------------------------------------- per-GPU context --
constexpr int kSlots = 3;

// Device buffers of the chunk ring.  They only grow (to the largest chunk
// seen, rounded up to 2 MiB) and live until hb_shutdown; the ring's total is
// bounded by the GPU's budget (GpuCtx::chunk_cap), so growth never fails for
// lack of HBM that cudaMemGetInfo said was there.
struct DevBuf {
    void* p = nullptr;
    uint64_t cap = 0;
    cudaError_t ensure(uint64_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        const uint64_t want = (bytes + (2ull << 20) - 1) & ~((2ull << 20) - 1);
        cudaError_t e = cudaMalloc(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
};
struct HostBuf {
    void* p = nullptr;
    uint64_t cap = 0;
    cudaError_t ensure(uint64_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        const uint64_t want = (bytes + 4095) & ~4095ull;
        cudaError_t e = cudaHostAlloc(&p, want, cudaHostAllocPortable);
        if (e == cudaSuccess) cap = want;
        return e;
    }
};

enum Stage { kH2D = 0, kKernel = 1, kD2H = 2 };

struct Slot {
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[6] = {};  // h2d0, h2d1, k0, k1, d2h0, d2h1
    DevBuf d_in, d_out, d_off, d_scratch;
    HostBuf h_in, h_out, h_off;
    bool in_use = false;
    bool has_h2d = false;
    bool timed = false;  // ev[0..4] recorded (the caller asked for hb_timing)
    uint64_t chunk = 0;  // chunk index of the work in flight
    // deferred copy-out (pageable destination)
    uint8_t* pend_dst = nullptr;
    uint64_t pend_bytes = 0;
};

struct GpuCtx {
    int dev = -1;
    std::mutex mu;
    bool ready = false;
    cudaEvent_t ev_ref = nullptr;  // t = 0 of a timed shard's timeline
    uint64_t budget = 0;           // HBM the ring may use: free at init - device_reserve
    uint64_t chunk_cap = 0;        // largest input chunk the ring is allowed
    Slot slots[kSlots];
};

static std::mutex g_ctx_mu;
static std::vector<std::unique_ptr<GpuCtx>> g_ctx;

static int get_ctx(int dev, GpuCtx** out) {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    const int nd = device_count();
    if (dev < 0 || dev >= nd) return fail(HB_ERR_NODEV, "device ordinal %d out of range (%d devices)", dev, nd);
    if ((int)g_ctx.size() < nd) g_ctx.resize(nd);
    if (!g_ctx[dev]) {
        g_ctx[dev].reset(new GpuCtx());
        g_ctx[dev]->dev = dev;
    }
    *out = g_ctx[dev].get();
    return HB_OK;
}

// The per-GPU memory pool of the reference's Arena (runtime/arena.py:28-63,
// capacity from the device spec) sized from what the device actually has:
// at first use, budget = free HBM - device_reserve; each of the kSlots slots
// may stage at most chunk_cap input bytes (plus its digests/offsets), so the
// ring never outgrows the budget; larger shards are sub-batched, as
// _run_group does for over-capacity groups (runtime/executor.py:603-699).
static int ctx_init(GpuCtx& c) {  // caller holds c.mu and has set the device
    if (c.ready) return HB_OK;
    for (Slot& s : c.slots) {
        HB_CK(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
        for (auto& e : s.ev) HB_CK(cudaEventCreate(&e));
    }
    HB_CK(cudaEventCreate(&c.ev_ref));
    size_t fr = 0, tot = 0;
    HB_CK(cudaMemGetInfo(&fr, &tot));
    const uint64_t reserve = tuning().device_reserve;
    c.budget = fr > reserve + (64ull << 20) ? fr - reserve : (64ull << 20);
    // input chunk + its digests (<= 1/2 of it for 64-byte rows: 32 B / 64 B) + offsets/scratch (<= 12 B per
    // 1-byte message, capped by the 64-byte-per-message chunk rule in run_shard_locked) ~ 2x the input chunk
    c.chunk_cap = std::max<uint64_t>(1ull << 20, c.budget / (2 * kSlots));
    c.ready = true;
    return HB_OK;
}

struct Span {
    int stage;
    uint64_t chunk;
    double t0, t1;  // ms since the shard's reference event
};

struct ShardStats {
    int dev = -1;
    double kernel_ms = 0, h2d_ms = 0, d2h_ms = 0;  // union of busy intervals per stage
    uint64_t h2d_bytes = 0, d2h_bytes = 0, chunks = 0, launches = 0;
    std::vector<Span> spans;
    const void* last_kernel = nullptr;
    int status = HB_OK;
    std::string err;
};

// Length of the union of [t0, t1) intervals of one stage (the slots' copies
// and kernels overlap each other: summing them would over-count).
static double union_ms(std::vector<Span>& v, int stage) {
    std::vector<std::pair<double, double>> iv;
    for (const Span& s : v)
        if (s.stage == stage && s.t1 > s.t0) iv.emplace_back(s.t0, s.t1);
    std::sort(iv.begin(), iv.end());
    double total = 0, cur0 = 0, cur1 = -1e300;
    for (auto& x : iv) {
        if (x.first > cur1) {
            if (cur1 > cur0) total += cur1 - cur0;
            cur0 = x.first;
            cur1 = x.second;
        } else {
            cur1 = std::max(cur1, x.second);
        }
    }
    if (cur1 > cur0) total += cur1 - cur0;
    return total;
}

// Wait for a slot's previous chunk, land its deferred copy-out, bank timings.
static int retire_slot(GpuCtx& c, Slot& s, ShardStats& st, int mt) {
    if (!s.in_use) return HB_OK;
    HB_CK(cudaEventSynchronize(s.ev[5]));
    if (s.timed) {
        float a = 0, b = 0;
        auto span = [&](int stage, int e0, int e1) {
            if (cudaEventElapsedTime(&a, c.ev_ref, s.ev[e0]) == cudaSuccess &&
                cudaEventElapsedTime(&b, c.ev_ref, s.ev[e1]) == cudaSuccess)
                st.spans.push_back({stage, s.chunk, (double)a, (double)b});
            else
                cudaGetLastError();
        };
        if (s.has_h2d) span(kH2D, 0, 1);
        span(kKernel, 2, 3);
        span(kD2H, 4, 5);
    }
    if (s.pend_bytes) {
        nvtxRangePushA("hb d2h staging memcpy");
        parallel_memcpy(s.pend_dst, s.h_out.p, s.pend_bytes, mt);
        nvtxRangePop();
    }
    s.pend_bytes = 0;
    s.in_use = false;
    return HB_OK;
}

// Stage a host range into a slot's device buffer (direct DMA when pinned).
static int stage_in(Slot& s, DevBuf& dst, HostBuf& stage, const void* src, uint64_t bytes, bool pinned, int mt) {
    if (!bytes) return HB_OK;
    if (pinned) {
        HB_CK(cudaMemcpyAsync(dst.p, src, bytes, cudaMemcpyHostToDevice, s.stream));
    } else {
        HB_CK(stage.ensure(bytes));
        nvtxRangePushA("hb h2d staging memcpy");
        parallel_memcpy(stage.p, src, bytes, mt);
        nvtxRangePop();
        HB_CK(cudaMemcpyAsync(dst.p, stage.p, bytes, cudaMemcpyHostToDevice, s.stream));
    }
    return HB_OK;
}

static int stage_out(Slot& s, uint8_t* dst, uint64_t bytes, bool pinned) {
    if (!bytes) return HB_OK;
    if (pinned) {
        HB_CK(cudaMemcpyAsync(dst, s.d_out.p, bytes, cudaMemcpyDeviceToHost, s.stream));
    } else {
        HB_CK(s.h_out.ensure(bytes));
        HB_CK(cudaMemcpyAsync(s.h_out.p, s.d_out.p, bytes, cudaMemcpyDeviceToHost, s.stream));
        s.pend_dst = dst;
        s.pend_bytes = bytes;
    }
    return HB_OK;
}

// A unit of work for one GPU: the shard [lo, hi) of the global message range.
struct ShardJob {
    int kind = 0;  // 0 fixed, 1 varlen, 2 decimal
    int alg = 0;
    int dev = 0;
    uint64_t lo = 0, hi = 0;
    // fixed
    const uint8_t* msgs = nullptr;
    uint64_t msg_len = 0;
    // varlen
    const uint8_t* data = nullptr;
    const uint64_t* offsets = nullptr;
    // decimal
    uint64_t start = 0;
    int width = 0;
    uint8_t* out = nullptr;
    bool in_pinned = false, off_pinned = false, out_pinned = false;
    uint32_t flags = 0;
    int mt = 1;
    bool timed = true;  // record per-stage events (hb_timing requested)
};

static int run_shard_locked(GpuCtx& c, const ShardJob& j, ShardStats& st) {
    int rc = ctx_init(c);
    if (rc) return rc;
    const int dlen = digest_len(j.alg);
    const uint64_t staged = j.kind == 0 ? (j.hi - j.lo) * j.msg_len
                          : j.kind == 1 ? j.offsets[j.hi] - j.offsets[j.lo]
                                        : (j.hi - j.lo) * (uint64_t)dlen;  // decimal: digests only
    const uint64_t budget = pipelined_budget(staged, (j.hi - j.lo) * (uint64_t)dlen, c.chunk_cap);
    uint64_t slot_k = 0;
    const uint64_t l0 = hb::launches_total();
    if (j.timed) HB_CK(cudaEventRecord(c.ev_ref, c.slots[0].stream));
    uint64_t i = j.lo;
    while (i < j.hi) {
        // ---- plan the chunk [i, e)
        uint64_t e, in_bytes = 0, in_off = 0;
        if (j.kind == 0) {
            uint64_t per = j.msg_len ? std::max<uint64_t>(1, budget / j.msg_len) : (j.hi - j.lo);
            // digests of a chunk of short rows stay within the same budget
            per = std::min<uint64_t>(per, std::max<uint64_t>(1, budget / (uint64_t)dlen));
            if (per >= 256) per &= ~127ull;
            e = std::min(j.hi, i + per);
            in_bytes = (e - i) * j.msg_len;
            in_off = i * j.msg_len;
        } else if (j.kind == 1) {
            const uint64_t lim = j.offsets[i] + budget;
            const uint64_t* ub = std::upper_bound(j.offsets + i + 1, j.offsets + j.hi + 1, lim);
            e = (uint64_t)(ub - j.offsets) - 1;  // last index whose offset <= lim
            if (e <= i) e = i + 1;                // one over-budget message: its own chunk
            const uint64_t max_msgs = std::max<uint64_t>(1024, budget / 64);
            e = std::min(e, i + max_msgs);
            in_off = j.offsets[i];
            in_bytes = j.offsets[e] - j.offsets[i];
            if (in_bytes > c.chunk_cap + (c.chunk_cap >> 1))
                return fail(HB_ERR_NOMEM, "message %llu (%llu bytes) exceeds the GPU %d chunk budget (%llu bytes)",
                            (unsigned long long)i, (unsigned long long)in_bytes, c.dev,
                            (unsigned long long)c.chunk_cap);
        } else {
            const uint64_t per = std::max<uint64_t>(1, budget / (uint64_t)dlen);
            e = std::min(j.hi, i + per);
        }
        const uint64_t cn = e - i;
        Slot& s = c.slots[slot_k % kSlots];
        rc = retire_slot(c, s, st, j.mt);
        if (rc) return rc;
        s.chunk = slot_k;
        ++slot_k;
        HB_CK(s.d_out.ensure(cn * dlen));
        if (in_bytes) HB_CK(s.d_in.ensure(in_bytes + 64));
        s.has_h2d = false;
        // ---- copy in (the per-stage events only when the caller wants hb_timing:
        // each record is a driver call on a small batch's critical path)
        s.timed = j.timed;
        if (j.timed) HB_CK(cudaEventRecord(s.ev[0], s.stream));
        if (j.kind == 0 && in_bytes) {
            rc = stage_in(s, s.d_in, s.h_in, j.msgs + in_off, in_bytes, j.in_pinned, j.mt);
            if (rc) return rc;
            s.has_h2d = true;
        } else if (j.kind == 1) {
            HB_CK(s.d_off.ensure((cn + 1) * 8));
            rc = stage_in(s, s.d_off, s.h_off, j.offsets + i, (cn + 1) * 8, j.off_pinned, j.mt);
            if (rc) return rc;
            if (in_bytes) {
                rc = stage_in(s, s.d_in, s.h_in, j.data + in_off, in_bytes, j.in_pinned, j.mt);
                if (rc) return rc;
            }
            s.has_h2d = true;
        }
        if (j.timed) HB_CK(cudaEventRecord(s.ev[1], s.stream));
        st.h2d_bytes += in_bytes + (j.kind == 1 ? (cn + 1) * 8 : 0);
        // ---- kernel
        if (j.timed) HB_CK(cudaEventRecord(s.ev[2], s.stream));
        uint8_t* dout = static_cast<uint8_t*>(s.d_out.p);
        if (j.kind == 0) {
            HB_CK(launch_fixed(j.alg, static_cast<const uint8_t*>(s.d_in.p), cn, j.msg_len, dout, s.stream, j.flags));
        } else if (j.kind == 1) {
            void* scratch = nullptr;
            if (!(j.flags & HB_FLAG_NO_SORT)) {
                HB_CK(s.d_scratch.ensure(varlen_scratch_bytes(cn)));
                scratch = s.d_scratch.p;
            }
            HB_CK(launch_varlen(j.alg, static_cast<const uint8_t*>(s.d_in.p), in_bytes,
                                static_cast<const uint64_t*>(s.d_off.p), j.offsets[i], cn, dout, scratch, s.stream,
                                j.flags));
        } else {
            HB_CK(launch_decimal(j.alg, j.start + i, cn, j.width, dout, s.stream));
        }
        if (j.timed) {
            HB_CK(cudaEventRecord(s.ev[3], s.stream));
            HB_CK(cudaEventRecord(s.ev[4], s.stream));
        }
        // ---- copy out (dst_off = s*dlen)
        rc = stage_out(s, j.out + i * dlen, cn * dlen, j.out_pinned);
        if (rc) return rc;
        HB_CK(cudaEventRecord(s.ev[5], s.stream));
        st.d2h_bytes += cn * dlen;
        st.chunks += 1;
        s.in_use = true;
        if (j.flags & HB_FLAG_SYNC_H2D) {
            rc = retire_slot(c, s, st, j.mt);
            if (rc) return rc;
        }
        i = e;
    }
    for (Slot& s : c.slots) {
        rc = retire_slot(c, s, st, j.mt);
        if (rc) return rc;
    }
    st.launches = hb::launches_total() - l0;
    st.h2d_ms = union_ms(st.spans, kH2D);
    st.kernel_ms = union_ms(st.spans, kKernel);
    st.d2h_ms = union_ms(st.spans, kD2H);
    return HB_OK;
}

// Pin the calling thread to the CPUs local to GPU `dev` (the sysfs
// local_cpulist of its PCI function), intersected with the allowed set.
// Called once by each GPU's worker thread when it starts: the GPU's pinned
// staging ring (first allocated by that thread) and the host-copy helpers it
// spawns then stay on the GPU's NUMA node.  Best effort; $HB_BIND_NUMA=0
// disables.  The caller's own affinity is never changed.
static void bind_thread_near_gpu(int dev) {
    if (!tuning().bind_numa) return;
    char bus[32];
    if (cudaDeviceGetPCIBusId(bus, sizeof bus, dev) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    for (char* q = bus; *q; ++q) *q = (char)tolower((unsigned char)*q);
    char path[128];
    snprintf(path, sizeof path, "/sys/bus/pci/devices/%s/local_cpulist", bus);
    FILE* f = fopen(path, "r");
    if (!f) return;
    char buf[4096];
    const size_t m = fread(buf, 1, sizeof buf - 1, f);
    fclose(f);
    buf[m] = '\0';
    cpu_set_t want;
    CPU_ZERO(&want);
    for (char* q = buf; *q;) {  // "0-15,32-47\n"
        char* e = nullptr;
        const long a = strtol(q, &e, 10);
        if (e == q) break;
        long b = a;
        q = e;
        if (*q == '-') {
            b = strtol(q + 1, &e, 10);
            q = e;
        }
        for (long c = a; c <= b && c < CPU_SETSIZE; ++c)
            if (c >= 0) CPU_SET((int)c, &want);
        while (*q == ',' || *q == '\n' || *q == ' ') ++q;
    }
    cpu_set_t have;
    if (pthread_getaffinity_np(pthread_self(), sizeof have, &have) != 0) return;
    CPU_AND(&want, &want, &have);
    if (CPU_COUNT(&want) > 0) pthread_setaffinity_np(pthread_self(), sizeof want, &want);
}

static void run_shard(const ShardJob& j, ShardStats& st) {
    GpuCtx* c = nullptr;
    st.dev = j.dev;
    int rc = get_ctx(j.dev, &c);
    if (rc == HB_OK) {
        std::lock_guard<std::mutex> lk(c->mu);
        DeviceGuard g(j.dev);
        char label[48];
        snprintf(label, sizeof label, "hb shard gpu %d", j.dev);
        nvtxRangePushA(label);
        rc = run_shard_locked(*c, j, st);
        nvtxRangePop();
        if (rc != HB_OK) {
            // leave the context reusable: drain whatever is in flight
            for (Slot& s : c->slots) {
                if (s.stream) cudaStreamSynchronize(s.stream);
                s.in_use = false;
                s.pend_bytes = 0;
            }
            cudaGetLastError();
        }
    }
    st.last_kernel = last_hash_kernel();
    st.status = rc;
    if (rc != HB_OK) st.err = g_err;
}

// ------------------------------------------------------ per-GPU workers --
// One persistent host thread per GPU (created on first multi-GPU call, NUMA-
// bound once) serves the shards of multi-GPU calls; a call whose work lands on
// a single GPU runs on the caller's own thread (no hand-off).  The reference
// calls the boundary concurrently from pool threads (executor.py:596-599,
// batch.py:310-313): shards of concurrent calls queue on each GPU's worker and
// serialise on that GPU's context mutex.
struct Worker {
    int dev = -1;
    std::thread th;
    std::mutex mu;
    std::condition_variable cv;
    std::deque<std::function<void()>> q;
    bool stop = false;
    void loop() {
        bind_thread_near_gpu(dev);
        for (;;) {
            std::function<void()> f;
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return stop || !q.empty(); });
                if (stop && q.empty()) return;
                f = std::move(q.front());
                q.pop_front();
            }
            f();
        }
    }
    void submit(std::function<void()> f) {
        {
            std::lock_guard<std::mutex> lk(mu);
            q.push_back(std::move(f));
        }
        cv.notify_one();
    }
};
// Leaked on purpose at exit (threads parked in cv.wait must not see their
// mutex destroyed by static destructors); hb_shutdown joins and frees them.
static std::vector<Worker*> g_workers;

static Worker* get_worker(int dev) {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    if ((int)g_workers.size() <= dev) g_workers.resize(dev + 1, nullptr);
    if (!g_workers[dev]) {
        Worker* w = new Worker();
        w->dev = dev;
        w->th = std::thread([w] { w->loop(); });
        g_workers[dev] = w;
    }
    return g_workers[dev];
}

// Per-device pool of small-call slots: a non-blocking stream, a 64-byte
// mapped pinned digest slot (hb_digest_small) and, allocated on first use,
// mapped pinned input / offsets / digest buffers for the zero-copy path of
// small batches (small_batch below).  A call takes one and returns it, so
// concurrent callers never share a slot and pool threads that come and go
// leak nothing.  hb_shutdown frees them.
struct SmallSlot {
    cudaStream_t stream = nullptr;
    uint8_t* h_out = nullptr;
    uint8_t* d_out = nullptr;
    uint32_t seq = 0;  // last value the kernel published at h_out + 48
    uint8_t* zc = nullptr;  // [in: zc_in_cap + 256][offsets: kZcOffBytes][digests: kZcOutBytes]
    uint64_t zc_in_cap = 0;
};
constexpr uint64_t kZcOffBytes = 64u << 10;
constexpr uint64_t kZcOutBytes = 128u << 10;
static std::mutex g_small_mu;
static std::vector<std::vector<SmallSlot>> g_small;

static int take_slot(int gpu, SmallSlot& sl) {  // on the current device == gpu
    {
        std::lock_guard<std::mutex> lk(g_small_mu);
        if ((int)g_small.size() <= gpu) g_small.resize(gpu + 1);
        if (!g_small[gpu].empty()) {
            sl = g_small[gpu].back();
            g_small[gpu].pop_back();
            return HB_OK;
        }
    }
    // Built in a local: the lease returns only complete slots to the pool.
    SmallSlot n;
    HB_CK(cudaHostAlloc(reinterpret_cast<void**>(&n.h_out), 64, cudaHostAllocMapped | cudaHostAllocPortable));
    memset(n.h_out, 0, 64);  // seq word starts at 0, the value no launch publishes
    HB_CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&n.d_out), n.h_out, 0));
    HB_CK(cudaStreamCreateWithFlags(&n.stream, cudaStreamNonBlocking));
    sl = n;
    return HB_OK;
}

static void give_slot(int gpu, const SmallSlot& sl) {
    std::lock_guard<std::mutex> lk(g_small_mu);
    g_small[gpu].push_back(sl);
}

// Returns the slot to the pool on every exit, error paths included (a call
// rejected at launch, e.g. for bad flags, leaves the slot usable; after a
// sticky error the context is gone anyway).
struct SlotLease {
    int gpu;
    SmallSlot sl;
    explicit SlotLease(int g) : gpu(g) {}
    ~SlotLease() {
        if (sl.stream) give_slot(gpu, sl);
    }
};

// Small batches (at most tuning().zc_max_bytes of messages, kZcOutBytes of
// digests, kZcOffBytes of offsets) skip the chunk ring: the bytes are copied
// into the slot's mapped pinned buffer and the kernel reads them over PCIe
// and stores its digests into mapped memory, so a call is memcpy + one
// launch + synchronise + memcpy instead of H2D copy, launch, D2H copy and
// their events: 31.7 -> 20.3 us for one 64-byte row, 44.8 -> 27.3 us for
// 64 KiB of 64-byte rows, even for 1 KiB rows (their per-thread row loads
// over PCIe are slower).  A GPU's own loads over PCIe reach only ~8-22 GB/s,
// so calls above 256 KiB keep the DMA-engine ring
// (profiles/r2/zero_copy_r2aw.txt).
static bool small_batch_fits(uint64_t in_bytes, uint64_t n, uint64_t out_bytes, bool varlen) {
    return in_bytes <= tuning().zc_max_bytes && out_bytes <= kZcOutBytes && (!varlen || (n + 1) * 8 <= kZcOffBytes);
}

static int small_batch(int kind, int alg, const uint8_t* data, uint64_t in_bytes, const uint64_t* offsets, uint64_t n,
                       uint64_t msg_len, uint8_t* out, uint64_t out_bytes, int gpu, uint32_t flags) {
    DeviceGuard g(gpu);
    SlotLease lease(gpu);
    SmallSlot& sl = lease.sl;
    if (int rc = take_slot(gpu, sl)) return rc;
    const uint64_t cap = std::max<uint64_t>(tuning().zc_max_bytes, 4096);
    if (!sl.zc || sl.zc_in_cap < in_bytes) {  // (an all-empty batch still needs the digest buffer)
        if (sl.zc) HB_CK(cudaFreeHost(sl.zc));
        sl.zc = nullptr;
        sl.zc_in_cap = 0;
        HB_CK(cudaHostAlloc(reinterpret_cast<void**>(&sl.zc), cap + 256 + kZcOffBytes + kZcOutBytes,
                            cudaHostAllocMapped | cudaHostAllocPortable));
        sl.zc_in_cap = cap;
    }
    uint8_t* h_in = sl.zc;
    uint64_t* h_off = reinterpret_cast<uint64_t*>(sl.zc + sl.zc_in_cap + 256);
    uint8_t* h_dig = sl.zc + sl.zc_in_cap + 256 + kZcOffBytes;
    uint8_t *d_in, *d_dig;
    uint64_t* d_off;
    HB_CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_in), h_in, 0));
    d_off = reinterpret_cast<uint64_t*>(d_in + sl.zc_in_cap + 256);
    d_dig = d_in + sl.zc_in_cap + 256 + kZcOffBytes;
    if (in_bytes) memcpy(h_in, data, in_bytes);
    flags = (flags & ~HB_FLAG_INPUT_READY) | HB_FLAG_NO_TMA;  // TMA descriptors address device memory
    if (kind == 0) {
        HB_CK(launch_fixed(alg, d_in, n, msg_len, d_dig, sl.stream, flags));
    } else {
        memcpy(h_off, offsets, (n + 1) * 8);
        HB_CK(launch_varlen(alg, d_in, in_bytes, d_off, offsets[0], n, d_dig, nullptr, sl.stream,
                            flags | HB_FLAG_NO_SORT));
    }
    HB_CK(cudaStreamSynchronize(sl.stream));
    memcpy(out, h_dig, out_bytes);
    return HB_OK;
}

// partition_range, pkg/src/hetoc/passes/partition.py:17-31 (same double
// arithmetic as the Python: cum += r; b = lb + floor(n*cum + 0.5)).
static int partition(int64_t lb, int64_t ub, const double* ratios, int k, int64_t* bounds) {
    if (lb > ub) return fail(HB_ERR_INVAL, "range [%lld, %lld) is inverted", (long long)lb, (long long)ub);
    if (k < 1 || !ratios) return fail(HB_ERR_INVAL, "need at least one ratio");
    const int64_t n = ub - lb;
    bounds[0] = lb;
    double cum = 0.0;
    for (int i = 0; i < k - 1; ++i) {
        cum += ratios[i];
        int64_t b = lb + (int64_t)std::floor((double)n * cum + 0.5);
        b = std::min(std::max(b, bounds[i]), ub);
        bounds[i + 1] = b;
    }
    bounds[k] = ub;
    return HB_OK;
}

// The default device set ("all GPUs") for a call of `bytes` staged bytes: a
// call below tuning().multi_gpu_min_bytes (32 MiB) would spend more on
// per-shard setup than it saves in PCIe time, so it runs on ONE GPU, picked
// per calling thread round-robin (pool threads of the reference's executor
// and hash_batch spread over the GPUs instead of all fanning out to all).
static int pick_default_gpu(int nd) {
    static std::atomic<int> next{0};
    static thread_local int mine = -1;
    if (mine < 0) mine = next.fetch_add(1, std::memory_order_relaxed);
    return mine % nd;
}

static int resolve_gpus(const int* gpus, int n_gpus, uint64_t bytes, std::vector<int>& out) {
    const int nd = device_count();
    if (nd == 0) return fail(HB_ERR_NODEV, "no CUDA device visible");
    out.clear();
    if (!gpus || n_gpus <= 0) {
        if (nd > 1 && bytes < tuning().multi_gpu_min_bytes) {
            out.push_back(pick_default_gpu(nd));
            return HB_OK;
        }
        for (int d = 0; d < nd; ++d) out.push_back(d);
    } else {
        for (int k = 0; k < n_gpus; ++k) {
            if (gpus[k] < 0 || gpus[k] >= nd)
                return fail(HB_ERR_NODEV, "device ordinal %d out of range (%d devices)", gpus[k], nd);
            out.push_back(gpus[k]);
        }
    }
    return HB_OK;
}

// Duty-ratio validation as the reference verifier does for hyper.for device
// bindings (pkg/src/hetoc/hir/verify.py:245-260, RATIO_SUM_TOL core.py:21).
static int check_ratios(const double* r, int k) {
    double total = 0.0;
    for (int i = 0; i < k; ++i) {
        if (!(r[i] >= 0.0 && r[i] <= 1.0)) return fail(HB_ERR_INVAL, "duty ratio %g outside [0, 1]", r[i]);
        total += r[i];
    }
    if (std::fabs(total - 1.0) > 1e-9) return fail(HB_ERR_INVAL, "duty ratios sum to %.10g", total);
    return HB_OK;
}

// Per calling thread: the stage timeline of its last timed call.
static thread_local std::vector<hb_span> t_timeline;

// Split [0, n) over the GPUs (equal ratios unless given), run the shards
// (one on the caller's thread, several on the GPUs' workers), merge stats.
static int run_sharded(ShardJob proto, uint64_t n, const std::vector<int>& devs, hb_timing* t,
                       const double* user_ratios = nullptr) {
    const auto t0 = std::chrono::steady_clock::now();
    const int k = (int)devs.size();
    std::vector<double> ratios(k, 1.0 / k);
    if (user_ratios) ratios.assign(user_ratios, user_ratios + k);
    std::vector<int64_t> bounds(k + 1);
    int rc = partition(0, (int64_t)n, ratios.data(), k, bounds.data());
    if (rc) return rc;
    proto.mt = memcpy_threads(k);
    proto.timed = t != nullptr;
    std::vector<ShardJob> jobs;
    for (int d = 0; d < k; ++d) {
        if (bounds[d + 1] <= bounds[d]) continue;
        ShardJob j = proto;
        j.dev = devs[d];
        j.lo = (uint64_t)bounds[d];
        j.hi = (uint64_t)bounds[d + 1];
        jobs.push_back(j);
    }
    std::vector<ShardStats> stats(jobs.size());
    if (jobs.size() == 1) {
        run_shard(jobs[0], stats[0]);
    } else {
        std::mutex mu;
        std::condition_variable cv;
        size_t left = jobs.size();
        for (size_t q = 0; q < jobs.size(); ++q)
            get_worker(jobs[q].dev)->submit([&, q] {
                run_shard(jobs[q], stats[q]);
                std::lock_guard<std::mutex> lk(mu);
                if (--left == 0) cv.notify_one();
            });
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return left == 0; });
    }
    hb_timing agg;
    memset(&agg, 0, sizeof agg);
    if (t) t_timeline.clear();
    for (auto& s : stats) {
        if (s.status != HB_OK) {
            g_err = s.err;
            return s.status;
        }
        agg.kernel_ms = std::max(agg.kernel_ms, s.kernel_ms);
        agg.h2d_ms = std::max(agg.h2d_ms, s.h2d_ms);
        agg.d2h_ms = std::max(agg.d2h_ms, s.d2h_ms);
        agg.h2d_bytes += s.h2d_bytes;
        agg.d2h_bytes += s.d2h_bytes;
        agg.chunks += s.chunks;
        agg.launches += s.launches;
        agg.shards += 1;
        if (s.dev >= 0 && s.dev < 64) agg.device_mask |= 1ull << s.dev;
        if (s.last_kernel) set_last_hash_kernel(s.last_kernel);
        if (t)
            for (const Span& sp : s.spans) t_timeline.push_back({s.dev, sp.stage, sp.chunk, sp.t0, sp.t1});
    }
    agg.total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (t) *t = agg;
    return HB_OK;
}

// gen_messages' range rule (batch.py:86-99: indices must fit in `width`
// digits) on 64-bit indices: start + count must not wrap, and must not
// exceed 10^width (10^20 > 2^64, so width 20 only needs the wrap check).
static int check_decimal_range(uint64_t start, uint64_t count, int width) {
    if (start > UINT64_MAX - count)
        return fail(HB_ERR_INVAL, "index range [%llu, +%llu) overflows 64 bits", (unsigned long long)start,
                    (unsigned long long)count);
    if (width < 20) {
        uint64_t p = 1;
        for (int k = 0; k < width; ++k) p *= 10u;
        if (start + count > p)
            return fail(HB_ERR_INVAL, "index range [%llu, %llu) does not fit in %d digits", (unsigned long long)start,
                        (unsigned long long)(start + count), width);
    }
    return HB_OK;
}

}  // namespace hb

using namespace hb;

// =========================================================================
// C ABI
// =========================================================================
extern "C" {

int hb_abi_version(void) { return HB_ABI_VERSION; }
const char* hb_last_error(void) { return g_err.c_str(); }
int hb_digest_len(int alg) { return digest_len(alg); }
uint64_t hb_launch_count(void) { return hb::launches_total(); }

int hb_device_count(int* n) {
    if (!n) return fail(HB_ERR_INVAL, "null pointer");
    *n = device_count();
    return HB_OK;
}

int hb_device_info(int ordinal, hb_device_info_t* info) {
    if (!info) return fail(HB_ERR_INVAL, "null pointer");
    const int nd = device_count();
    if (ordinal < 0 || ordinal >= nd) return fail(HB_ERR_NODEV, "device ordinal %d out of range", ordinal);
    cudaDeviceProp p;
    HB_CK(cudaGetDeviceProperties(&p, ordinal));
    memset(info, 0, sizeof *info);
    info->ordinal = ordinal;
    info->sm_count = p.multiProcessorCount;
    info->cc_major = p.major;
    info->cc_minor = p.minor;
    info->total_mem = p.totalGlobalMem;
    info->pci_bus_id = p.pciBusID;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, ordinal);
    info->clock_khz = clk;
    {
        DeviceGuard g(ordinal);
        size_t fr = 0, tot = 0;
        if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) info->free_mem = fr;
        cudaGetLastError();
    }
    snprintf(info->name, sizeof info->name, "%s", p.name);
    return HB_OK;
}

int hb_partition_range(int64_t lb, int64_t ub, const double* ratios, int k, int64_t* bounds_out) {
    if (!bounds_out) return fail(HB_ERR_INVAL, "null pointer");
    return partition(lb, ub, ratios, k, bounds_out);
}

int hb_hash_fixed(int alg, const uint8_t* msgs, uint64_t n, uint64_t msg_len, uint8_t* out, const int* gpus,
                  int n_gpus, uint32_t flags, hb_timing* t) {
    const int dlen = digest_len(alg);
    if (dlen < 0) return fail(HB_ERR_ALG, "unknown hash algorithm id %d", alg);
    if (t) memset(t, 0, sizeof *t);
    if (n == 0) return HB_OK;
    if (!out || (!msgs && msg_len)) return fail(HB_ERR_INVAL, "null buffer");
    if (msg_len && n > UINT64_MAX / msg_len) return fail(HB_ERR_INVAL, "n*msg_len overflows");
    std::vector<int> devs;
    int rc = resolve_gpus(gpus, n_gpus, n * msg_len, devs);
    if (rc) return rc;
    if (!t && devs.size() == 1 && small_batch_fits(n * msg_len, n, n * (uint64_t)dlen, false))
        return small_batch(0, alg, msgs, n * msg_len, nullptr, n, msg_len, out, n * (uint64_t)dlen, devs[0], flags);
    nvtxRangePushA("hb_hash_fixed");
    ShardJob j;
    j.kind = 0;
    j.alg = alg;
    j.msgs = msgs;
    j.msg_len = msg_len;
    j.out = out;
    j.flags = flags;
    j.in_pinned = is_pinned(msgs, n * msg_len);
    j.out_pinned = is_pinned(out, n * (uint64_t)dlen);
    rc = run_sharded(j, n, devs, t);
    nvtxRangePop();
    return rc;
}

int hb_hash_fixed_split(int alg, const uint8_t* msgs, uint64_t n, uint64_t msg_len, uint8_t* out, const int* gpus,
                        const double* ratios, int n_gpus, uint32_t flags, hb_timing* t) {
    const int dlen = digest_len(alg);
    if (dlen < 0) return fail(HB_ERR_ALG, "unknown hash algorithm id %d", alg);
    if (t) memset(t, 0, sizeof *t);
    if (!gpus || !ratios || n_gpus < 1) return fail(HB_ERR_INVAL, "need at least one (gpu, ratio) binding");
    int rc = check_ratios(ratios, n_gpus);
    if (rc) return rc;
    if (n == 0) return HB_OK;
    if (!out || (!msgs && msg_len)) return fail(HB_ERR_INVAL, "null buffer");
    if (msg_len && n > UINT64_MAX / msg_len) return fail(HB_ERR_INVAL, "n*msg_len overflows");
    std::vector<int> devs;
    rc = resolve_gpus(gpus, n_gpus, n * msg_len, devs);
    if (rc) return rc;
    ShardJob j;
    j.kind = 0;
    j.alg = alg;
    j.msgs = msgs;
    j.msg_len = msg_len;
    j.out = out;
    j.flags = flags;
    j.in_pinned = is_pinned(msgs, n * msg_len);
    j.out_pinned = is_pinned(out, n * (uint64_t)dlen);
    return run_sharded(j, n, devs, t, ratios);
}

int hb_hash_varlen(int alg, const uint8_t* data, const uint64_t* offsets, uint64_t n, uint8_t* out,
                   const int* gpus, int n_gpus, uint32_t flags, hb_timing* t) {
    const int dlen = digest_len(alg);
    if (dlen < 0) return fail(HB_ERR_ALG, "unknown hash algorithm id %d", alg);
    if (t) memset(t, 0, sizeof *t);
    if (n == 0) return HB_OK;
    if (!out || !offsets) return fail(HB_ERR_INVAL, "null buffer");
    for (uint64_t i = 0; i < n; ++i)
        if (offsets[i + 1] < offsets[i]) return fail(HB_ERR_INVAL, "offsets must be non-decreasing (at %llu)", (unsigned long long)i);
    if (!data && offsets[n] > offsets[0]) return fail(HB_ERR_INVAL, "null data");
    std::vector<int> devs;
    int rc = resolve_gpus(gpus, n_gpus, offsets[n] - offsets[0], devs);
    if (rc) return rc;
    if (!t && devs.size() == 1 && small_batch_fits(offsets[n] - offsets[0], n, n * (uint64_t)dlen, true))
        return small_batch(1, alg, data + offsets[0], offsets[n] - offsets[0], offsets, n, 0, out, n * (uint64_t)dlen,
                           devs[0], flags);
    nvtxRangePushA("hb_hash_varlen");
    ShardJob j;
    j.kind = 1;
    j.alg = alg;
    j.data = data;
    j.offsets = offsets;
    j.out = out;
    j.flags = flags;
    j.in_pinned = is_pinned(data + offsets[0], offsets[n] - offsets[0]);
    j.off_pinned = is_pinned(offsets, (n + 1) * 8);
    j.out_pinned = is_pinned(out, n * (uint64_t)dlen);
    rc = run_sharded(j, n, devs, t);
    nvtxRangePop();
    return rc;
}

int hb_digest_small(int alg, const uint8_t* msg, uint64_t len, uint8_t* out, int gpu) {
    const int dlen = digest_len(alg);
    if (dlen < 0) return fail(HB_ERR_ALG, "unknown hash algorithm id %d", alg);
    if (len > HB_DIGEST_SMALL_MAX)
        return fail(HB_ERR_INVAL, "message of %llu bytes exceeds HB_DIGEST_SMALL_MAX (%u)", (unsigned long long)len,
                    HB_DIGEST_SMALL_MAX);
    if (!out || (!msg && len)) return fail(HB_ERR_INVAL, "null buffer");
    const int nd = device_count();
    if (nd == 0) return fail(HB_ERR_NODEV, "no CUDA device visible");
    if (gpu < 0) gpu = nd > 1 ? pick_default_gpu(nd) : 0;
    else if (gpu >= nd) return fail(HB_ERR_NODEV, "device ordinal %d out of range (%d devices)", gpu, nd);
    DeviceGuard g(gpu);
    SlotLease lease(gpu);
    SmallSlot& sl = lease.sl;
    if (int rc = take_slot(gpu, sl)) return rc;
    if (tuning().small_poll) {
        // Spin on the slot's sequence word (a few us sooner than a stream
        // synchronise); a launch that fails never publishes, so the stream is
        // queried now and then and its error returned.
        sl.seq = sl.seq + 1 ? sl.seq + 1 : 1;
        HB_CK(launch_digest_small(alg, msg, len, sl.d_out, sl.seq, sl.stream));
        const volatile uint32_t* flag = reinterpret_cast<const volatile uint32_t*>(sl.h_out + 48);
        for (uint32_t k = 1; *flag != sl.seq; ++k) {
#if defined(__x86_64__)
            __builtin_ia32_pause();
#endif
            if ((k & 1023u) == 0) {
                const cudaError_t e = cudaStreamQuery(sl.stream);
                if (e == cudaSuccess && *flag != sl.seq)
                    return fail(HB_ERR_CUDA, "hb_digest_small: kernel completed without publishing its digest");
                if (e != cudaSuccess && e != cudaErrorNotReady) HB_CK(e);
            }
        }
        std::atomic_thread_fence(std::memory_order_acquire);
    } else {
        HB_CK(launch_digest_small(alg, msg, len, sl.d_out, 0, sl.stream));
        HB_CK(cudaStreamSynchronize(sl.stream));
    }
    memcpy(out, sl.h_out, (size_t)dlen);
    return HB_OK;
}

int hb_hash_decimal(int alg, uint64_t start, uint64_t count, int width, uint8_t* out, const int* gpus, int n_gpus,
                    uint32_t flags, hb_timing* t) {
    const int dlen = digest_len(alg);
    if (dlen < 0) return fail(HB_ERR_ALG, "unknown hash algorithm id %d", alg);
    if (t) memset(t, 0, sizeof *t);
    if (width < 1 || width > 20) return fail(HB_ERR_INVAL, "width must be in [1, 20] for on-device generation");
    if (count == 0) return HB_OK;
    if (!out) return fail(HB_ERR_INVAL, "null buffer");
    int rc = check_decimal_range(start, count, width);
    if (rc) return rc;
    std::vector<int> devs;
    rc = resolve_gpus(gpus, n_gpus, count * (uint64_t)dlen, devs);
    if (rc) return rc;
    ShardJob j;
    j.kind = 2;
    j.alg = alg;
    j.start = start;
    j.width = width;
    j.out = out;
    j.flags = flags;
    j.out_pinned = is_pinned(out, count * (uint64_t)dlen);
    return run_sharded(j, count, devs, t);
}

int hb_hash_fixed_dev(int alg, int gpu, const void* d_msgs, uint64_t n, uint64_t msg_len, void* d_out, void* stream,
                      uint32_t flags) {
    if (digest_len(alg) < 0) return fail(HB_ERR_ALG, "unknown hash algorithm id %d", alg);
    if (n == 0) return HB_OK;
    if (!d_out || (!d_msgs && msg_len)) return fail(HB_ERR_INVAL, "null buffer");
    const int nd = device_count();
    if (gpu < 0 || gpu >= nd) return fail(HB_ERR_NODEV, "device ordinal %d out of range (%d devices)", gpu, nd);
    DeviceGuard g(gpu);
    HB_CK(launch_fixed(alg, static_cast<const uint8_t*>(d_msgs), n, msg_len, static_cast<uint8_t*>(d_out),
                       static_cast<cudaStream_t>(stream), flags));
    return HB_OK;
}

uint64_t hb_varlen_scratch_bytes(uint64_t n) { return varlen_scratch_bytes(n); }

int hb_hash_varlen_dev(int alg, int gpu, const void* d_data, uint64_t data_bytes, const uint64_t* d_offsets,
                       uint64_t offset_base, uint64_t n, void* d_out, void* d_scratch, void* stream, uint32_t flags) {
    if (digest_len(alg) < 0) return fail(HB_ERR_ALG, "unknown hash algorithm id %d", alg);
    if (n == 0) return HB_OK;
    if (!d_out || !d_offsets) return fail(HB_ERR_INVAL, "null buffer");
    const int nd = device_count();
    if (gpu < 0 || gpu >= nd) return fail(HB_ERR_NODEV, "device ordinal %d out of range (%d devices)", gpu, nd);
    DeviceGuard g(gpu);
    HB_CK(launch_varlen(alg, static_cast<const uint8_t*>(d_data), data_bytes, d_offsets, offset_base, n,
                        static_cast<uint8_t*>(d_out), d_scratch, static_cast<cudaStream_t>(stream), flags));
    return HB_OK;
}

int hb_hash_decimal_dev(int alg, int gpu, uint64_t start, uint64_t count, int width, void* d_out, void* stream) {
    if (digest_len(alg) < 0) return fail(HB_ERR_ALG, "unknown hash algorithm id %d", alg);
    if (width < 1 || width > 20) return fail(HB_ERR_INVAL, "width must be in [1, 20]");
    if (count == 0) return HB_OK;
    if (!d_out) return fail(HB_ERR_INVAL, "null buffer");
    if (int rc = check_decimal_range(start, count, width)) return rc;
    const int nd = device_count();
    if (gpu < 0 || gpu >= nd) return fail(HB_ERR_NODEV, "device ordinal %d out of range (%d devices)", gpu, nd);
    DeviceGuard g(gpu);
    HB_CK(launch_decimal(alg, start, count, width, static_cast<uint8_t*>(d_out), static_cast<cudaStream_t>(stream)));
    return HB_OK;
}

int hb_fill_random_dev(int gpu, void* d_buf, uint64_t nbytes, uint64_t seed, uint64_t byte_offset, void* stream) {
    if (nbytes == 0) return HB_OK;
    if (!d_buf || (reinterpret_cast<uintptr_t>(d_buf) & 7u) || (byte_offset & 7u))
        return fail(HB_ERR_INVAL, "d_buf and byte_offset must be 8-byte aligned");
    const int nd = device_count();
    if (gpu < 0 || gpu >= nd) return fail(HB_ERR_NODEV, "device ordinal %d out of range (%d devices)", gpu, nd);
    DeviceGuard g(gpu);
    HB_CK(launch_fill_random(static_cast<uint8_t*>(d_buf), nbytes, seed, byte_offset, static_cast<cudaStream_t>(stream)));
    return HB_OK;
}

int hb_gen_decimal_dev(int gpu, uint64_t start, uint64_t count, int width, void* d_out, void* stream) {
    if (width < 1) return fail(HB_ERR_INVAL, "width must be positive");
    if (count == 0) return HB_OK;
    if (int rc = check_decimal_range(start, count, width)) return rc;
    if (!d_out) return fail(HB_ERR_INVAL, "null buffer");
    const int nd = device_count();
    if (gpu < 0 || gpu >= nd) return fail(HB_ERR_NODEV, "device ordinal %d out of range (%d devices)", gpu, nd);
    DeviceGuard g(gpu);
    HB_CK(launch_gen_decimal(start, count, width, static_cast<uint8_t*>(d_out), static_cast<cudaStream_t>(stream)));
    return HB_OK;
}

void* hb_alloc_pinned(uint64_t bytes) {
    if (!bytes) bytes = 1;
    void* p = nullptr;
    cudaError_t e = cudaHostAlloc(&p, bytes, cudaHostAllocPortable);
    if (e != cudaSuccess) {
        cudaGetLastError();
        fail(HB_ERR_NOMEM, "cudaHostAlloc(%llu) failed: %s", (unsigned long long)bytes, cudaGetErrorString(e));
        return nullptr;
    }
    return p;
}

int hb_free_pinned(void* p) {
    if (!p) return HB_OK;
    HB_CK(cudaFreeHost(p));
    return HB_OK;
}

int hb_sync_device(int gpu) {
    const int nd = device_count();
    if (gpu < 0 || gpu >= nd) return fail(HB_ERR_NODEV, "device ordinal %d out of range (%d devices)", gpu, nd);
    DeviceGuard g(gpu);
    HB_CK(cudaDeviceSynchronize());
    return HB_OK;
}

// ---- peer-mapped digest buffers (fused gather) -------------------------
// IPC handles name whole cudaMalloc allocations; a pointer inside one (e.g. a
// tensor carved out of PyTorch's caching allocator) is exported as the
// handle of its allocation plus the byte offset of the pointer in it.
typedef CUresult (*PFN_memGetAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr);
static PFN_memGetAddressRange get_mem_range() {
    static PFN_memGetAddressRange fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuMemGetAddressRange", &p, 12000, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_memGetAddressRange>(p);
    });
    return fn;
}

int hb_ipc_handle(const void* d_ptr, uint8_t* handle_out, uint64_t* offset_out) {
    if (!d_ptr || !handle_out || !offset_out) return fail(HB_ERR_INVAL, "null pointer");
    static_assert(sizeof(cudaIpcMemHandle_t) == HB_IPC_HANDLE_BYTES, "IPC handle size");
    cudaPointerAttributes a;
    HB_CK(cudaPointerGetAttributes(&a, d_ptr));
    if (a.type != cudaMemoryTypeDevice) return fail(HB_ERR_INVAL, "not a device allocation");
    DeviceGuard g(a.device);
    PFN_memGetAddressRange range = get_mem_range();
    if (!range) return fail(HB_ERR_CUDA, "cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, reinterpret_cast<CUdeviceptr>(d_ptr)) != CUDA_SUCCESS)
        return fail(HB_ERR_CUDA, "cuMemGetAddressRange failed");
    cudaIpcMemHandle_t h;
    HB_CK(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
    memcpy(handle_out, &h, sizeof h);
    *offset_out = reinterpret_cast<uint64_t>(d_ptr) - (uint64_t)base;
    return HB_OK;
}

int hb_ipc_open(int gpu, const uint8_t* handle, void** d_ptr_out) {
    if (!handle || !d_ptr_out) return fail(HB_ERR_INVAL, "null pointer");
    const int nd = device_count();
    if (gpu < 0 || gpu >= nd) return fail(HB_ERR_NODEV, "device ordinal %d out of range (%d devices)", gpu, nd);
    DeviceGuard g(gpu);
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof h);
    HB_CK(cudaIpcOpenMemHandle(d_ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
    return HB_OK;
}

int hb_ipc_close(int gpu, void* d_ptr) {
    if (!d_ptr) return HB_OK;
    const int nd = device_count();
    if (gpu < 0 || gpu >= nd) return fail(HB_ERR_NODEV, "device ordinal %d out of range (%d devices)", gpu, nd);
    DeviceGuard g(gpu);
    HB_CK(cudaIpcCloseMemHandle(d_ptr));
    return HB_OK;
}

int hb_tuning_reload(void) {
    tuning_reload();
    return HB_OK;
}

int hb_built_with_ab(void) { return built_with_ab() ? 1 : 0; }

int hb_last_kernel_name(char* buf, int cap) {
    if (!buf || cap < 1) return fail(HB_ERR_INVAL, "null buffer");
    buf[0] = '\0';
    const void* fn = last_hash_kernel();
    if (!fn) return fail(HB_ERR_INVAL, "no hash kernel launched by this thread yet");
    const char* mangled = nullptr;
    HB_CK(cudaFuncGetName(&mangled, fn));
    int st = 0;
    char* dem = abi::__cxa_demangle(mangled, nullptr, nullptr, &st);
    snprintf(buf, (size_t)cap, "%s", st == 0 && dem ? dem : mangled);
    free(dem);
    return HB_OK;
}

int hb_last_timeline(hb_span* out, int cap) {
    const int n = (int)t_timeline.size();
    if (out)
        for (int i = 0; i < n && i < cap; ++i) out[i] = t_timeline[i];
    return n;
}

int hb_engine_budget(int gpu, uint64_t* budget, uint64_t* chunk_cap) {
    if (!budget || !chunk_cap) return fail(HB_ERR_INVAL, "null pointer");
    GpuCtx* c = nullptr;
    int rc = get_ctx(gpu, &c);
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(gpu);
    rc = ctx_init(*c);
    if (rc) return rc;
    *budget = c->budget;
    *chunk_cap = std::min(c->chunk_cap, tuning().chunk_bytes);
    return HB_OK;
}

int hb_shutdown(void) {
    std::vector<Worker*> ws;
    {
        std::lock_guard<std::mutex> lk(g_ctx_mu);
        ws.swap(g_workers);
    }
    for (Worker* w : ws) {
        if (!w) continue;
        {
            std::lock_guard<std::mutex> lk(w->mu);
            w->stop = true;
        }
        w->cv.notify_one();
        w->th.join();
        delete w;
    }
    {
        std::lock_guard<std::mutex> lk(g_small_mu);
        for (size_t d = 0; d < g_small.size(); ++d) {
            if (g_small[d].empty()) continue;
            DeviceGuard g((int)d);
            for (SmallSlot& sl : g_small[d]) {
                cudaStreamSynchronize(sl.stream);
                cudaStreamDestroy(sl.stream);
                cudaFreeHost(sl.h_out);
                if (sl.zc) cudaFreeHost(sl.zc);
            }
        }
        g_small.clear();
    }
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    for (auto& cp : g_ctx) {
        if (!cp) continue;
        std::lock_guard<std::mutex> lk2(cp->mu);
        DeviceGuard g(cp->dev);
        for (Slot& s : cp->slots) {
            if (s.stream) cudaStreamSynchronize(s.stream);
            if (s.d_in.p) cudaFree(s.d_in.p);
            if (s.d_out.p) cudaFree(s.d_out.p);
            if (s.d_off.p) cudaFree(s.d_off.p);
            if (s.d_scratch.p) cudaFree(s.d_scratch.p);
            if (s.h_in.p) cudaFreeHost(s.h_in.p);
            if (s.h_out.p) cudaFreeHost(s.h_out.p);
            if (s.h_off.p) cudaFreeHost(s.h_off.p);
            for (auto& e : s.ev)
                if (e) cudaEventDestroy(e);
            if (s.stream) cudaStreamDestroy(s.stream);
        }
        if (cp->ev_ref) cudaEventDestroy(cp->ev_ref);
        cp.reset();
    }
    g_ctx.clear();
    return HB_OK;
}

}  // extern "C"
