// hb_kernels.cu -- sm_100a kernels of the batched-hash engine and their
// launchers.  One thread owns one message: chaining state and message
// schedule live in registers; message bytes reach the thread either through a
// TMA-staged, 64B-swizzled shared-memory ring (fixed width, 16B-aligned rows:
// the HBM-streaming hot path) or through direct unaligned loads (any width,
// variable length).  Padding is generated in registers (md_finish) -- the
// padded (n, nblocks, 16) array of the reference (batch.py:128-138) never
// exists in memory.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <mutex>

#include "hb_algos.cuh"
#include "hb_internal.h"
#include "hb_ptx.cuh"
#include "../../include/hetoc_b200.h"
#include "hb_kernels.cuh"

namespace hb {

// ------------------------------------------------------------------ tuning --
static uint64_t env_u64(const char* name, uint64_t dflt) {
    const char* v = getenv(name);
    if (!v || !*v) return dflt;
    char* end = nullptr;
    const unsigned long long x = strtoull(v, &end, 0);
    return (end && *end == '\0') ? (uint64_t)x : dflt;
}
#ifdef HB_AB
static bool env_set(const char* name) {
    const char* v = getenv(name);
    return v && *v;
}
#endif

static Tuning parse_tuning() {
    Tuning t;
    t.chunk_bytes = std::max<uint64_t>(1ull << 16, env_u64("HB_CHUNK_BYTES", t.chunk_bytes));
    t.pipe_min_out = env_u64("HB_PIPE_MIN_OUT", t.pipe_min_out);
    t.pipe_chunks = std::max<uint64_t>(1, env_u64("HB_PIPE_CHUNKS", t.pipe_chunks));
    t.min_chunk_bytes = std::max<uint64_t>(1ull << 16, env_u64("HB_MIN_CHUNK_BYTES", t.min_chunk_bytes));
    t.memcpy_threads = env_u64("HB_MEMCPY_THREADS", 0);
    t.bind_numa = env_u64("HB_BIND_NUMA", 1) != 0;
    t.multi_gpu_min_bytes = env_u64("HB_MULTI_GPU_MIN_BYTES", t.multi_gpu_min_bytes);
    t.device_reserve = env_u64("HB_DEVICE_RESERVE", t.device_reserve);
    t.pdl = env_u64("HB_PDL", 1) != 0;
    t.small_n = env_u64("HB_SMALL_N", t.small_n);
    t.chain_n = env_u64("HB_CHAIN_N", t.chain_n);
    t.md5_nb3_n = env_u64("HB_MD5_NB3_N", t.md5_nb3_n);
    t.late_wait = env_u64("HB_LATE_WAIT", 1) != 0;
    t.trigger_wave_pct = (uint32_t)env_u64("HB_TRIGGER_WAVE_PCT", 100);
    t.varlen_pf = env_u64("HB_VARLEN_PF", 1) != 0;
    t.sort_qmajor = env_u64("HB_SORT_QMAJOR", 1) != 0;
    t.direct_max_len = env_u64("HB_DIRECT_MAX_L", t.direct_max_len);
    t.small_pair = env_u64("HB_SMALL_PAIR", 1) != 0;
    t.dec_run = env_u64("HB_DEC_RUN", 1) != 0;
    t.small_poll = env_u64("HB_SMALL_POLL", 1) != 0;
    t.zc_max_bytes = std::min<uint64_t>(env_u64("HB_ZERO_COPY_MAX", t.zc_max_bytes), 16ull << 20);
    if (const char* v = getenv("HB_VARLEN_SORT")) t.varlen_sort = strcmp(v, "global") == 0 ? 0 : 1;
#ifdef HB_AB
    static const char* const kCfgNames[] = {"1x3", "2x2", "2x3", "ws2", "ws3", "1x2", "ws2x2", "ws3x2",
                                            "ws3u", "ws3x2u", "ws3n", "w1x1", "w1x2", "w1x4", "w1x4s2", "w1x2p", "ws3v6", "w1x2s4", "w1x2s2", "w1x3", "w1x4p"};
    if (const char* v = getenv("HB_TMA_CFG"))
        for (int k = 0; k < (int)(sizeof kCfgNames / sizeof *kCfgNames); ++k)
            if (!strcmp(v, kCfgNames[k])) t.tma_cfg = k;
    if (const char* v = getenv("HB_VARIANT"))
        if (*v >= '0' && *v <= '9' && v[1] == '\0') t.variant = *v - '0';
    if (t.tma_cfg >= 0) t.direct_max_len = env_u64("HB_DIRECT_MAX_L", 0);  // a forced tile applies to every width
    t.tma_l2 = (uint32_t)env_u64("HB_TMA_L2", 256);
    t.tma_evict_first = (uint32_t)env_u64("HB_TMA_EVICT_FIRST", 0);
    t.small_kernel = !env_set("HB_NO_SMALL_KERNEL");
    t.const_variant = env_set("HB_CONST_VARIANT") ? (int)env_u64("HB_CONST_VARIANT", 1) : -1;
    t.small_cta = (uint32_t)env_u64("HB_SMALL_CTA", 128);
    t.small_pair_all = env_u64("HB_SMALL_PAIR_ALL", 0) != 0;
    t.input_ready = env_u64("HB_INPUT_READY", 0) != 0;
    t.small_kernel_ab = t.const_variant == 0 || t.const_variant == 3 || t.const_variant == 4 || t.small_cta != 128 ||
                        t.small_pair_all;
    t.dec_pair = env_set("HB_DEC_PAIR") ? (int)env_u64("HB_DEC_PAIR", 0) : -1;
    t.fma_digits = env_u64("HB_FMA_DIGITS", 1) != 0;
    t.dec_ab = t.dec_pair >= 0 || !t.fma_digits || t.const_variant >= 0;
    t.sort_window = (uint32_t)env_u64("HB_SORT_WINDOW", 8192);
    t.varlen_ld = (uint32_t)env_u64("HB_VARLEN_LD", 16);
    t.varlen_q = (uint32_t)env_u64("HB_VARLEN_Q", 8);
    t.varlen_prefetch = (uint32_t)env_u64("HB_VARLEN_PREFETCH", 0);
    t.varlen_bulk = (uint32_t)env_u64("HB_VARLEN_BULK", 0);
    t.varlen_kernel = env_set("HB_VARLEN_KERNEL") ? (int)env_u64("HB_VARLEN_KERNEL", 0) : -1;
    t.vc_stages = env_set("HB_VC_STAGES") ? (int)env_u64("HB_VC_STAGES", 4) : -1;
    t.vc_pf = (uint32_t)env_u64("HB_VC_PF", 256);
#endif
    return t;
}

static Tuning g_tuning;
static std::once_flag g_tuning_once;
const Tuning& tuning() {
    std::call_once(g_tuning_once, [] { g_tuning = parse_tuning(); });
    return g_tuning;
}
// Not synchronised against concurrent launches: call it between hash calls
// (tests and A/B tools do, after changing the environment).
void tuning_reload() {
    tuning();
    g_tuning = parse_tuning();
}
bool built_with_ab() {
#ifdef HB_AB
    return true;
#else
    return false;
#endif
}

// ----------------------------------------------------------- bookkeeping --
static std::atomic<uint64_t> g_launches{0};
static thread_local const void* t_last_hash_kernel = nullptr;
void note_launches(uint64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
void note_launch(const void* kernel, bool hash_kernel) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (hash_kernel) t_last_hash_kernel = kernel;
}
const void* last_hash_kernel() { return t_last_hash_kernel; }
void set_last_hash_kernel(const void* kernel) { t_last_hash_kernel = kernel; }
uint64_t launches_total() { return g_launches.load(std::memory_order_relaxed); }

// The global sort's four kernels may run as programmatic dependents
// (HB_FLAG_INPUT_READY, launch_varlen_sort): k_sort_zero starts while the
// previous varlen hash kernel drains (released once every thread of it has
// read its permutation entry); each later kernel does its offsets-only work
// first and calls griddepcontrol.wait before touching the shared counters or
// the permutation.  Launched normally, the waits and triggers are no-ops.
__global__ void __launch_bounds__(1024) k_sort_zero(uint32_t* __restrict__ hist) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    for (int k = threadIdx.x; k < kSortBuckets; k += 1024) hist[k] = 0;
}

__global__ void __launch_bounds__(kSortThreads) k_sort_hist(const uint64_t* __restrict__ offsets, uint64_t n,
                                                            uint64_t addr_bias, uint32_t* __restrict__ hist) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    __shared__ uint32_t h[kSortBuckets];
    for (int k = threadIdx.x; k < kSortBuckets; k += kSortThreads) h[k] = 0;
    __syncthreads();
    const uint64_t base = (uint64_t)blockIdx.x * kSortThreads * kSortItems;
#pragma unroll 4
    for (int it = 0; it < kSortItems; ++it) {
        const uint64_t i = base + (uint64_t)it * kSortThreads + threadIdx.x;
        if (i < n) atomicAdd(&h[sort_bucket(offsets, i, addr_bias)], 1u);
    }
    __syncthreads();
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the counters are zeroed
    for (int k = threadIdx.x; k < kSortBuckets; k += kSortThreads)
        if (h[k]) atomicAdd(&hist[k], h[k]);
}

__global__ void __launch_bounds__(1024) k_sort_scan(uint32_t* __restrict__ hist) {
    // exclusive scan of kSortBuckets in place; thread t owns kPer consecutive buckets
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    constexpr int kPer = kSortBuckets / 1024;
    __shared__ uint32_t warp_sums[32];
    const int t = threadIdx.x;
    uint32_t v[kPer];
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kPer; ++k) { v[k] = hist[kPer * t + k]; s += v[k]; }
    uint32_t incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if ((t & 31) >= o) incl += x;
    }
    if ((t & 31) == 31) warp_sums[t >> 5] = incl;
    __syncthreads();
    if (t < 32) {
        uint32_t w = warp_sums[t], wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_up_sync(0xFFFFFFFFu, wi, o);
            if (t >= o) wi += x;
        }
        warp_sums[t] = wi - w;  // exclusive warp prefix
    }
    __syncthreads();
    uint32_t run = warp_sums[t >> 5] + incl - s;
#pragma unroll
    for (int k = 0; k < kPer; ++k) { hist[kPer * t + k] = run; run += v[k]; }
}

__global__ void __launch_bounds__(kSortThreads) k_sort_scatter(const uint64_t* __restrict__ offsets, uint64_t n,
                                                               uint64_t addr_bias, uint32_t* __restrict__ cursor,
                                                               uint32_t* __restrict__ perm) {
    __shared__ uint32_t h[kSortBuckets];
    __shared__ uint32_t base[kSortBuckets];
    for (int k = threadIdx.x; k < kSortBuckets; k += kSortThreads) h[k] = 0;
    __syncthreads();
    const uint64_t b0 = (uint64_t)blockIdx.x * kSortThreads * kSortItems;
    uint32_t bucket[kSortItems];
#pragma unroll
    for (int it = 0; it < kSortItems; ++it) {
        const uint64_t i = b0 + (uint64_t)it * kSortThreads + threadIdx.x;
        bucket[it] = (i < n) ? sort_bucket(offsets, i, addr_bias) : 0xFFFFFFFFu;
        if (i < n) atomicAdd(&h[bucket[it]], 1u);
    }
    __syncthreads();
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the cursors are scanned
    for (int k = threadIdx.x; k < kSortBuckets; k += kSortThreads) {
        base[k] = h[k] ? atomicAdd(&cursor[k], h[k]) : 0u;
        h[k] = 0;
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < kSortItems; ++it) {
        const uint64_t i = b0 + (uint64_t)it * kSortThreads + threadIdx.x;
        if (bucket[it] != 0xFFFFFFFFu) perm[base[bucket[it]] + atomicAdd(&h[bucket[it]], 1u)] = (uint32_t)i;
    }
}

// Windowed variant (the default): the same (block count, alignment) key, but
// sorted only inside windows of kSortWindow consecutive messages, one CTA per
// window, in shared memory.  Warps still see near-equal lengths (a window of
// 4,096 messages has ~60 per block-count class at U(1, 4096)) while the
// messages a window's warps read concurrently stay within a few MB of each
// other: L2 lines fetched for one message (256 B promotion) are still
// resident when its neighbours are hashed, instead of being re-fetched from
// HBM after a global sort scattered the neighbours across the whole batch.
template <int kSortWindow, int Q, bool QMAJOR = false>
__global__ void __launch_bounds__(1024) k_sort_window(const uint64_t* __restrict__ offsets, uint64_t n,
                                                      uint64_t addr_bias, uint32_t* __restrict__ perm) {
    constexpr int kBuckets = kSortNbClasses * Q;
    __shared__ uint32_t h[kBuckets];
    __shared__ uint32_t wsum[32];
    const uint32_t t = threadIdx.x;
    const uint64_t w0 = (uint64_t)blockIdx.x * kSortWindow;
    for (int k = t; k < kBuckets; k += 1024) h[k] = 0;
    __syncthreads();
    constexpr int kItems = kSortWindow / 1024;
    uint32_t key[kItems], rank[kItems];
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
        const uint64_t i = w0 + (uint64_t)it * 1024u + t;
        key[it] = 0xFFFFFFFFu;
        if (i < n) {
            key[it] = sort_bucket_q<Q, QMAJOR>(offsets, i, addr_bias);
            rank[it] = atomicAdd(&h[key[it]], 1u);
        }
    }
    __syncthreads();
    // exclusive scan of the bucket counts; thread t owns buckets kPer*t .. kPer*t + kPer-1
    constexpr int kPer = kBuckets / 1024;
    uint32_t v[kPer], sum = 0;
#pragma unroll
    for (int k = 0; k < kPer; ++k) { v[k] = h[kPer * t + k]; sum += v[k]; }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if ((t & 31) >= (uint32_t)o) incl += x;
    }
    if ((t & 31) == 31) wsum[t >> 5] = incl;
    __syncthreads();
    if (t < 32) {
        const uint32_t w = wsum[t];
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_up_sync(0xFFFFFFFFu, wi, o);
            if (t >= (uint32_t)o) wi += x;
        }
        wsum[t] = wi - w;
    }
    __syncthreads();
    uint32_t run = wsum[t >> 5] + incl - sum;
#pragma unroll
    for (int k = 0; k < kPer; ++k) { h[kPer * t + k] = run; run += v[k]; }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < kItems; ++it)
        if (key[it] != 0xFFFFFFFFu) perm[w0 + h[key[it]] + rank[it]] = (uint32_t)(w0 + (uint64_t)it * 1024u + t);
}

// Length/alignment-bucket permutation for the varlen kernels (null when not
// sorting).  Shared by the per-algorithm translation units.
cudaError_t launch_varlen_sort(int alg, const uint8_t* d_data, const uint64_t* d_offsets, uint64_t offset_base,
                               uint64_t n, void* d_scratch, cudaStream_t stream, uint32_t flags,
                               const uint32_t** perm_out, int qclasses) {
    const uint32_t* perm = nullptr;
    const uint64_t bias0 = reinterpret_cast<uintptr_t>(d_data) - offset_base;  // address = offsets[i] + bias
    // Sort mode: windowed for MD5 (HBM-bound: locality wins), global for SHA-1/SM3
    // (ALU-bound: full (block count, alignment) uniformity wins); B200 A/B in
    // profiles/ab_varlen_r1b.txt.  $HB_VARLEN_SORT = window | global, $HB_SORT_WINDOW.
    const Tuning& T = tuning();
    const bool window = T.varlen_sort >= 0 ? T.varlen_sort == 1 : alg == kMd5;
    if (!(flags & HB_FLAG_NO_SORT) && n >= 1024 && d_scratch && window) {
        uint32_t* p = static_cast<uint32_t*>(d_scratch) + kSortBuckets;
#ifdef HB_AB
        const uint64_t w = T.sort_window;
        const bool q8 = qclasses == 8;
#define HB_WIN(W)                                                                                            \
    q8 ? (T.sort_qmajor ? k_sort_window<W, 8, true><<<(unsigned)((n + W - 1) / W), 1024, 0, stream>>>(d_offsets, n, bias0, p) \
                        : k_sort_window<W, 8><<<(unsigned)((n + W - 1) / W), 1024, 0, stream>>>(d_offsets, n, bias0, p)) \
    : T.sort_qmajor ? k_sort_window<W, 4, true><<<(unsigned)((n + W - 1) / W), 1024, 0, stream>>>(d_offsets, n, bias0, p) \
       : k_sort_window<W, 4><<<(unsigned)((n + W - 1) / W), 1024, 0, stream>>>(d_offsets, n, bias0, p)
        if (w >= 16384)
            HB_WIN(16384);
        else if (w >= 8192)
            HB_WIN(8192);
        else
            HB_WIN(4096);
#undef HB_WIN
#else
        (void)qclasses;
        const unsigned g = (unsigned)((n + 8191) / 8192);
        if (T.sort_qmajor && (flags & HB_FLAG_INPUT_READY) && T.pdl) {
            // HB_FLAG_INPUT_READY: the offsets are not written by the preceding
            // kernel, so the sort may start while it drains (programmatic
            // dependent launch without griddepcontrol.wait).  A preceding
            // k_varlen16l releases it once all its threads have read their
            // permutation entries, so overwriting perm here is safe; any other
            // preceding kernel releases it at its end or after its last read of
            // the scratch.  41 us of a 1.93 ms configs[3] step
            // (profiles/r2/launches_varlen_r2ab.csv) overlap the previous step.
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(g);
            cfg.blockDim = dim3(1024);
            cfg.stream = stream;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, k_sort_window<8192, 4, true>, d_offsets, n, bias0, p);
        } else if (T.sort_qmajor) {
            k_sort_window<8192, 4, true><<<g, 1024, 0, stream>>>(d_offsets, n, bias0, p);
        } else {
            k_sort_window<8192, 4><<<g, 1024, 0, stream>>>(d_offsets, n, bias0, p);
        }
#endif
        note_launch(nullptr, false);
        perm = p;
    } else if (!(flags & HB_FLAG_NO_SORT) && n >= 1024 && d_scratch) {
        uint32_t* hist = static_cast<uint32_t*>(d_scratch);
        uint32_t* p = hist + kSortBuckets;
        const uint64_t per_cta = (uint64_t)kSortThreads * kSortItems;
        const unsigned g = (unsigned)((n + per_cta - 1) / per_cta);
        const uint64_t bias = reinterpret_cast<uintptr_t>(d_data) - offset_base;  // address = offsets[i] + bias
        // HB_FLAG_INPUT_READY: programmatic dependents, so the sort runs while the
        // previous varlen step drains (see k_sort_zero); otherwise plain launches.
        const bool pdl = (flags & HB_FLAG_INPUT_READY) && T.pdl;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        const auto launch = [&](auto kernel, unsigned grid, unsigned block, auto... args) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(grid);
            cfg.blockDim = dim3(block);
            cfg.stream = stream;
            cfg.attrs = at;
            cfg.numAttrs = pdl ? 1 : 0;
            return cudaLaunchKernelEx(&cfg, kernel, args...);
        };
        cudaError_t e = launch(k_sort_zero, 1u, 1024u, hist);
        if (e == cudaSuccess) e = launch(k_sort_hist, g, (unsigned)kSortThreads, d_offsets, n, bias, hist);
        if (e == cudaSuccess) e = launch(k_sort_scan, 1u, 1024u, hist);
        if (e == cudaSuccess) e = launch(k_sort_scatter, g, (unsigned)kSortThreads, d_offsets, n, bias, hist, p);
        if (e != cudaSuccess) return e;
        note_launches(4);
        perm = p;
    }
    *perm_out = perm;
    return cudaGetLastError();
}

// ------------------------------------------------------- synthetic bytes --
__device__ __forceinline__ uint64_t mix64(uint64_t seed, uint64_t idx) {  // == oracle mix64
    uint64_t z = (idx + 1ull) * 0x9E3779B97F4A7C15ull + seed * 0xD1B54A32D192ED03ull;
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27; z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

__global__ void k_fill_random(uint8_t* __restrict__ buf, uint64_t nbytes, uint64_t seed, uint64_t w0) {
    const uint64_t nwords = (nbytes + 7) / 8;
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwords;
         w += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t v = mix64(seed, w0 + w);
        if (8 * w + 8 <= nbytes) {
            reinterpret_cast<uint64_t*>(buf)[w] = v;
        } else {
            for (uint64_t k = 0; 8 * w + k < nbytes; ++k) buf[8 * w + k] = (uint8_t)(v >> (8 * k));
        }
    }
}

__global__ void k_gen_decimal(uint64_t start, uint64_t count, int width, uint8_t* __restrict__ out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    uint64_t v = start + i;
    for (int pos = width - 1; pos >= 0; --pos) {
        out[i * (uint64_t)width + pos] = (uint8_t)('0' + v % 10u);
        v /= 10u;
    }
}

// =========================================================================
// Host-side launchers
// =========================================================================

PFN_encodeTiled get_encode_tiled() {
    static PFN_encodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(p);
    });
    return fn;
}

static thread_local char g_tma_err[kTmaErrLen];
const char* tma_error() { return g_tma_err; }
char* tma_error_buf() { return g_tma_err; }

// Per-algorithm launchers (hb_alg_*.cu).
#define HB_DECL(A)                                                                                               \
    cudaError_t launch_fixed_##A(const uint8_t*, uint64_t, uint64_t, uint8_t*, cudaStream_t, uint32_t);          \
    cudaError_t launch_varlen_##A(const uint8_t*, uint64_t, const uint64_t*, uint64_t, uint64_t, uint8_t*, void*, \
                                  cudaStream_t, uint32_t);                                                      \
    cudaError_t launch_decimal_##A(uint64_t, uint64_t, int, uint8_t*, cudaStream_t);
HB_DECL(sha1)
HB_DECL(md5)
HB_DECL(sm3)
#undef HB_DECL

cudaError_t launch_fixed(int alg, const uint8_t* d_msgs, uint64_t n, uint64_t msg_len, uint8_t* d_out,
                         cudaStream_t stream, uint32_t flags) {
    if (n == 0) return cudaSuccess;
    switch (alg) {
    case kSha1: return launch_fixed_sha1(d_msgs, n, msg_len, d_out, stream, flags);
    case kMd5: return launch_fixed_md5(d_msgs, n, msg_len, d_out, stream, flags);
    case kSm3: return launch_fixed_sm3(d_msgs, n, msg_len, d_out, stream, flags);
    default: return cudaErrorInvalidValue;
    }
}

uint64_t varlen_scratch_bytes(uint64_t n) { return (uint64_t)kSortBuckets * 4u + n * 4u + 256u; }

cudaError_t launch_varlen(int alg, const uint8_t* d_data, uint64_t data_bytes, const uint64_t* d_offsets,
                          uint64_t offset_base, uint64_t n, uint8_t* d_out, void* d_scratch, cudaStream_t stream,
                          uint32_t flags) {
    if (n == 0) return cudaSuccess;
    if (n >= (1ull << 32)) return cudaErrorInvalidValue;
    switch (alg) {
    case kSha1: return launch_varlen_sha1(d_data, data_bytes, d_offsets, offset_base, n, d_out, d_scratch, stream, flags);
    case kMd5: return launch_varlen_md5(d_data, data_bytes, d_offsets, offset_base, n, d_out, d_scratch, stream, flags);
    case kSm3: return launch_varlen_sm3(d_data, data_bytes, d_offsets, offset_base, n, d_out, d_scratch, stream, flags);
    default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_fill_random(uint8_t* d_buf, uint64_t nbytes, uint64_t seed, uint64_t byte_offset,
                               cudaStream_t stream) {
    if (nbytes == 0) return cudaSuccess;
    const uint64_t nwords = (nbytes + 7) / 8;
    uint64_t grid = (nwords + 255) / 256;
    if (grid > 148ull * 64) grid = 148ull * 64;
    k_fill_random<<<(unsigned)grid, 256, 0, stream>>>(d_buf, nbytes, seed, byte_offset / 8);
    note_launch(nullptr, false);
    return cudaGetLastError();
}

cudaError_t launch_decimal(int alg, uint64_t start, uint64_t count, int width, uint8_t* d_out, cudaStream_t stream) {
    if (count == 0) return cudaSuccess;
    if (count >= (1ull << 40)) return cudaErrorInvalidValue;
    switch (alg) {
    case kSha1: return launch_decimal_sha1(start, count, width, d_out, stream);
    case kMd5: return launch_decimal_md5(start, count, width, d_out, stream);
    case kSm3: return launch_decimal_sm3(start, count, width, d_out, stream);
    default: return cudaErrorInvalidValue;
    }
}

// hb_digest_small: the message rides in the parameter block (k_digest_small).
// One thread's latency is the block chain, so the round variant is the one
// with the shortest dependency chain, not the batch kernels' issue-balanced
// one (tools/digest_probe.py; the A/B build takes $HB_VARIANT).
template <int ALG, int CAP, int V>
static void digest_small_launch(const SmallMsg<CAP>& m, uint8_t* out, cudaStream_t s) {
    launch_plain(k_digest_small<ALG, CAP, V>, 1, 32, s, m, out);
}

template <int ALG, int CAP>
static void digest_small_alg(const SmallMsg<CAP>& m, uint8_t* out, cudaStream_t s) {
#ifdef HB_AB
    switch (tuning().variant) {
    case 0: return digest_small_launch<ALG, CAP, 0>(m, out, s);
    case 1: return digest_small_launch<ALG, CAP, 1>(m, out, s);
    case 2: return digest_small_launch<ALG, CAP, 2>(m, out, s);
    case 3: return digest_small_launch<ALG, CAP, 3>(m, out, s);
    case 5: if constexpr (ALG == kMd5) return digest_small_launch<ALG, CAP, 5>(m, out, s);
    default: break;
    }
#endif
    digest_small_launch<ALG, CAP, kSmallVariant<ALG>>(m, out, s);
}

template <int CAP>
static cudaError_t digest_small_cap(int alg, const uint8_t* msg, uint64_t len, uint8_t* out, uint32_t seq,
                                    cudaStream_t s) {
    SmallMsg<CAP> m;
    if (len) memcpy(m.w, msg, len);
    // Zero the rest of the tail block (md_finish expects bytes >= r clear);
    // words past it are never read.
    memset(reinterpret_cast<uint8_t*>(m.w) + len, 0, (len / 64u + 1u) * 64u - len);
    m.len = len;
    m.seq = seq;
    switch (alg) {
    case kSha1: digest_small_alg<kSha1>(m, out, s); break;
    case kMd5: digest_small_alg<kMd5>(m, out, s); break;
    case kSm3: digest_small_alg<kSm3>(m, out, s); break;
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_digest_small(int alg, const uint8_t* msg, uint64_t len, uint8_t* out, uint32_t seq,
                                cudaStream_t stream) {
    if (len > HB_DIGEST_SMALL_MAX) return cudaErrorInvalidValue;
    if (len <= 256) return digest_small_cap<256>(alg, msg, len, out, seq, stream);
    return digest_small_cap<HB_DIGEST_SMALL_MAX>(alg, msg, len, out, seq, stream);
}

cudaError_t launch_gen_decimal(uint64_t start, uint64_t count, int width, uint8_t* d_out, cudaStream_t stream) {
    if (count == 0) return cudaSuccess;
    k_gen_decimal<<<(unsigned)((count + 127) / 128), 128, 0, stream>>>(start, count, width, d_out);
    note_launch(nullptr, false);
    return cudaGetLastError();
}

}  // namespace hb
