// hb_kernels.cuh -- the hash kernels (templates over the algorithm) and
// their per-algorithm launchers.  Included by one translation unit per
// algorithm (hb_alg_{sha1,md5,sm3}.cu) so the three compile in parallel;
// algorithm-independent kernels (length sort, synthetic bytes) and the
// dispatchers live in hb_kernels.cu.
//  One thread owns one message: chaining state and message
// schedule live in registers; message bytes reach the thread either through a
// TMA-staged, 64B-swizzled shared-memory ring (fixed width, 16B-aligned rows:
// the HBM-streaming hot path) or through direct unaligned loads (any width,
// variable length).  Padding is generated in registers (md_finish) -- the
// padded (n, nblocks, 16) array of the reference (batch.py:128-138) never
// exists in memory.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "hb_algos.cuh"
#include "hb_internal.h"
#include "hb_ptx.cuh"
#include "../../include/hetoc_b200.h"

namespace hb {

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PFN_encodeTiled get_encode_tiled();
char* tma_error_buf();  // thread-local, 160 bytes
constexpr size_t kTmaErrLen = 160;


// Launch with programmatic stream serialization: the kernel may be scheduled
// while the previous kernel in the stream drains; it orders itself with
// griddepcontrol.wait.  tuning().pdl = false ($HB_PDL=0) launches normally.
// Every launch is recorded (note_launch) so the C ABI can name the kernel
// that actually ran (hb_last_kernel_name).
template <class... KArgs, class... Args>
static void launch_pdl_smem(void (*kernel)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t s,
                            bool pdl, Args... args) {
    note_launch(reinterpret_cast<const void*>(kernel), true);
    if (!pdl || !tuning().pdl) {
        kernel<<<grid, block, smem, s>>>(args...);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

template <class... KArgs, class... Args>
static void launch_pdl(void (*kernel)(KArgs...), unsigned grid, unsigned block, cudaStream_t s, Args... args) {
    launch_pdl_smem(kernel, grid, block, 0, s, true, args...);
}

// Plain launch of a hash kernel, recorded like launch_pdl.
template <class... KArgs, class... Args>
static void launch_plain(void (*kernel)(KArgs...), unsigned grid, unsigned block, cudaStream_t s, Args... args) {
    note_launch(reinterpret_cast<const void*>(kernel), true);
    kernel<<<grid, block, 0, s>>>(static_cast<KArgs>(args)...);
}

// SMs of the current device (cached per device).
static int device_sms() {
    static std::atomic<int> cache[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    int v = cache[dev].load(std::memory_order_relaxed);
    if (!v) {
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        cache[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}

// =========================================================================
// Fixed-width, TMA-staged kernel (the hot path).
//
// CTA = 4 warps; warp w owns 32 consecutive messages (rows).  Each warp runs
// its own kStages-deep ring of 2 KiB stages: lane 0 issues one 2-D TMA load
// per 64-byte message block ({64 B, 32 rows} box over the (n, msg_len) byte
// matrix, SWIZZLE_64B), completion lands on the stage's mbarrier, all lanes
// wait on the phase and read their row with four conflict-free 16-byte
// shared loads.  TMA zero-fills columns >= msg_len, so the final partial
// block arrives already masked.
// =========================================================================
constexpr int kTmaWarps = 4;

// Tunable tile configuration: NB messages per thread (ILP), STAGES-deep ring.
// W warps per CTA.  W = 1 is the small-batch shape: a batch of n messages
// becomes n/32 single-warp CTAs spread evenly over all 148 SMs (with 4-warp
// CTAs a 65,536-message batch fills only 512 CTAs, 3-4 per SM, unevenly).
template <int NB, int STAGES, int W = kTmaWarps> struct TmaCfg {
    static constexpr int kRows = 32 * NB;           // rows (messages) per warp
    static constexpr int kStageBytes = 64 * kRows;  // one 64-byte block of every row
    static constexpr int kSmem = W * STAGES * kStageBytes + 1024 /*align slack*/ + W * STAGES * 8;
};
template <int ALG, int NB, int STAGES, int W = kTmaWarps> struct TmaOcc {  // CTAs per SM the budget targets
    static constexpr int kMinCtas =
        W == 1 ? (NB >= 4 ? 6 : NB == 2 ? 12 : 16)
        : NB == 1 ? (STAGES == 2 ? (ALG == kMd5 ? 12 : ALG == kSha1 ? 9 : 8) : (ALG == kSm3 ? 6 : 8))
                  : (STAGES == 2 && ALG != kSm3 ? 6 : 4);
};


// -------------------------------------------------------------------------
// Warp-specialised variant: 4 compute warps + 1 producer warp per CTA.  The
// producer's lane 0 streams one {64 B, 128 rows} TMA tile per message block
// into a STAGES-deep CTA ring (full/empty mbarrier pair per stage); compute
// warps only wait on `full`, read their row (4 x LDS.128) and arrive on
// `empty` -- no TMA-issue path, fence or lane-0 branch in their loop.
// -------------------------------------------------------------------------
constexpr int kWsComputeWarps = 4;
constexpr uint32_t kEarlyLoad = 1u;     // read the messages before griddepcontrol.wait (HB_FLAG_INPUT_READY)
constexpr uint32_t kEarlyTrigger = 2u;  // release the next grid right after griddepcontrol.wait
// kLateWait (with kEarlyLoad, HB_FLAG_INPUT_READY): compute before
// griddepcontrol.wait, wait only before the digest stores.  Under the flag the
// previous grid writes none of this grid's inputs, so the only ordering left
// is on `out` (this grid's stores after everything the previous one did), and
// consecutive batches then compute concurrently -- a batch too small to fill
// the GPU (2^16 messages: 3.5 warps per scheduler) overlaps its successor.
constexpr uint32_t kLateWait = 4u;
// SLACK: reserve 1 KiB to align the ring to 1024 B at run time.  Without it
// (the dynamic window of a kernel with no static shared memory starts 1 KiB
// aligned -- checked in-kernel) a 3-stage CTA needs 24 KiB and 9 CTAs fit an
// SM instead of 8.
template <int NB, int STAGES, bool SLACK = true> struct WsCfg {
    static constexpr int kRows = 32 * kWsComputeWarps * NB;  // rows per CTA tile (TMA box height <= 256)
    static constexpr int kStageBytes = 64 * kRows;            // 8 KiB per message slot
    static constexpr int kSmem = STAGES * kStageBytes + (SLACK ? 1024 : 0) + 2 * STAGES * 8;
};
template <int ALG, int NB, int STAGES, bool SLACK = true> struct WsOcc {
    static constexpr int kMinCtas =
        !SLACK && NB == 1 && STAGES == 3 && ALG != kSm3 ? 9
        : NB == 2 ? (STAGES == 2 ? 6 : 4) : ALG == kSm3 ? 6 : (STAGES == 2 ? (ALG == kMd5 ? 10 : 8) : 8);
};

// UNR: the compute warps' main loop is unrolled by STAGES so every ring
// index is a compile-time constant (no stage/phase bookkeeping, immediate
// shared-memory offsets); the remainder blocks take the generic loop.
template <int ALG, int V, int NB, int STAGES, bool UNR = false, bool SLACK = true>
__global__ void __launch_bounds__((kWsComputeWarps + 1) * 32, (WsOcc<ALG, NB, STAGES, SLACK>::kMinCtas))
k_fixed_tma_ws(const __grid_constant__ CUtensorMap tmap, uint32_t n, uint32_t msg_len, uint8_t* __restrict__ out,
               uint32_t evict_first, uint32_t early) {
    using H = HashAlg<ALG, V>;
    using C = WsCfg<NB, STAGES, SLACK>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t row0 = blockIdx.x * C::kRows;
    const uint32_t base_s = smem_u32(smem_raw);
    if (!SLACK && (base_s & 1023u)) __trap();  // the swizzled ring needs 1 KiB alignment
    uint8_t* ring = smem_raw + (((base_s + 1023u) & ~1023u) - base_s);
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + STAGES * C::kStageBytes);
    uint64_t* empty = full + STAGES;
    const uint32_t nload = (msg_len + 63u) >> 6;

    if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kWsComputeWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();
    // Programmatic dependent launch (launch_pdl_smem): the barrier setup above
    // overlaps the previous grid's tail; global memory is touched only after it
    // completes.  The next grid is triggered once the digests are computed.
    // early & kEarlyLoad (HB_FLAG_INPUT_READY: the caller guarantees the
    // previous grid does not write the messages): the first ring stages are
    // loaded before the wait, so the HBM latency of this grid's first blocks
    // overlaps the previous grid's tail.  Digests are still stored only after
    // the wait.  early & kEarlyTrigger (a grid that leaves room for the next
    // one on every SM): the next grid is released right after the wait, so it
    // is resident -- barriers set up, first stages loading -- while this one runs.
    const uint32_t pro = (early & kEarlyLoad) ? (nload < (uint32_t)STAGES ? nload : (uint32_t)STAGES) : 0u;
    if (pro && warp == kWsComputeWarps && lane == 0) {
        prefetch_tmap(&tmap);
        for (uint32_t b = 0; b < pro; ++b) {
            mbar_arrive_expect_tx(&full[b], C::kStageBytes);
            tma_load_2d(ring + b * C::kStageBytes, &tmap, &full[b], (int)(b * 64u), (int)row0);
        }
    }
    if (!(early & kLateWait)) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (early & kEarlyTrigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (warp == kWsComputeWarps) {  // ---------------- producer warp
        if (lane == 0) {
            if (!pro) prefetch_tmap(&tmap);
            const uint64_t pol = evict_first ? policy_evict_first() : 0;
            uint32_t s = pro % (uint32_t)STAGES, ph = pro == (uint32_t)STAGES ? 1u : 0u;
            for (uint32_t b = pro; b < nload; ++b) {
                if (b >= (uint32_t)STAGES) mbar_wait_parity(&empty[s], ph ^ 1u);
                mbar_arrive_expect_tx(&full[s], C::kStageBytes);
                if (evict_first)
                    tma_load_2d_hint(ring + s * C::kStageBytes, &tmap, &full[s], (int)(b * 64u), (int)row0, pol);
                else
                    tma_load_2d(ring + s * C::kStageBytes, &tmap, &full[s], (int)(b * 64u), (int)row0);
                if (++s == (uint32_t)STAGES) { s = 0; ph ^= 1u; }
            }
        }
        return;
    }

    // ------------------------------------------------- compute warps
    // Thread (warp, lane) owns tile rows warp*32 + lane + 128*q, q < NB.
    uint32_t st[NB][H::kStateWords];
#pragma unroll
    for (int q = 0; q < NB; ++q) H::init(st[q]);
    const uint32_t row = warp * 32u + lane;  // row inside the tile (q = 0)
    const uint32_t swz = (row >> 1) & 3u;    // SWIZZLE_64B (same for row + 128q)
    uint32_t choff[NB][4];
#pragma unroll
    for (int q = 0; q < NB; ++q)
#pragma unroll
        for (uint32_t c = 0; c < 4; ++c) choff[q][c] = smem_u32(ring) + (row + 128u * q) * 64u + ((c ^ swz) << 4);
    uint32_t raw[NB][16];
    auto read_stage = [&](uint32_t s) {
        const uint32_t sbase = s * C::kStageBytes;
#pragma unroll
        for (int q = 0; q < NB; ++q) {
#pragma unroll
            for (uint32_t c = 0; c < 4; ++c) {
                uint32_t x, y, z, w;
                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(x), "=r"(y), "=r"(z), "=r"(w)
                             : "r"(choff[q][c] + sbase)
                             : "memory");
                raw[q][4 * c + 0] = x; raw[q][4 * c + 1] = y; raw[q][4 * c + 2] = z; raw[q][4 * c + 3] = w;
            }
        }
    };
    const uint32_t nfull = msg_len >> 6;
    uint32_t s = 0, ph = 0;
    uint32_t b = 0;
    if (UNR) {
        for (; b + STAGES <= nfull; b += STAGES) {
#pragma unroll
            for (int k = 0; k < STAGES; ++k) {
                mbar_wait_parity(&full[k], ph);
                read_stage(k);
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[k]);
                H::template compress_n<NB>(st, raw);
            }
            ph ^= 1u;
        }
    }
    for (; b < nfull; ++b) {
        mbar_wait_parity(&full[s], ph);
        read_stage(s);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);  // this warp is done with stage s
        H::template compress_n<NB>(st, raw);
        if (++s == (uint32_t)STAGES) { s = 0; ph ^= 1u; }
    }
    const uint32_t r = msg_len & 63u;
    if (r) {
        mbar_wait_parity(&full[s], ph);
        read_stage(s);
    } else {
#pragma unroll
        for (int q = 0; q < NB; ++q)
#pragma unroll
            for (int j = 0; j < 16; ++j) raw[q][j] = 0u;
    }
    md_finish_n<ALG, V, NB>(st, raw, r, msg_len);
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (early & kLateWait) asm volatile("griddepcontrol.wait;" ::: "memory");
#pragma unroll
    for (int q = 0; q < NB; ++q) {
        const uint32_t grow = row0 + row + 128u * q;
        if (grow < n) store_digest<ALG>(out + (uint64_t)grow * H::kDigestBytes, st[q]);
    }
}

// -------------------------------------------------------------------------
// Single-warp CTAs, NB messages per thread (MD5 from 2^16 messages).  Each
// CTA is one warp with its own STAGES-deep ring of {64 B, 32·NB rows} TMA
// tiles; lane 0 refills a stage right after the warp has read it.  Against
// the 4+1-warp tile: two independent round chains per thread (MD5's rounds
// are a 3-op dependency chain, ncu: 35-42 % `wait` stalls), and 32-thread
// CTAs spread a batch evenly over the SMs' sub-partitions (a 2^16-message
// batch is 3.46 warps per scheduler: 4-warp CTAs put 4 on some, 3 on others).
// -9 / -13 / -9 / -5 % at 2^16 x 1 KiB / 2^16 x 4 KiB / 2^18 x 1 KiB /
// 2^20 x 1 KiB with round variants 4 / 6 (profiles/r2/ab_v467_r2o.txt).  Chain-
// bound grids (< 2^16 messages) keep the 4+1-warp tile: halving the thread
// count there lengthens the critical path.  Programmatic dependent launch
// and early loads as in k_fixed_tma_ws.
// -------------------------------------------------------------------------
template <int ALG, int V, int NB, int STAGES>
__global__ void __launch_bounds__(32, (TmaOcc<ALG, NB, STAGES, 1>::kMinCtas))
k_fixed_tma_w1(const __grid_constant__ CUtensorMap tmap, uint32_t n, uint32_t msg_len, uint8_t* __restrict__ out,
               uint32_t early) {
    using H = HashAlg<ALG, V>;
    using C = TmaCfg<NB, STAGES, 1>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t lane = threadIdx.x;
    const uint32_t row0 = blockIdx.x * C::kRows;
    const uint32_t base_s = smem_u32(smem_raw);
    uint8_t* ring = smem_raw + (((base_s + 1023u) & ~1023u) - base_s);  // SWIZZLE_64B needs 1 KiB alignment
    uint64_t* bars = reinterpret_cast<uint64_t*>(ring + STAGES * C::kStageBytes);
    const uint32_t nload = (msg_len + 63u) >> 6;
    const uint32_t pro = nload < (uint32_t)STAGES ? nload : (uint32_t)STAGES;
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
        if (early & kEarlyLoad) {  // HB_FLAG_INPUT_READY: the first stages load before the wait
            prefetch_tmap(&tmap);
            for (uint32_t b = 0; b < pro; ++b) {
                mbar_arrive_expect_tx(&bars[b], C::kStageBytes);
                tma_load_2d(ring + b * C::kStageBytes, &tmap, &bars[b], (int)(b * 64u), (int)row0);
            }
        }
    }
    if (!(early & kLateWait)) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (early & kEarlyTrigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (lane == 0 && !(early & kEarlyLoad)) {
        prefetch_tmap(&tmap);
        for (uint32_t b = 0; b < pro; ++b) {
            mbar_arrive_expect_tx(&bars[b], C::kStageBytes);
            tma_load_2d(ring + b * C::kStageBytes, &tmap, &bars[b], (int)(b * 64u), (int)row0);
        }
    }
    __syncwarp();

    uint32_t st[NB][H::kStateWords];
#pragma unroll
    for (int q = 0; q < NB; ++q) H::init(st[q]);
    const uint32_t swz = (lane >> 1) & 3u;  // SWIZZLE_64B: rows lane and lane + 32q share it
    uint32_t choff[NB][4];
#pragma unroll
    for (int q = 0; q < NB; ++q)
#pragma unroll
        for (uint32_t c = 0; c < 4; ++c) choff[q][c] = smem_u32(ring) + (lane + 32u * q) * 64u + ((c ^ swz) << 4);
    uint32_t raw[NB][16];
    auto read_stage = [&](uint32_t s) {
        const uint32_t sbase = s * C::kStageBytes;
#pragma unroll
        for (int q = 0; q < NB; ++q) {
#pragma unroll
            for (uint32_t c = 0; c < 4; ++c) {
                uint32_t x, y, z, w;
                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(x), "=r"(y), "=r"(z), "=r"(w)
                             : "r"(choff[q][c] + sbase)
                             : "memory");
                raw[q][4 * c + 0] = x; raw[q][4 * c + 1] = y; raw[q][4 * c + 2] = z; raw[q][4 * c + 3] = w;
            }
        }
    };
    const uint32_t nfull = msg_len >> 6;
    uint32_t stage = 0, phase = 0;
    for (uint32_t b = 0; b < nfull; ++b) {
        mbar_wait_parity(&bars[stage], phase);
        read_stage(stage);
        __syncwarp();  // every lane has its registers: the stage may be refilled
        if (lane == 0 && b + STAGES < nload) {
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&bars[stage], C::kStageBytes);
            tma_load_2d(ring + stage * C::kStageBytes, &tmap, &bars[stage], (int)((b + STAGES) * 64u), (int)row0);
        }
        H::template compress_n<NB>(st, raw);
        if (++stage == (uint32_t)STAGES) { stage = 0; phase ^= 1u; }
    }
    const uint32_t r = msg_len & 63u;
    if (r) {  // partial data block: TMA zero-filled the columns >= msg_len
        mbar_wait_parity(&bars[stage], phase);
        read_stage(stage);
    } else {
#pragma unroll
        for (int q = 0; q < NB; ++q)
#pragma unroll
            for (int j = 0; j < 16; ++j) raw[q][j] = 0u;
    }
    md_finish_n<ALG, V, NB>(st, raw, r, msg_len);
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (early & kLateWait) asm volatile("griddepcontrol.wait;" ::: "memory");
#pragma unroll
    for (int q = 0; q < NB; ++q) {
        const uint32_t row = row0 + lane + 32u * q;
        if (row < n) store_digest<ALG>(out + (uint64_t)row * H::kDigestBytes, st[q]);
    }
}

// =========================================================================
// Fixed-width direct-load kernel (HB_FLAG_NO_TMA; 16B-aligned rows only).
// Kept as the A/B baseline for the TMA staging: each thread streams its own
// row with 128-bit read-only loads.
// =========================================================================
template <int ALG>
__global__ void __launch_bounds__(128, (TmaOcc<ALG, 1, 3>::kMinCtas))
k_fixed_direct(const uint8_t* __restrict__ msgs, uint64_t n, uint32_t msg_len, uint8_t* __restrict__ out) {
    using H = HashAlg<ALG>;
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint4* p = reinterpret_cast<const uint4*>(msgs + i * msg_len);
    uint32_t st[H::kStateWords];
    H::init(st);
    const uint32_t nfull = msg_len >> 6;
    for (uint32_t b = 0; b < nfull; ++b) {
        uint32_t raw[16];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const uint4 v = __ldg(p + 4 * b + c);
            raw[4 * c + 0] = v.x; raw[4 * c + 1] = v.y; raw[4 * c + 2] = v.z; raw[4 * c + 3] = v.w;
        }
        compress1<ALG>(st, raw);
    }
    const uint32_t r = msg_len & 63u;
    uint32_t raw[16];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        uint4 v = make_uint4(0, 0, 0, 0);
        if ((uint32_t)(16 * c) < r) v = __ldg(p + 4 * nfull + c);  // r is a multiple of 16 here
        raw[4 * c + 0] = v.x; raw[4 * c + 1] = v.y; raw[4 * c + 2] = v.z; raw[4 * c + 3] = v.w;
    }
    md_finish<ALG>(st, raw, r, msg_len);
    store_digest<ALG>(out + i * H::kDigestBytes, st);
}

// -------------------------------------------------------------------------
// Short fixed-width messages, width known at compile time (L in {16, 32, 48,
// 64, 128}: the powers of two of the configs[4] sweep below 256 B, plus 48).
// One message per thread, L/16 LDG.128 loads; the padding words (0x80, zero
// fill, bit length) are immediates, so the last block costs nothing beyond
// its compression (the generic direct kernel places them with select chains,
// a visible share of a single-block MD5 message).
// -------------------------------------------------------------------------
__host__ __device__ constexpr uint32_t bswap_c(uint32_t x) {
    return (x >> 24) | ((x >> 8) & 0xFF00u) | ((x << 8) & 0xFF0000u) | (x << 24);
}

template <int ALG, int L, int V = -1, int NB = 1>
__global__ void __launch_bounds__(128) k_fixed_small(const uint8_t* __restrict__ msgs, uint64_t n,
                                                     uint8_t* __restrict__ out, uint32_t early = 0) {
    using H = HashAlg<ALG, V>;
    static_assert(L % 16 == 0 && L >= 16 && L <= 128, "width");
    static_assert(NB == 1 || NB == 2, "messages per thread");
    constexpr int kNb = (L + 8) / 64 + 1;  // blocks including padding
    constexpr uint64_t kBits = (uint64_t)L * 8u;
    constexpr uint32_t kL14 = H::kBigEndian ? bswap_c((uint32_t)(kBits >> 32)) : (uint32_t)kBits;
    constexpr uint32_t kL15 = H::kBigEndian ? bswap_c((uint32_t)kBits) : (uint32_t)(kBits >> 32);
    // Programmatic dependent launch (launch_pdl): wait for the previous grid's
    // completion and memory before touching global memory; the trigger for
    // the next grid comes once this thread's hash is done (both no-ops for a
    // normal launch).  A stream of short batches then hides the launch gap.
    // early: as in k_fixed_tma_ws -- kEarlyLoad reads the row before the wait
    // (the caller guarantees the previous grid does not write it; digests are
    // stored after the wait), kEarlyTrigger releases the next grid right after it.
    if (!(early & kEarlyLoad)) asm volatile("griddepcontrol.wait;" ::: "memory");
    // NB = 2: rows 2t and 2t+1 (contiguous bytes) hashed as two independent
    // chains in one compress call; a missing second row re-hashes the first
    // and is not stored.
    const uint64_t i0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * NB;
    if (i0 >= n) {
        if (early & kEarlyLoad) asm volatile("griddepcontrol.wait;" ::: "memory");
        return;
    }
    uint32_t w[NB][L / 4];
#pragma unroll
    for (int q = 0; q < NB; ++q) {
        const uint64_t row = i0 + q < n ? i0 + q : i0;
        const uint4* p = reinterpret_cast<const uint4*>(msgs + row * L);
#pragma unroll
        for (int c = 0; c < L / 16; ++c) {
            const uint4 v = __ldg(p + c);
            w[q][4 * c] = v.x; w[q][4 * c + 1] = v.y; w[q][4 * c + 2] = v.z; w[q][4 * c + 3] = v.w;
        }
    }
    if ((early & kEarlyLoad) && !(early & kLateWait)) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (early & kEarlyTrigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    uint32_t st[NB][H::kStateWords];
#pragma unroll
    for (int q = 0; q < NB; ++q) H::init(st[q]);
#pragma unroll
    for (int b = 0; b < kNb; ++b) {
        uint32_t raw[NB][16];
#pragma unroll
        for (int q = 0; q < NB; ++q) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int pos = 64 * b + 4 * j;  // _pad: data, 0x80, zeros, 64-bit bit length
                raw[q][j] = pos < L ? w[q][pos / 4] : pos == L ? 0x80u : 0u;
            }
            if (b == kNb - 1) { raw[q][14] = kL14; raw[q][15] = kL15; }
        }
        if (NB == 1)
            compress1<ALG, V>(st[0], raw[0]);
        else
            H::template compress_n<NB>(st, raw);
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (early & kLateWait) asm volatile("griddepcontrol.wait;" ::: "memory");
#pragma unroll
    for (int q = 0; q < NB; ++q)
        if (i0 + q < n) store_digest<ALG>(out + (i0 + q) * H::kDigestBytes, st[q]);
}

// =========================================================================
// Generic kernel: any width / alignment, and variable length.
// Message bytes are fetched as aligned 32-bit words and realigned with one
// funnel shift per word; the tail is masked and padded in registers.
// For variable length, `perm` (optional) is a length-descending permutation
// so the 32 lanes of a warp run (nearly) the same number of blocks.
// =========================================================================
__device__ __forceinline__ void load_block_unaligned(const uint8_t* p, const uint8_t* end, uint32_t raw[16]) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    const uint32_t* q = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
    const uint32_t sh = (uint32_t)(a & 3u) * 8u;
    uint32_t c[17];
#pragma unroll
    for (int k = 0; k < 16; ++k) c[k] = __ldg(q + k);
    c[16] = (sh != 0u && reinterpret_cast<const uint8_t*>(q + 16) < end) ? __ldg(q + 16) : 0u;
#pragma unroll
    for (int j = 0; j < 16; ++j) raw[j] = __funnelshift_r(c[j], c[j + 1], sh);
}

__device__ __forceinline__ void load_partial_unaligned(const uint8_t* p, uint32_t r, uint32_t raw[16]) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    const uint32_t* q = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
    const uint32_t sh = (uint32_t)(a & 3u) * 8u;
    const uint8_t* e = p + r;
    uint32_t c[17];
#pragma unroll
    for (int k = 0; k < 17; ++k) c[k] = (reinterpret_cast<const uint8_t*>(q + k) < e) ? __ldg(q + k) : 0u;
#pragma unroll
    for (int j = 0; j < 16; ++j) raw[j] = __funnelshift_r(c[j], c[j + 1], sh);
    mask_tail(raw, r);
}

template <int ALG, bool VARLEN>
__global__ void __launch_bounds__(128)
k_generic(const uint8_t* __restrict__ data, const uint8_t* data_end, const uint64_t* __restrict__ offsets,
          uint64_t offset_base, const uint32_t* __restrict__ perm, uint64_t msg_len, uint64_t n,
          uint8_t* __restrict__ out) {
    using H = HashAlg<ALG>;
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint64_t i = (VARLEN && perm) ? (uint64_t)perm[t] : t;
    uint64_t start, len;
    if (VARLEN) {
        start = offsets[i] - offset_base;
        len = offsets[i + 1] - offsets[i];
    } else {
        start = i * msg_len;
        len = msg_len;
    }
    const uint8_t* p = data + start;
    uint32_t st[H::kStateWords];
    H::init(st);
    const uint64_t nfull = len >> 6;
    for (uint64_t b = 0; b < nfull; ++b) {
        uint32_t raw[16];
        load_block_unaligned(p + 64 * b, data_end, raw);
        compress1<ALG>(st, raw);
    }
    uint32_t raw[16];
    load_partial_unaligned(p + 64 * nfull, (uint32_t)(len & 63u), raw);
    md_finish<ALG>(st, raw, (uint32_t)(len & 63u), len);
    store_digest<ALG>(out + i * H::kDigestBytes, st);
}

// -------------------------------------------------------------------------
// Variable-length kernel: per message, 128-bit read-only loads of the 16-byte
// aligned window around each block (4-5 LDG.128 instead of 17 LDG.32), then a
// realignment by the message's byte offset a%16: a word select by q=(a>>2)&3
// (a switch that is warp-uniform because the length sort also groups messages
// by q) and one funnel shift per word by (a%4)*8.
// -------------------------------------------------------------------------
__device__ __forceinline__ void realign16(const uint32_t (&c)[20], uint32_t q, uint32_t sh, uint32_t (&raw)[16]) {
#define HB_RA(Q)                                                                    \
    _Pragma("unroll") for (int j = 0; j < 16; ++j) raw[j] = __funnelshift_r(c[j + Q], c[j + Q + 1], sh);
    switch (q) {
    case 0: HB_RA(0) break;
    case 1: HB_RA(1) break;
    case 2: HB_RA(2) break;
    default: HB_RA(3) break;
    }
#undef HB_RA
}

// PF: software pipelining -- block b+1's loads are issued right after block b
// is realigned out of c[], so they are in flight during b's compression
// (+20 registers; pays off once the windowed sort makes a warp's loads L2-
// friendly, see profiles/ab_varlen_r1d.txt).
// 16-byte chunk at p, never reading at or past `dend` (bytes there are zero):
// used only for the granule that straddles the end of the data buffer.
static __device__ __noinline__ uint4 ld16_bounded(const uint4* p, uintptr_t dend) {
    const uint8_t* b = reinterpret_cast<const uint8_t*>(p);
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        uint32_t x = 0;
        for (int j = 0; j < 4; ++j) {
            const uintptr_t q = reinterpret_cast<uintptr_t>(b + 4 * k + j);
            if (q < dend) x |= (uint32_t)__ldg(b + 4 * k + j) << (8 * j);
        }
        w[k] = x;
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

// Chunk k of a 16-byte window, bounded by the data end when `edge` (the
// message's last granule straddles it -- only ever the batch's final bytes).
__device__ __forceinline__ uint4 ld16_edge(const uint4* p, bool edge, uintptr_t dend) {
    return (edge && reinterpret_cast<uintptr_t>(p + 1) > dend) ? ld16_bounded(p, dend) : __ldg(p);
}

// LD: 0 = plain read-only loads; 1 = with an L2 256-byte prefetch hint (a
// miss fills the next three blocks of the message into L2); 2 = the same and
// no L1 allocation.
template <int LD>
__device__ __forceinline__ uint4 ld16(const uint4* p) {
    if constexpr (LD == 0) {
        return __ldg(p);
    } else {
        uint4 v;
        if constexpr (LD == 1)
            asm volatile("ld.global.nc.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
        else
            asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
        return v;
    }
}

template <int LD = 0>
__device__ __forceinline__ void load_full_window(const uint4* src, bool misaligned, uint32_t (&c)[20],
                                                 bool edge = false, uintptr_t dend = 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {  // chunks 0-3 end inside the block: never past the message
        const uint4 v = ld16<LD>(src + k);
        c[4 * k] = v.x; c[4 * k + 1] = v.y; c[4 * k + 2] = v.z; c[4 * k + 3] = v.w;
    }
    uint4 v4 = make_uint4(0, 0, 0, 0);
    if (misaligned) v4 = (edge && reinterpret_cast<uintptr_t>(src + 5) > dend) ? ld16_bounded(src + 4, dend)
                                                                                 : ld16<LD>(src + 4);
    c[16] = v4.x; c[17] = v4.y; c[18] = v4.z; c[19] = v4.w;
}

// One message of k_varlen16; EDGE: the message's last 16-byte granule
// straddles the end of the data buffer (only the batch's final bytes), so the
// granules that can cross it are loaded bounded.  The common path carries no
// bounds checks at all.
// PF >= 2: prefetch instructions instead of register pipelining (no
// registers held across the compression): 2 = the window of block b+2 into L2
// while block b is compressed, 3 = block b+1's window into L1, 4 = both.
__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
__device__ __forceinline__ void prefetch_l1(const void* p) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
template <int PF>
__device__ __forceinline__ void varlen_prefetch(const uint4* w16, uint64_t b, uint64_t nfull) {
    if constexpr (PF == 2 || PF == 4) {
        if (b + 2 <= nfull) {
            const uint8_t* p = reinterpret_cast<const uint8_t*>(w16 + 4 * (b + 2));
            prefetch_l2(p);
            prefetch_l2(p + 79);
        }
    }
    if constexpr (PF == 3 || PF == 4) {
        if (b + 1 <= nfull) {
            const uint8_t* p = reinterpret_cast<const uint8_t*>(w16 + 4 * (b + 1));
            prefetch_l1(p);
            prefetch_l1(p + 79);
        }
    }
}

template <int ALG, int PF, bool EDGE, int LD = 0>
__device__ __forceinline__ void varlen16_message(const uint4* w16, uintptr_t a, uint64_t len, uintptr_t dend,
                                                 uint8_t* dout) {
    using H = HashAlg<ALG>;
    const uint32_t q = (uint32_t)(a >> 2) & 3u, sh = (uint32_t)(a & 3u) * 8u;
    const bool misaligned = (a & 15u) != 0;
    uint32_t st[H::kStateWords];
    H::init(st);
    uint32_t c[20];
    uint32_t raw[16];
    const uint64_t nfull = len >> 6;
    if (PF == 1) {
        if (nfull) load_full_window<LD>(w16, misaligned, c, EDGE, dend);
        for (uint64_t b = 0; b < nfull; ++b) {
            realign16(c, q, sh, raw);
            if (b + 1 < nfull) load_full_window<LD>(w16 + 4 * (b + 1), misaligned, c, EDGE, dend);
            compress1<ALG>(st, raw);
        }
    } else if (PF == 5) {
        // Carry: a misaligned window's fifth chunk is the next block's first,
        // so it is kept in registers -- 4 loads per block instead of 5.
        uint4 carry = make_uint4(0, 0, 0, 0);
        for (uint64_t b = 0; b < nfull; ++b) {
            const uint4* src = w16 + 4 * b;
            const uint4 v0 = (b != 0 && misaligned) ? carry : ld16<LD>(src);
            c[0] = v0.x; c[1] = v0.y; c[2] = v0.z; c[3] = v0.w;
#pragma unroll
            for (int k = 1; k < 4; ++k) {
                const uint4 v = ld16<LD>(src + k);
                c[4 * k] = v.x; c[4 * k + 1] = v.y; c[4 * k + 2] = v.z; c[4 * k + 3] = v.w;
            }
            uint4 v4 = make_uint4(0, 0, 0, 0);
            if (misaligned) v4 = (EDGE && reinterpret_cast<uintptr_t>(src + 5) > dend) ? ld16_bounded(src + 4, dend)
                                                                                       : ld16<LD>(src + 4);
            c[16] = v4.x; c[17] = v4.y; c[18] = v4.z; c[19] = v4.w;
            carry = v4;
            realign16(c, q, sh, raw);
            compress1<ALG>(st, raw);
        }
    } else {
        if (PF == 2 || PF == 4) varlen_prefetch<2>(w16, (uint64_t)-1, nfull);  // block 1 (b = -1: b + 2 = 1)
        for (uint64_t b = 0; b < nfull; ++b) {
            load_full_window<LD>(w16 + 4 * b, misaligned, c, EDGE, dend);
            varlen_prefetch<PF>(w16, b, nfull);
            realign16(c, q, sh, raw);
            compress1<ALG>(st, raw);
        }
    }
    // tail: the r = len % 64 remaining bytes (chunks that overlap [p, p+r) only)
    const uint32_t r = (uint32_t)(len & 63u);
    const uintptr_t tail_end = a + len;
    const uint4* src = w16 + 4 * nfull;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        uint4 v = make_uint4(0, 0, 0, 0);
        if (reinterpret_cast<uintptr_t>(src + k) < tail_end) v = ld16_edge(src + k, EDGE, dend);
        c[4 * k] = v.x; c[4 * k + 1] = v.y; c[4 * k + 2] = v.z; c[4 * k + 3] = v.w;
    }
    realign16(c, q, sh, raw);
    mask_tail(raw, r);
    md_finish<ALG>(st, raw, r, len);
    store_digest<ALG>(dout, st);
}

template <int ALG, int PF = 0, int LD = 0, int MINB = 1>
__global__ void __launch_bounds__(128, MINB)
k_varlen16(const uint8_t* __restrict__ data, const uint8_t* data_end, const uint64_t* __restrict__ offsets,
           uint64_t offset_base, const uint32_t* __restrict__ perm, uint64_t n, uint8_t* __restrict__ out) {
    using H = HashAlg<ALG>;
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint64_t i = perm ? (uint64_t)perm[t] : t;
    const uint64_t start = offsets[i] - offset_base;
    const uint64_t len = offsets[i + 1] - offsets[i];
    // perm[t] read (see k_varlen16l): a length sort launched after this kernel
    // with HB_FLAG_INPUT_READY may now overwrite the permutation
    if (len != ~0ull) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uintptr_t a = reinterpret_cast<uintptr_t>(data + start);
    const uint4* w16 = reinterpret_cast<const uint4*>(a & ~uintptr_t(15));
    const uintptr_t dend = reinterpret_cast<uintptr_t>(data_end);
    if (((a + len + 15u) & ~uintptr_t(15)) > dend)
        varlen16_message<ALG, PF, true, LD>(w16, a, len, dend, out + i * H::kDigestBytes);
    else
        varlen16_message<ALG, PF, false, LD>(w16, a, len, dend, out + i * H::kDigestBytes);
}

// -------------------------------------------------------------------------
// Variable-length kernel with a lean block loop.  MD5's varlen kernel is
// issue-bound (ncu: issue 75 %, ALU 77 %, LSU 81 %), and around the ~315
// instructions of a compression k_varlen16 spends ~45 per block: the
// realignment switch (7 branch instructions), a bounds branch for the fifth
// granule, 64-bit block counters.  Here the fifth granule is one predicated
// load (a 16-byte-aligned window does not use it, and for an aligned message
// it may lie past the data end), the block counters are 32-bit, and with QT
// the word offset q = (a >> 2) & 3 is a template parameter of the whole
// block loop -- entered once per message, warp-uniform after the q-major
// sort -- so the loop body has no realignment branches at all (four copies
// of the loop).  Block b+1's window is in flight during b's compression.
// -------------------------------------------------------------------------
__device__ __forceinline__ uint4 ld16_pred(const uint4* p, uint32_t pred) {
    uint4 v = make_uint4(0, 0, 0, 0);
    asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %5, 0;\n\t@p ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];\n\t}"
        : "+r"(v.x), "+r"(v.y), "+r"(v.z), "+r"(v.w)
        : "l"(p), "r"(pred));
    return v;
}

// ... with an L2 cache policy (createpolicy) on every granule.
__device__ __forceinline__ uint4 ld16_pred_hint(const uint4* p, uint32_t pred, uint64_t pol) {
    uint4 v = make_uint4(0, 0, 0, 0);
    asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %5, 0;\n\t"
        "@p ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %6;\n\t}"
        : "+r"(v.x), "+r"(v.y), "+r"(v.z), "+r"(v.w)
        : "l"(p), "r"(pred), "l"(pol));
    return v;
}

__device__ __forceinline__ void load_window5_hint(const uint4* src, uint32_t mis, uint32_t (&c)[20], uint64_t pol) {
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const uint4 v = ld16_pred_hint(src + k, k < 4 ? 1u : mis, pol);
        c[4 * k] = v.x; c[4 * k + 1] = v.y; c[4 * k + 2] = v.z; c[4 * k + 3] = v.w;
    }
}

__device__ __forceinline__ void load_window5(const uint4* src, uint32_t mis, uint32_t (&c)[20]) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint4 v = __ldg(src + k);
        c[4 * k] = v.x; c[4 * k + 1] = v.y; c[4 * k + 2] = v.z; c[4 * k + 3] = v.w;
    }
    const uint4 v4 = ld16_pred(src + 4, mis);
    c[16] = v4.x; c[17] = v4.y; c[18] = v4.z; c[19] = v4.w;
}

template <int Q>
__device__ __forceinline__ void realign_q(const uint32_t (&c)[20], uint32_t sh, uint32_t (&raw)[16]) {
#pragma unroll
    for (int j = 0; j < 16; ++j) raw[j] = __funnelshift_r(c[j + Q], c[j + Q + 1], sh);
}

// Full blocks 0 .. nfull-1 of one message (not at the data end).  Q < 0: the
// realignment class is read at run time (one loop for every class).
// HINT: the first window (whose leading granule holds the previous message's
// last bytes, read by that message's thread much later) is loaded evict_last,
// so the shared granule is still in L2 then instead of coming from HBM twice.
template <int ALG, int Q, int V, bool HINT = false>
__device__ __forceinline__ void varlen16l_blocks(const uint4* w16, uint32_t mis, uint32_t q, uint32_t sh,
                                                 uint32_t nfull, uint32_t* st) {
    uint32_t c[20], raw[16];
    if (HINT) {
        if (nfull) load_window5_hint(w16, mis, c, policy_evict_last());
    } else {
        if (nfull) load_window5(w16, mis, c);
    }
    for (uint32_t b = 0; b < nfull; ++b) {
        if constexpr (Q < 0) realign16(c, q, sh, raw);
        else realign_q<Q>(c, sh, raw);
        if (b + 1 < nfull) load_window5(w16 + 4 * (b + 1), mis, c);
        compress1<ALG, V>(st, raw);
    }
}

template <int ALG, bool QT, int V = -1, bool HINT = false>
__global__ void __launch_bounds__(128)
k_varlen16l(const uint8_t* __restrict__ data, const uint8_t* data_end, const uint64_t* __restrict__ offsets,
            uint64_t offset_base, const uint32_t* __restrict__ perm, uint64_t n, uint8_t* __restrict__ out) {
    using H = HashAlg<ALG>;
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint64_t i = perm ? (uint64_t)perm[t] : t;
    const uint64_t start = offsets[i] - offset_base;
    const uint64_t len = offsets[i + 1] - offsets[i];
    // perm[t] has been read (the offsets loads depend on it, and the trigger
    // is predicated on their value): a length sort launched after this kernel
    // with HB_FLAG_INPUT_READY may now overwrite the permutation while this
    // grid drains.
    if (len != ~0ull) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uintptr_t a = reinterpret_cast<uintptr_t>(data + start);
    const uint4* w16 = reinterpret_cast<const uint4*>(a & ~uintptr_t(15));
    const uintptr_t dend = reinterpret_cast<uintptr_t>(data_end);
    uint8_t* dout = out + i * H::kDigestBytes;
    if (((a + len + 15u) & ~uintptr_t(15)) > dend || (len >> 38)) {  // the batch's last bytes, or > 2^32 blocks
        varlen16_message<ALG, 1, true>(w16, a, len, dend, dout);
        return;
    }
    const uint32_t q = (uint32_t)(a >> 2) & 3u, sh = (uint32_t)(a & 3u) * 8u;
    const uint32_t mis = (a & 15u) != 0;
    const uint32_t nfull = (uint32_t)(len >> 6);
    uint32_t st[H::kStateWords];
    H::init(st);
    if constexpr (QT) {
        switch (q) {
        case 0: varlen16l_blocks<ALG, 0, V, HINT>(w16, mis, q, sh, nfull, st); break;
        case 1: varlen16l_blocks<ALG, 1, V, HINT>(w16, mis, q, sh, nfull, st); break;
        case 2: varlen16l_blocks<ALG, 2, V, HINT>(w16, mis, q, sh, nfull, st); break;
        default: varlen16l_blocks<ALG, 3, V, HINT>(w16, mis, q, sh, nfull, st); break;
        }
    } else {
        varlen16l_blocks<ALG, -1, V, HINT>(w16, mis, q, sh, nfull, st);
    }
    // tail: the r = len % 64 remaining bytes (granules that overlap [.., a + len) only)
    const uint32_t r = (uint32_t)(len & 63u);
    const uintptr_t tail_end = a + len;
    const uint4* src = w16 + 4 * (uint64_t)nfull;
    uint32_t c[20], raw[16];
    const uint64_t pol_tail = HINT ? policy_evict_first() : 0;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const uint32_t live = reinterpret_cast<uintptr_t>(src + k) < tail_end;
        const uint4 v = HINT ? ld16_pred_hint(src + k, live, pol_tail) : ld16_pred(src + k, live);
        c[4 * k] = v.x; c[4 * k + 1] = v.y; c[4 * k + 2] = v.z; c[4 * k + 3] = v.w;
    }
    realign16(c, q, sh, raw);
    mask_tail(raw, r);
    md_finish<ALG, V>(st, raw, r, len);
    store_digest<ALG>(dout, st);
}

// -------------------------------------------------------------------------
// Lean block loop with a uniform finish (SM3 default).  A message of block
// count nb (data + 0x80 + length) needs nb compressions, but k_varlen16(l)
// runs its full-block loop to len/64 and then md_finish's one or two: a lane
// whose last r = len % 64 bytes are >= 56 has one full block fewer and one
// tail block more, so a warp holding both kinds (nearly every warp: P(r >= 56)
// = 1/8 per lane) executes nb + 1 compressions.  Here every lane runs nb - 1
// loop iterations -- the r >= 56 lanes' partial block, with its 0x80 patched
// into words 14-15, is the last one -- and then one final block: the remaining
// data, 0x80 (r < 56) and the bit length.  Every window, the one after the
// last full block included, is loaded whole (its bytes past the message are
// masked off; they belong to the next message), so the hot loop carries no
// tail-specific loads; a message whose final window can reach past the data
// end takes the bounded path.  HINT: L2 policies as in
// k_varlen16l -- the first window evict_last (its leading granule holds the
// previous message's last bytes, read by that message's thread much later),
// the final window evict_first (it releases that granule).
template <int ALG, bool HINT = false>
__global__ void __launch_bounds__(128)
k_varlen16g(const uint8_t* __restrict__ data, const uint8_t* data_end, const uint64_t* __restrict__ offsets,
            uint64_t offset_base, const uint32_t* __restrict__ perm, uint64_t n, uint8_t* __restrict__ out) {
    using H = HashAlg<ALG>;
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint64_t i = perm ? (uint64_t)perm[t] : t;
    const uint64_t start = offsets[i] - offset_base;
    const uint64_t len = offsets[i + 1] - offsets[i];
    // perm[t] read (see k_varlen16l): a length sort launched after this kernel
    // with HB_FLAG_INPUT_READY may now overwrite the permutation
    if (len != ~0ull) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uintptr_t a = reinterpret_cast<uintptr_t>(data + start);
    const uint4* w16 = reinterpret_cast<const uint4*>(a & ~uintptr_t(15));
    const uintptr_t dend = reinterpret_cast<uintptr_t>(data_end);
    uint8_t* dout = out + i * H::kDigestBytes;
    // the final window ends before (a & ~15) + 64 * (len / 64 + 1) + 80
    if ((a & ~uintptr_t(15)) + (len & ~uint64_t(63)) + 144u > dend || (len >> 38)) {
        varlen16_message<ALG, 1, true>(w16, a, len, dend, dout);
        return;
    }
    const uint32_t q = (uint32_t)(a >> 2) & 3u, sh = (uint32_t)(a & 3u) * 8u;
    const uint32_t mis = (a & 15u) != 0;
    const uint32_t nfull = (uint32_t)(len >> 6), r = (uint32_t)(len & 63u);
    const uint32_t nmain = nfull + (r >= 56u ? 1u : 0u);  // every block but the final one
    const uint32_t pad = 0x80u << ((r & 3u) * 8u), pw = r >> 2;
    uint32_t st[H::kStateWords];
    H::init(st);
    uint32_t c[20], raw[16];
    uint64_t pol_norm = 0, pol_last = 0;
    if (HINT) {
        pol_norm = policy_evict_normal();
        pol_last = policy_evict_first();
        load_window5_hint(w16, mis, c, nmain ? policy_evict_last() : pol_last);
    } else {
        load_window5(w16, mis, c);
    }
    for (uint32_t b = 0; b < nmain; ++b) {
        realign16(c, q, sh, raw);
        if (HINT) load_window5_hint(w16 + 4 * (b + 1), mis, c, b + 1 == nmain ? pol_last : pol_norm);
        else load_window5(w16 + 4 * (b + 1), mis, c);
        if (b == nfull) {
            // r >= 56: the partial data block carries the 0x80.  Only words 14-15
            // change (bytes 56 .. r-1 are data, byte r is 0x80, the rest zero): a
            // few predicated instructions, no full mask_tail in the hot loop.
            const uint32_t k = r - 56u;
            const uint64_t w = ((uint64_t)raw[15] << 32) | raw[14];
            const uint64_t m = k ? (~0ull >> (64u - 8u * k)) : 0ull;
            const uint64_t v = (w & m) | (0x80ull << (8u * k));
            raw[14] = (uint32_t)v;
            raw[15] = (uint32_t)(v >> 32);
        }
        compress1<ALG>(st, raw);
    }
    realign16(c, q, sh, raw);
    mask_tail(raw, r < 56u ? r : 0u);
    if (r < 56u) {
#pragma unroll
        for (int j = 0; j < 16; ++j) raw[j] |= (pw == (uint32_t)j) ? pad : 0u;
    }
    const uint64_t bits = len * 8ull;
    raw[14] = H::kBigEndian ? bswap((uint32_t)(bits >> 32)) : (uint32_t)bits;
    raw[15] = H::kBigEndian ? bswap((uint32_t)bits) : (uint32_t)(bits >> 32);
    compress1<ALG>(st, raw);
    store_digest<ALG>(dout, st);
}

// ---------------------------------------------------- length-bucket sort --
// Counting sort of message indices by block count, longest first.  Three
// small kernels: per-CTA shared-memory histograms -> global histogram, one
// exclusive scan, per-CTA reservation + scatter.  Order inside a bucket is
// irrelevant (digests are written to out[i]).
// 1024 block-count classes (longest first; >= 1023 blocks share the first)
// x 4 word-alignment classes q = (address >> 2) & 3, so a warp's messages
// have similar lengths AND the same realignment path in k_varlen16.
constexpr int kSortNbClasses = 1024;
constexpr int kSortBuckets = kSortNbClasses * 4;
constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;  // per thread

// Sort key: block-count class (longest first) x Q word-alignment classes
// q = (address >> 2) mod Q -- Q = 4 for the 16-byte-window kernels, 8 for the
// 32-byte-window one -- so a warp's messages take the same realignment path.
// QMAJOR: alignment class first, then block count -- a window of 8,192
// messages has ~31 per (block count, q) bucket, so with the block count as
// the major key nearly every warp straddles two q classes (the realignment
// switch then runs two paths); q-major warps are q-uniform and straddle at
// most two adjacent block counts instead.
template <int Q, bool QMAJOR = false>
__device__ __forceinline__ uint32_t sort_bucket_q(const uint64_t* offsets, uint64_t i, uint64_t addr_bias) {
    const uint64_t len = offsets[i + 1] - offsets[i];
    const uint64_t nb = (len + 8u) / 64u + 1u;
    const uint64_t c = nb < (uint64_t)(kSortNbClasses - 1) ? nb : (uint64_t)(kSortNbClasses - 1);
    const uint32_t q = (uint32_t)((offsets[i] + addr_bias) >> 2) & (uint32_t)(Q - 1);
    if (QMAJOR) return q * (uint32_t)kSortNbClasses + ((uint32_t)(kSortNbClasses - 1) - (uint32_t)c);
    return ((uint32_t)(kSortNbClasses - 1) - (uint32_t)c) * (uint32_t)Q + q;
}
__device__ __forceinline__ uint32_t sort_bucket(const uint64_t* offsets, uint64_t i, uint64_t addr_bias) {
    return sort_bucket_q<4>(offsets, i, addr_bias);
}

// -------------------------------------------- decimal messages in-register --
// gen_messages (batch.py:86-99): message i is the zero-padded decimal
// rendering of start+i, WIDTH bytes.  The bytes are built in registers and
// hashed directly; only digests touch HBM.
// FMA_DIGITS: below 2^30 the digits are produced entirely on the FMA pipe --
// q = umulhi(v, 0x1999999A) is exactly v / 10 for v < 2^30 (the reciprocal's
// excess 0.4 * v / 2^32 stays under 0.1), d = v - 10 q, and each digit is
// placed with a multiply by an opaque 2^(8k) -- leaving the ALU pipe (the
// bottleneck: booleans, rotates) to the compression.
template <int ALG, int WIDTH, int V = -1, bool FMA_DIGITS = false>
__global__ void __launch_bounds__(128) k_decimal(uint64_t start, uint64_t count, uint8_t* __restrict__ out) {
    using H = HashAlg<ALG, V>;
    static_assert(WIDTH >= 1 && WIDTH <= 20, "width");
    // One message per thread, one-shot CTAs: a grid-stride loop measured 4-8 %
    // slower (profiles/ab_decimal_r1.txt).
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    uint64_t v = start + i;
    uint32_t raw[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) raw[j] = 0u;
    if (FMA_DIGITS && WIDTH <= 9 && start + count <= (1ull << 30)) {  // grid-uniform
        uint32_t v32 = (uint32_t)v;
#pragma unroll
        for (int pos = WIDTH - 1; pos >= 0; --pos) {  // batch.py:96-98
            const uint32_t q = __umulhi(v32, 0x1999999Au);
            const uint32_t d = v32 - q * 10u;
            raw[pos >> 2] = d * c_opaque[8 * (pos & 3)] + raw[pos >> 2];  // IMAD: d << 8(pos%4)
            v32 = q;
        }
        // the '0' (0x30) of every digit byte, as one add per word (compile-time constants)
#pragma unroll
        for (int w = 0; w < (WIDTH + 3) / 4; ++w) {
            uint32_t ascii = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (4 * w + k < WIDTH) ascii |= 0x30u << (8 * k);
            raw[w] += ascii;
        }
    } else if (start + count <= 0xFFFFFFFFull) {  // grid-uniform: 32-bit digit extraction (IMAD.HI, not 64-bit division)
        uint32_t v32 = (uint32_t)v;
#pragma unroll
        for (int pos = WIDTH - 1; pos >= 0; --pos) {  // batch.py:96-98
            const uint32_t q = v32 / 10u;
            raw[pos >> 2] |= (0x30u + (v32 - q * 10u)) << ((pos & 3) * 8);
            v32 = q;
        }
    } else {
#pragma unroll
        for (int pos = WIDTH - 1; pos >= 0; --pos) {  // batch.py:96-98
            const uint32_t d = (uint32_t)(v % 10u);
            v /= 10u;
            raw[pos >> 2] |= (0x30u + d) << ((pos & 3) * 8);
        }
    }
    uint32_t st[H::kStateWords];
    H::init(st);
    md_finish<ALG, V>(st, raw, (uint32_t)WIDTH, (uint64_t)WIDTH);
    store_digest<ALG>(out + i * H::kDigestBytes, st);
}

// Runs of ten: thread t renders u = start/10 + t once into the first WIDTH-1
// digit bytes and hashes v = 10u + j, j = 0..9 (the messages that fall inside
// [start, start+count)), changing only the last digit byte between messages.
// The digit extraction -- 27 FMA-pipe ops per 9-digit message in k_decimal --
// is amortised ten ways, so the compression's pipe balance is what remains.
// Same bytes as gen_messages (batch.py:96-98): the low WIDTH digits of v are
// the low WIDTH-1 digits of u followed by v mod 10 = j.  Needs u < 2^30
// (umulhi reciprocal exact) -- v below ~1.07e10.
template <int ALG, int WIDTH, int V = -1, bool PAIR = false>
__global__ void __launch_bounds__(128) k_decimal_run(uint64_t start, uint64_t count, uint8_t* __restrict__ out) {
    using H = HashAlg<ALG, V>;
    static_assert(WIDTH >= 2 && WIDTH <= 10, "width");
    const uint64_t u = start / 10u + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t end = start + count;
    if (u * 10u >= end) return;
    uint32_t pre[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) pre[j] = 0u;
    uint32_t u32 = (uint32_t)u;
#pragma unroll
    for (int pos = WIDTH - 2; pos >= 0; --pos) {
        const uint32_t q = __umulhi(u32, 0x1999999Au);
        const uint32_t d = u32 - q * 10u;
        pre[pos >> 2] = d * c_opaque[8 * (pos & 3)] + pre[pos >> 2];
        u32 = q;
    }
#pragma unroll
    for (int w = 0; w < (WIDTH + 3) / 4; ++w) {  // '0' of every digit byte, the last one included
        uint32_t ascii = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (4 * w + k < WIDTH) ascii |= 0x30u << (8 * k);
        pre[w] += ascii;
    }
    constexpr int kLastW = (WIDTH - 1) >> 2, kLastSh = 8 * ((WIDTH - 1) & 3);
    auto one = [&](uint32_t j, uint8_t* dst) {
        uint32_t raw[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) raw[k] = pre[k];
        raw[kLastW] = pre[kLastW] + (j << kLastSh);
        uint32_t st[H::kStateWords];
        H::init(st);
        md_finish<ALG, V>(st, raw, (uint32_t)WIDTH, (uint64_t)WIDTH);
        store_digest<ALG>(dst, st);
    };
    if (PAIR && u * 10u >= start && u * 10u + 10u <= end) {
        // messages j and j+5 compressed together (two independent chains per
        // thread for the scheduler to interleave; MD5 default, $HB_DEC_PAIR)
        uint8_t* dst = out + (u * 10u - start) * H::kDigestBytes;
        constexpr uint32_t kPad = 0x80u << ((WIDTH & 3) * 8);
        constexpr uint64_t kBits = (uint64_t)WIDTH * 8u;
        constexpr uint32_t kL14 = H::kBigEndian ? 0u : (uint32_t)kBits;
        constexpr uint32_t kL15 = H::kBigEndian ? bswap_c((uint32_t)kBits) : 0u;
#pragma unroll 1
        for (uint32_t j = 0; j < 5u; ++j) {
            uint32_t raw[2][16], st[2][H::kStateWords];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
#pragma unroll
                for (int k = 0; k < 16; ++k) raw[q][k] = pre[k];
                raw[q][kLastW] = pre[kLastW] + ((j + 5u * q) << kLastSh);
                raw[q][WIDTH >> 2] |= kPad;
                raw[q][14] = kL14;
                raw[q][15] = kL15;
                H::init(st[q]);
            }
            H::template compress_n<2>(st, raw);
            store_digest<ALG>(dst + j * H::kDigestBytes, st[0]);
            store_digest<ALG>(dst + (j + 5u) * H::kDigestBytes, st[1]);
        }
    } else if (u * 10u >= start && u * 10u + 10u <= end) {  // all but the first / last thread: no range checks
        uint8_t* dst = out + (u * 10u - start) * H::kDigestBytes;
#pragma unroll 1
        for (uint32_t j = 0; j < 10u; ++j) one(j, dst + j * H::kDigestBytes);
    } else {
#pragma unroll 1
        for (uint32_t j = 0; j < 10u; ++j) {
            const uint64_t v = u * 10u + j;
            if (v >= start && v < end) one(j, out + (v - start) * H::kDigestBytes);
        }
    }
}

// =========================================================================
// Host-side launchers.  Every knob comes from tuning() (parsed once from the
// environment when the library loads, hb_tuning_reload() re-reads it), so a
// launch costs no getenv/strcmp.  The default build instantiates only the
// tuned kernel shapes; the A/B arms measured in profiles/ (per-warp TMA rings,
// other tile configurations and round variants, the 32-byte / bulk-copy /
// cooperative varlen kernels) exist only in a -DHB_AB build (hb_ab_kernels.cuh).
// =========================================================================

// Run `set` (a cudaFuncSetAttribute call) once per device: kernel attributes
// such as the dynamic shared-memory limit are per device, so a process driving
// several GPUs must set them on each (a process-wide call_once would not).
template <class F>
static cudaError_t set_smem_attr_once(std::atomic<uint64_t>& done, F set) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    e = set();
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}

// The (n, L) byte matrix as a 2-D TMA tensor: dim0 = bytes of a row
// (contiguous), dim1 = rows with stride L.  Box = one 64-byte block of `rows`
// rows, 64-byte swizzle, L2 promotion `l2` bytes.
static cudaError_t encode_rows_map_uncached(CUtensorMap* map, const uint8_t* d_msgs, uint32_t n, uint32_t L,
                                            uint32_t rows, uint32_t l2);
static cudaError_t encode_rows_map(CUtensorMap* map, const uint8_t* d_msgs, uint32_t n, uint32_t L, uint32_t rows,
                                   uint32_t l2) {
    // The last few descriptors of this thread, reused when a caller hashes the
    // same buffer shape again (rotating input copies, graph capture, the
    // reference executor's repeated chunks): the encode is ~1 us of host time
    // on a launch that can be shorter than that.
    struct Entry { const uint8_t* p; uint32_t n, L, rows, l2; CUtensorMap map; };
    constexpr int kCache = 8;
    thread_local Entry cache[kCache] = {};
    thread_local int next = 0;
    for (int k = 0; k < kCache; ++k) {
        const Entry& c = cache[k];
        if (c.p == d_msgs && c.n == n && c.L == L && c.rows == rows && c.l2 == l2 && c.p) {
            *map = c.map;
            return cudaSuccess;
        }
    }
    const cudaError_t e = encode_rows_map_uncached(map, d_msgs, n, L, rows, l2);
    if (e == cudaSuccess) {
        cache[next] = Entry{d_msgs, n, L, rows, l2, *map};
        next = (next + 1) % kCache;
    }
    return e;
}

static cudaError_t encode_rows_map_uncached(CUtensorMap* map, const uint8_t* d_msgs, uint32_t n, uint32_t L,
                                            uint32_t rows, uint32_t l2) {
    PFN_encodeTiled enc = get_encode_tiled();
    if (!enc) {
        snprintf(tma_error_buf(), kTmaErrLen, "cuTensorMapEncodeTiled unavailable");
        return cudaErrorNotSupported;
    }
    const cuuint64_t dims[2] = {L, n};
    const cuuint64_t strides[1] = {L};
    const cuuint32_t box[2] = {64, rows};
    const cuuint32_t estr[2] = {1, 1};
    const CUtensorMapL2promotion prom = l2 == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                        : l2 == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                        : l2 == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                    : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    const CUresult rc = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(d_msgs), dims, strides, box,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, prom,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rc != CUDA_SUCCESS) {
        snprintf(tma_error_buf(), kTmaErrLen, "cuTensorMapEncodeTiled failed (CUresult %d)", (int)rc);
        return cudaErrorInvalidValue;
    }
    return cudaSuccess;
}

// Resident CTAs per SM of `kernel` at this launch shape (the occupancy API,
// cached per device in `cache`; `fallback` if the query fails).
template <class K>
static int resident_ctas(K kernel, int threads, size_t smem, int fallback, std::atomic<int> (&cache)[64]) {
    int dev = 0, occ = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && dev >= 0 && dev < 64) occ = cache[dev].load(std::memory_order_relaxed);
    if (!occ) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem) != cudaSuccess || occ <= 0)
            occ = fallback;
        if (dev >= 0 && dev < 64) cache[dev].store(occ, std::memory_order_relaxed);
    }
    return occ;
}

template <int ALG, int V, int NB, int STAGES, bool UNR = false, bool SLACK = true>
static cudaError_t launch_fixed_tma_ws(const uint8_t* d_msgs, uint32_t n, uint32_t L, uint8_t* d_out,
                                       cudaStream_t stream, bool input_ready = false) {
    using C = WsCfg<NB, STAGES, SLACK>;
    const Tuning& T = tuning();
    CUtensorMap map;
    cudaError_t e = encode_rows_map(&map, d_msgs, n, L, (uint32_t)C::kRows, T.tma_l2);
    if (e != cudaSuccess) return e;
    static std::atomic<uint64_t> attr_done{0};  // function attributes are per device
    e = set_smem_attr_once(attr_done, [] {
        return cudaFuncSetAttribute(k_fixed_tma_ws<ALG, V, NB, STAGES, UNR, SLACK>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    });
    if (e != cudaSuccess) return e;
    const uint32_t grid = (n + C::kRows - 1) / C::kRows;
    // PDL pays for short kernels (launch gap hidden: +5-17 %) and for grids
    // that fill every SM anyway.  A sub-wave grid of long messages is bound by
    // each message's dependent chain; early-launched CTAs can land two to an
    // SM there and run up to 30 % slower (profiles/ab_pdl_r1.txt), so those
    // launch normally.
    const bool pdl = grid >= (uint32_t)device_sms() || (L + 8u) / 64u + 1u <= 17u;
    // The next grid is released early (at entry) if this one is resident in a
    // single wave: at most $HB_TRIGGER_WAVE_PCT (100) % of the SMs' resident
    // CTA slots.  With the late wait the released grid computes beside this
    // one; half a wave (the round-1 rule) kept SM3 / SHA-1's 512-CTA grids of
    // 2^16 messages out: 0.74 -> 0.92 of the ALU bound at 2^16 x 1 KiB SM3
    // (profiles/r2/trigger_r2al/).
    static std::atomic<int> occ_cache[64];
    const int occ = resident_ctas(k_fixed_tma_ws<ALG, V, NB, STAGES, UNR, SLACK>, (kWsComputeWarps + 1) * 32,
                                  C::kSmem, WsOcc<ALG, NB, STAGES, SLACK>::kMinCtas, occ_cache);
    const uint32_t half_wave = (uint32_t)((uint64_t)device_sms() * (uint64_t)occ * T.trigger_wave_pct / 100u);
    const uint32_t early = input_ready && pdl && T.pdl
                               ? kEarlyLoad | (grid <= half_wave ? kEarlyTrigger : 0u) | (T.late_wait ? kLateWait : 0u)
                               : 0u;
    launch_pdl_smem(k_fixed_tma_ws<ALG, V, NB, STAGES, UNR, SLACK>, grid, (kWsComputeWarps + 1) * 32, C::kSmem,
                    stream, pdl, map, n, L, d_out, (uint32_t)T.tma_evict_first, early);
    return cudaGetLastError();
}

template <int ALG, int V, int NB, int STAGES>
static cudaError_t launch_fixed_tma_w1(const uint8_t* d_msgs, uint32_t n, uint32_t L, uint8_t* d_out,
                                       cudaStream_t stream, bool input_ready = false) {
    using C = TmaCfg<NB, STAGES, 1>;
    const Tuning& T = tuning();
    CUtensorMap map;
    cudaError_t e = encode_rows_map(&map, d_msgs, n, L, (uint32_t)C::kRows, T.tma_l2);
    if (e != cudaSuccess) return e;
    static std::atomic<uint64_t> attr_done{0};
    e = set_smem_attr_once(attr_done, [] {
        return cudaFuncSetAttribute(k_fixed_tma_w1<ALG, V, NB, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    C::kSmem);
    });
    if (e != cudaSuccess) return e;
    // resident CTAs per SM (shared memory bounds it, ~17 at 3 stages), queried once per device
    static std::atomic<int> occ_cache[64];
    const int occ = resident_ctas(k_fixed_tma_w1<ALG, V, NB, STAGES>, 32, C::kSmem,
                                  TmaOcc<ALG, NB, STAGES, 1>::kMinCtas, occ_cache);
    const uint32_t grid = (n + C::kRows - 1) / C::kRows;
    const bool pdl = grid >= (uint32_t)device_sms() || (L + 8u) / 64u + 1u <= 17u;  // as launch_fixed_tma_ws
    const uint32_t half_wave = (uint32_t)((uint64_t)device_sms() * (uint64_t)occ * T.trigger_wave_pct / 100u);
    const uint32_t early = input_ready && pdl && T.pdl
                               ? kEarlyLoad | (grid <= half_wave ? kEarlyTrigger : 0u) | (T.late_wait ? kLateWait : 0u)
                               : 0u;
    launch_pdl_smem(k_fixed_tma_w1<ALG, V, NB, STAGES>, grid, 32, C::kSmem, stream, pdl, map, n, L, d_out, early);
    return cudaGetLastError();
}

#ifdef HB_AB
#include "hb_ab_kernels.cuh"
#endif

// Default tile per algorithm (B200-measured, profiles/variant_sweep_r1d.txt and
// _r1e.txt, interleaved rounds): the warp-specialised 3-stage ring with round
// variant 1 for MD5 and SM3 (SM3's 61 registers make two messages per thread
// lose occupancy); SHA-1 gains 4 % from two messages per thread (7.38 vs
// 7.69 ms at 2^24 x 1 KiB).  Below tuning().small_n messages (2^18) one
// message per thread so the grid still covers every SM (SHA-1's NB=2 tiles
// halve the CTA count: 4096 x 64 KiB 251 vs 428 GB/s, profiles/ab_small_r1.txt).
template <int ALG>
static cudaError_t launch_tma_dispatch(const uint8_t* src, uint32_t n, uint32_t L, uint8_t* dst, cudaStream_t s,
                                       bool input_ready) {
#ifdef HB_AB
    if (tuning().tma_cfg >= 0 || tuning().variant >= 0) return launch_tma_ab<ALG>(src, n, L, dst, s);
#endif
    // MD5: from 2^16 messages single-warp CTAs with two messages per thread and
    // round variant 6 (every other round sums a + M + K in one IADD3: 4
    // instead of 5 instructions there), 5-13 % faster than the 4+1-warp tile
    // from 2^16 to 2^22 x 1 KiB (profiles/r2/ab_v467_r2o.txt, ab_mid_r2p.txt:
    // variant 6 beats 4 by 2-5 % in this tile from 2^20 messages).  Smaller,
    // chain-bound batches keep one message per thread in the 4+1-warp tile
    // with variant 6 (variant 3's short f -> add -> rotate chain, every other
    // round's off-chain sum in one IADD3): -7 % against variant 3 there.
    // From 2^22 messages (>= 14 warps per scheduler) three messages per thread:
    // -2 % at configs[1] (profiles/r2/ab_headline_r2y.txt), even at 2^18-2^22,
    // -20 % at 2^16 (too few warps left).
    if constexpr (ALG == kMd5) {
        if ((uint64_t)n < tuning().chain_n) return launch_fixed_tma_ws<ALG, 6, 1, 3>(src, n, L, dst, s, input_ready);
        if ((uint64_t)n >= tuning().md5_nb3_n) return launch_fixed_tma_w1<ALG, 6, 3, 3>(src, n, L, dst, s, input_ready);
        return launch_fixed_tma_w1<ALG, 6, 2, 3>(src, n, L, dst, s, input_ready);
    }
    if ((uint64_t)n < tuning().small_n || ALG != kSha1)
        return launch_fixed_tma_ws<ALG, kVarBal, 1, 3>(src, n, L, dst, s, input_ready);
    return launch_fixed_tma_ws<ALG, kVarBal, 2, 3>(src, n, L, dst, s, input_ready);
}

// Compile-time-width kernel for L in {16, 32, 48, 64, 128}; MD5 one-block
// rows (<= 32 B) in batches >= 2^20 take two adjacent rows per thread (+3-4 %;
// 48-byte rows lose 2 %, two-block rows 1-9 %, profiles/ab_small_r1d.txt).
template <int ALG, int L>
static void launch_small(const uint8_t* d_msgs, uint64_t n, uint8_t* d_out, cudaStream_t s, bool input_ready) {
    constexpr unsigned kBlk = 128;
    // early start (see k_fixed_small): the next grid is released early when
    // this one is resident in one wave ($HB_TRIGGER_WAVE_PCT of the SM's 16
    // CTA slots).
    const auto early = [&](unsigned grid) -> uint32_t {
        return input_ready && tuning().pdl ? kEarlyLoad |
                                                 (grid <= 16u * tuning().trigger_wave_pct / 100u * (unsigned)device_sms()
                                                      ? kEarlyTrigger : 0u) |
                                                 (tuning().late_wait ? kLateWait : 0u)
                                           : 0u;
    };
    if constexpr (ALG == kMd5 && L <= 32) {
        if (n >= (1ull << 20) && tuning().small_pair) {
            const unsigned g = (unsigned)(((n + 1) / 2 + kBlk - 1) / kBlk);
            launch_pdl(k_fixed_small<ALG, L, kVarBal, 2>, g, kBlk, s, d_msgs, n, d_out, early(g));
            return;
        }
    }
    const unsigned g = (unsigned)((n + kBlk - 1) / kBlk);
    launch_pdl(k_fixed_small<ALG, L, kVarBal>, g, kBlk, s, d_msgs, n, d_out, early(g));
}

template <int ALG>
static cudaError_t launch_fixed_alg(const uint8_t* d_msgs, uint64_t n, uint64_t L, uint8_t* d_out,
                                    cudaStream_t stream, uint32_t flags) {
    using H = HashAlg<ALG>;
    const Tuning& T = tuning();
    const bool aligned = L > 0 && (L % 16) == 0 && (reinterpret_cast<uintptr_t>(d_msgs) % 16) == 0 &&
                         L < (1ull << 31);
    const bool direct = (flags & HB_FLAG_NO_TMA) || L <= T.direct_max_len;
    bool input_ready = (flags & HB_FLAG_INPUT_READY) != 0;
#ifdef HB_AB
    input_ready = input_ready || T.input_ready;
#endif
    if (aligned && !direct) {
        // TMA coordinates are int32: split very large batches into row slabs.
        const uint64_t slab = 1ull << 30;
        for (uint64_t r0 = 0; r0 < n; r0 += slab) {
            const uint64_t rn = (n - r0) < slab ? (n - r0) : slab;
            const cudaError_t e = launch_tma_dispatch<ALG>(d_msgs + r0 * L, (uint32_t)rn, (uint32_t)L,
                                                           d_out + r0 * H::kDigestBytes, stream, input_ready);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }
#ifdef HB_AB
    if (aligned && T.small_kernel_ab) return launch_small_ab<ALG>(d_msgs, n, L, d_out, stream);
#endif
    const unsigned grid = (unsigned)((n + 127) / 128);
    const bool small_ok = aligned && T.small_kernel;
    if (small_ok && L == 16) launch_small<ALG, 16>(d_msgs, n, d_out, stream, input_ready);
    else if (small_ok && L == 32) launch_small<ALG, 32>(d_msgs, n, d_out, stream, input_ready);
    else if (small_ok && L == 48) launch_small<ALG, 48>(d_msgs, n, d_out, stream, input_ready);
    else if (small_ok && L == 64) launch_small<ALG, 64>(d_msgs, n, d_out, stream, input_ready);
    else if (small_ok && L == 128) launch_small<ALG, 128>(d_msgs, n, d_out, stream, input_ready);
    else if (aligned) launch_plain(k_fixed_direct<ALG>, grid, 128, stream, d_msgs, n, (uint32_t)L, d_out);
    else launch_plain(k_generic<ALG, false>, grid, 128, stream, d_msgs, d_msgs + n * L,
                      (const uint64_t*)nullptr, (uint64_t)0, (const uint32_t*)nullptr, L, n, d_out);
    return cudaGetLastError();
}

template <int ALG>
static cudaError_t launch_varlen_alg(const uint8_t* d_data, uint64_t data_bytes, const uint64_t* d_offsets,
                                     uint64_t offset_base, uint64_t n, uint8_t* d_out, void* d_scratch,
                                     cudaStream_t stream, uint32_t flags) {
#ifdef HB_AB
    if (varlen_ab_selected(flags)) return launch_varlen_ab<ALG>(d_data, data_bytes, d_offsets, offset_base, n, d_out,
                                                                d_scratch, stream, flags);
#endif
    if (flags & (HB_FLAG_VARLEN_WORDS | HB_FLAG_VARLEN_COOP)) {
        snprintf(tma_error_buf(), kTmaErrLen, "A/B varlen kernel flags need a -DHB_AB build");
        return cudaErrorInvalidValue;
    }
    const uint32_t* perm = nullptr;
    cudaError_t e = launch_varlen_sort(ALG, d_data, d_offsets, offset_base, n, d_scratch, stream, flags, &perm, 4);
    if (e != cudaSuccess) return e;
    // MD5 (issue-bound, windowed q-major sort): the lean software-pipelined
    // block loop -- block b+1's window in flight during b's compression (-6 %
    // vs the plain kernel, profiles/ab_varlen_r2d.txt), ~18 fewer instructions
    // per block than k_varlen16<MD5, 1> (-1.4 %, profiles/r2/ab_varlen_r2o.txt)
    // -- with L2 policies on the first window (evict_last: its leading granule
    // is the previous message's tail, read by that message's thread much later)
    // and on the tail (evict_first): DRAM traffic 1.063 -> 1.040 x algorithmic
    // at equal time (profiles/r2/ncu_varlen_r2.md).  SM3 (ALU-bound): the
    // uniform-finish loop, nb compressions per warp instead of nb + 1 (-3 %,
    // profiles/r2/ab_varlen_r2s.txt).  SHA-1 keeps the plain kernel (the
    // uniform finish costs it 12 %).
    const unsigned grid = (unsigned)((n + 127) / 128);
    if (ALG == kMd5 && tuning().varlen_pf)
        launch_plain(k_varlen16l<ALG, false, -1, true>, grid, 128, stream, d_data, d_data + data_bytes, d_offsets,
                     offset_base, perm, n, d_out);
    else if (ALG == kSm3)
        launch_plain(k_varlen16g<ALG>, grid, 128, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm,
                     n, d_out);
    else
        launch_plain(k_varlen16<ALG, 0>, (unsigned)((n + 127) / 128), 128, stream, d_data, d_data + data_bytes,
                     d_offsets, offset_base, perm, n, d_out);
    return cudaGetLastError();
}

// Paper workload.  Widths 2-10 below ~1.07e10: the runs-of-ten kernel (MD5
// compresses messages j and j+5 together, +3 %; SHA-1 / SM3 lose 28 / 6 % that
// way); otherwise one message per thread with FMA-pipe digits (round variant
// 3 for SHA-1, 1 otherwise; profiles/ab_decimal_r1b-d.txt).
template <int ALG, int W>
static void dec_launch(uint64_t start, uint64_t count, uint8_t* d_out, cudaStream_t s) {
    const Tuning& T = tuning();
    if (count == 0) return;
#ifdef HB_AB
    if (T.dec_ab) { dec_launch_ab<ALG, W>(start, count, d_out, s); return; }
#endif
    if constexpr (W >= 2 && W <= 10) {
        if (T.dec_run && (start + count) / 10u < (1ull << 30) - 1) {
            const uint64_t threads = (start + count + 9u) / 10u - start / 10u;
            const unsigned g = (unsigned)((threads + 127) / 128);
            launch_plain(k_decimal_run<ALG, W, kVarBal, ALG == kMd5>, g, 128, s, start, count, d_out);
            return;
        }
    }
    const unsigned grid = (unsigned)((count + 127) / 128);
    launch_plain(k_decimal<ALG, W, ALG == kSha1 ? kVarBal3 : kVarBal, true>, grid, 128, s, start, count, d_out);
}

template <int ALG>
static cudaError_t launch_decimal_alg(uint64_t start, uint64_t count, int width, uint8_t* d_out, cudaStream_t s) {
    switch (width) {
#define HB_DEC_CASE(W) case W: dec_launch<ALG, W>(start, count, d_out, s); break;
    HB_DEC_CASE(1) HB_DEC_CASE(2) HB_DEC_CASE(3) HB_DEC_CASE(4) HB_DEC_CASE(5) HB_DEC_CASE(6) HB_DEC_CASE(7)
    HB_DEC_CASE(8) HB_DEC_CASE(9) HB_DEC_CASE(10) HB_DEC_CASE(11) HB_DEC_CASE(12) HB_DEC_CASE(13)
    HB_DEC_CASE(14) HB_DEC_CASE(15) HB_DEC_CASE(16) HB_DEC_CASE(17) HB_DEC_CASE(18) HB_DEC_CASE(19)
    HB_DEC_CASE(20)
#undef HB_DEC_CASE
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// -------------------------------------------------------------------------
// One short message (hb_digest_small, crypto.digest: batch.py:102-109).  The
// latency of a single digest is copies and launches, not hashing: the bytes
// travel in the kernel's parameter block (host-zero-padded little-endian
// words, so no H2D copy and no tail masking) and the digest is stored
// straight into mapped pinned host memory (no D2H copy) -- one launch and
// one stream synchronise per call.  One thread runs the block chain, as the
// batch kernels do per message.  Two parameter sizes so a short
// message does not ship 4 KiB of zeros with its launch.
template <int ALG> constexpr int kSmallVariant = ALG == kMd5 ? 5 : kVarBal;

template <int CAP>
struct SmallMsg {
    uint32_t w[CAP / 4 + 16];  // message bytes, then zeros through the tail block
    uint64_t len;
    uint32_t seq;  // != 0: publish seq at out + kSmallSeqOffset after the digest
};
constexpr int kSmallSeqOffset = 48;

template <int ALG, int CAP, int V>
__global__ void __launch_bounds__(32) k_digest_small(const __grid_constant__ SmallMsg<CAP> m, uint8_t* out) {
    using H = HashAlg<ALG, V>;
    // The parameter bank is read through the constant cache: a dependent
    // per-block read there costs a miss in the chain (1.5x at 4 KiB), so the
    // warp first stages the used words in shared memory (8-byte loads), then
    // lane 0 runs the chain with the next block's words loaded ahead.
    __shared__ uint2 sw[(CAP / 4 + 16) / 2];
    const uint32_t nfull = (uint32_t)(m.len >> 6);
    const uint2* pw = reinterpret_cast<const uint2*>(m.w);
    for (uint32_t i = threadIdx.x; i < 8u * (nfull + 1u); i += 32u) sw[i] = pw[i];
    __syncwarp();
    if (threadIdx.x != 0) return;
    const uint32_t* w = reinterpret_cast<const uint32_t*>(sw);
    uint32_t st[H::kStateWords];
    H::init(st);
    uint32_t nxt[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) nxt[j] = w[j];
#pragma unroll 1
    for (uint32_t b = 0; b < nfull; ++b) {
        uint32_t raw[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            raw[j] = nxt[j];
            nxt[j] = w[16 * (b + 1) + j];
        }
        compress1<ALG, V>(st, raw);
    }
    md_finish<ALG, V>(st, nxt, (uint32_t)(m.len & 63u), m.len);
    store_digest<ALG>(out, st);
    // The host polls this word instead of synchronising the stream; the
    // release orders the digest stores before it at system scope.
    if (m.seq) asm volatile("st.release.sys.u32 [%0], %1;" ::"l"(out + kSmallSeqOffset), "r"(m.seq) : "memory");
}

}  // namespace hb
