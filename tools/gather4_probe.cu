// Feasibility probe: can TMA tile::gather4 feed the variable-length kernels?
//
// The varlen MD5 kernel is bound by L1 wavefronts of per-thread 16-byte loads
// from 32 different messages.  gather4 fetches four 2-D tensor
// rows at arbitrary row indices in one TMA op.  Viewing the data buffer as
// rows of 80 bytes (one 64-byte block + the 16-byte realignment slack) at a
// 16-byte row pitch -- overlapping rows -- one op would stage the current
// block of four messages.  This measures (1) whether the tensor map encodes,
// (2) bytes/s the TMA engine sustains for that access pattern, against plain
// per-thread LDG.128 windows over the same messages.  No hashing.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2407_09333_b200/csrc \
//      -o tools/gather4_probe tools/gather4_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <random>
#include <vector>

#include "hb_ptx.cuh"

using namespace hb;

#define CK(x)                                                                             \
    do {                                                                                  \
        cudaError_t e_ = (x);                                                             \
        if (e_ != cudaSuccess) {                                                          \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                      \
        }                                                                                 \
    } while (0)

constexpr int kWin = 80;            // bytes per staged window
constexpr int kMsgs = 128;          // messages per CTA (4 consumer warps)
constexpr int kGroupPitch = 384;    // 4 windows (320 B) padded to a 128-byte multiple
constexpr int kStageBytes = kMsgs / 4 * kGroupPitch;  // 12 KiB
constexpr int kStages = 4;

__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int r0, int r1,
                                            int r2, int r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
        : "memory");
}

// One CTA = 128 messages of `nblocks` blocks; message m's window for block b
// is tensor row rows[m] + 4b.
__global__ void __launch_bounds__(160) k_gather4(const __grid_constant__ CUtensorMap map, const uint32_t* rows,
                                                 int nblocks, uint32_t* sink) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* ring = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    uint64_t* empty = full + kStages;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t* r = rows + (size_t)blockIdx.x * kMsgs;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 4);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == 4) {
        if (lane == 0) {
            prefetch_tmap(&map);
            uint32_t s = 0, ph = 0;
            for (int b = 0; b < nblocks; ++b) {
                if (b >= kStages) mbar_wait_parity(&empty[s], ph ^ 1u);
                mbar_arrive_expect_tx(&full[s], kMsgs * kWin);
                uint8_t* st = ring + s * kStageBytes;
                for (int g = 0; g < kMsgs / 4; ++g)
                    tma_gather4(st + g * kGroupPitch, &map, &full[s], 0, r[4 * g] + 4 * b, r[4 * g + 1] + 4 * b,
                                r[4 * g + 2] + 4 * b, r[4 * g + 3] + 4 * b);
                if (++s == kStages) { s = 0; ph ^= 1u; }
            }
        }
        return;
    }
    const uint32_t t = threadIdx.x;
    const uint32_t off = (t >> 2) * kGroupPitch + (t & 3) * kWin;
    uint32_t acc = 0, s = 0, ph = 0;
    for (int b = 0; b < nblocks; ++b) {
        mbar_wait_parity(&full[s], ph);
        const uint4* w = reinterpret_cast<const uint4*>(ring + s * kStageBytes + off);
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const uint4 v = w[k];
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (++s == kStages) { s = 0; ph ^= 1u; }
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

// Baseline: per-thread 128-bit loads of the same windows (k_varlen16's pattern).
__global__ void __launch_bounds__(128) k_ldg(const uint8_t* data, const uint32_t* rows, int nblocks, uint32_t* sink) {
    const uint32_t m = blockIdx.x * kMsgs + threadIdx.x;
    const uint4* w = reinterpret_cast<const uint4*>(data) + rows[m];
    uint32_t acc = 0;
    for (int b = 0; b < nblocks; ++b) {
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const uint4 v = __ldg(w + 4 * b + k);
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

typedef CUresult (*PFN_encode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
    const int nblocks = argc > 1 ? atoi(argv[1]) : 32;  // blocks per message (2 KiB messages)
    const uint64_t nmsg = argc > 2 ? strtoull(argv[2], 0, 10) : (1ull << 22);
    const int window = argc > 3 ? atoi(argv[3]) : 8192;  // shuffle messages within windows (the windowed sort)
    const uint64_t msg_bytes = (uint64_t)nblocks * 64 + 16;
    const uint64_t bytes = nmsg * msg_bytes + 256;
    uint8_t* d = nullptr;
    CK(cudaMalloc(&d, bytes));
    CK(cudaMemset(d, 1, bytes));
    std::vector<uint32_t> rows(nmsg);
    std::vector<uint32_t> order(nmsg);
    for (uint64_t i = 0; i < nmsg; ++i) order[i] = (uint32_t)i;
    std::mt19937 rng(7);
    for (uint64_t w0 = 0; w0 < nmsg; w0 += window)
        std::shuffle(order.begin() + w0, order.begin() + std::min<uint64_t>(nmsg, w0 + window), rng);
    for (uint64_t i = 0; i < nmsg; ++i) rows[i] = (uint32_t)(((uint64_t)order[i] * msg_bytes) / 16);
    uint32_t *d_rows = nullptr, *d_sink = nullptr;
    CK(cudaMalloc(&d_rows, nmsg * 4));
    CK(cudaMalloc(&d_sink, 16));
    CK(cudaMemcpy(d_rows, rows.data(), nmsg * 4, cudaMemcpyHostToDevice));

    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q));
    PFN_encode enc = reinterpret_cast<PFN_encode>(fn);
    CUtensorMap map;
    const uint64_t nrows = (bytes - kWin) / 16 + 1;
    const cuuint64_t dims[2] = {(cuuint64_t)kWin, nrows};
    const cuuint64_t strides[1] = {16};
    const cuuint32_t box[2] = {(cuuint32_t)kWin, 1};
    const cuuint32_t estr[2] = {1, 1};
    CUresult rc = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, d, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode 80-byte rows at 16-byte pitch: CUresult %d\n", (int)rc);
    if (rc != CUDA_SUCCESS) return 2;

    const int smem = kStages * kStageBytes + 2 * kStages * 8;
    CK(cudaFuncSetAttribute(k_gather4, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const unsigned grid = (unsigned)(nmsg / kMsgs);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const double useful = (double)nmsg * nblocks * 64;
    for (int rep = 0; rep < 3; ++rep) {
        for (int mode = 0; mode < 2; ++mode) {
            CK(cudaEventRecord(e0));
            for (int it = 0; it < 5; ++it) {
                if (mode == 0)
                    k_gather4<<<grid, 160, smem>>>(map, d_rows, nblocks, d_sink);
                else
                    k_ldg<<<grid, 128>>>(d, d_rows, nblocks, d_sink);
            }
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            CK(cudaGetLastError());
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            ms /= 5;
            printf("{\"mode\": \"%s\", \"nblocks\": %d, \"msgs\": %llu, \"window\": %d, \"ms\": %.4f, "
                   "\"useful_GBps\": %.1f, \"window_GBps\": %.1f}\n",
                   mode == 0 ? "tma_gather4" : "ldg128_per_thread", nblocks, (unsigned long long)nmsg, window, ms,
                   useful / ms / 1e6, useful * 80 / 64 / ms / 1e6);
        }
    }
    return 0;
}
