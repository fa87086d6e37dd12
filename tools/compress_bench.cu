// compress_bench.cu -- compute-only ceiling of each compression variant.
// Every thread chains R compressions on register-resident data (no memory
// traffic), at the occupancy of the real kernels; prints ns and SM-cycles per
// 64-byte block per SM, so the TMA kernels can be compared against the pure
// instruction-issue limit of the same round code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2407_09333_b200/csrc -o tools/compress_bench tools/compress_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "hb_algos.cuh"

using namespace hb;
constexpr int kR = 256;

template <int ALG, int V, int NB>
__global__ void __launch_bounds__(128) kern(uint32_t seed, uint32_t* out) {
    using H = HashAlg<ALG, V>;
    uint32_t st[NB][H::kStateWords];
    uint32_t raw[NB][16];
#pragma unroll
    for (int q = 0; q < NB; ++q) {
        H::init(st[q]);
#pragma unroll
        for (int j = 0; j < 16; ++j) raw[q][j] = seed * (threadIdx.x + 17 * j + 1) + blockIdx.x + q;
    }
    for (int r = 0; r < kR; ++r) {
        H::template compress_n<NB>(st, raw);
#pragma unroll
        for (int q = 0; q < NB; ++q) raw[q][r & 15] ^= st[q][0];  // loop-carried, defeats hoisting
    }
    uint32_t acc = 0;
#pragma unroll
    for (int q = 0; q < NB; ++q)
#pragma unroll
        for (int i = 0; i < H::kStateWords; ++i) acc ^= st[q][i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int ALG, int V, int NB>
static void run(const char* name, int ctas_per_sm, int sms, uint32_t* out, int clk_mhz) {
    const int grid = sms * ctas_per_sm * 4;
    kern<ALG, V, NB><<<grid, 128>>>(3u, out);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<ALG, V, NB><<<grid, 128>>>(5u, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double blocks = (double)grid * 128 * NB * kR;
    const double ns_blk_sm = ms * 1e6 * sms / blocks;
    printf("%-8s V%d NB%d: %8.3f ms  %.4f ns/block/SM  %.3f cycles/block/SM @%d MHz\n", name, V, NB, ms, ns_blk_sm,
           ns_blk_sm * clk_mhz / 1000.0, clk_mhz);
}

template <int ALG>
static void run_lat(const char* name, int sms, uint32_t* out, int clk_mhz) {
    kern<ALG, -1, 1><<<sms, 32>>>(3u, out);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<ALG, -1, 1><<<sms, 32>>>(5u, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double ns = ms * 1e6 / kR;
    printf("%-8s chain latency (1 warp/SM): %.1f ns = %.0f cycles per compression @%d MHz\n", name, ns,
           ns * clk_mhz / 1000.0, clk_mhz);
}

int main(int argc, char** argv) {
    int sms = 0, clk_khz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const int clk = clk_khz / 1000;
    uint32_t* out;
    cudaMalloc(&out, sizeof(uint32_t) * sms * 64 * 128 * 4);
    run<kMd5, 0, 1>("md5", 8, sms, out, clk);
    run<kMd5, 1, 1>("md5", 8, sms, out, clk);
    run<kMd5, 2, 1>("md5", 8, sms, out, clk);
    run<kMd5, 3, 1>("md5", 8, sms, out, clk);
    run<kMd5, 1, 2>("md5", 4, sms, out, clk);
    run<kMd5, 3, 2>("md5", 4, sms, out, clk);
    run<kSha1, 0, 1>("sha1", 8, sms, out, clk);
    run<kSha1, 1, 1>("sha1", 8, sms, out, clk);
    run<kSha1, 2, 1>("sha1", 8, sms, out, clk);
    run<kSha1, 1, 2>("sha1", 4, sms, out, clk);
    run<kSm3, 0, 1>("sm3", 6, sms, out, clk);
    run<kSm3, 1, 1>("sm3", 6, sms, out, clk);
    run<kSm3, 2, 1>("sm3", 6, sms, out, clk);
    run<kSm3, 3, 1>("sm3", 6, sms, out, clk);
    // Dependent-chain latency: ONE warp per SM (32 threads per CTA, one CTA
    // per SM), so nothing hides the round-to-round dependency -- cycles per
    // compression of a single message = the latency bound of a batch with
    // fewer messages than the GPU can overlap (configs[4] small-n points).
    run_lat<kMd5>("md5", sms, out, clk);
    run_lat<kSha1>("sha1", sms, out, clk);
    run_lat<kSm3>("sm3", sms, out, clk);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
