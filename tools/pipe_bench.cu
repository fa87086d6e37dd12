// pipe_bench.cu -- measured integer-pipe throughput on B200 (sm_100a) for the
// SASS the hash kernels are made of (LOP3, SHF, IADD3/VIADD, LEA.HI, IMAD,
// IMAD.HI, PRMT) alone and in mixes.  One 1024-thread CTA per SM, 8
// independent dependency chains per thread; prints lanes/clk/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_bench pipe_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kChains = 8;

#define BODY_LOP3(x, y, z) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x) : "r"(y), "r"(z))
#define BODY_SHF(x) asm volatile("shf.l.wrap.b32 %0, %0, %0, 7;" : "+r"(x))
#define BODY_ADDI(x) asm volatile("add.u32 %0, %0, 0x5a827999;" : "+r"(x))
#define BODY_ADD3(x, y, z) asm volatile("{ .reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %2; }" : "+r"(x) : "r"(y), "r"(z))
#define BODY_IMAD(x, y, z) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(y), "r"(z))
#define BODY_IMADHI(x, y, z) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(y), "r"(z))
#define BODY_PRMT(x, y) asm volatile("prmt.b32 %0, %0, %1, 0x0123;" : "+r"(x) : "r"(y))
// rotate-then-add: b + rotl(x, 7) -- ptxas emits LEA.HI
#define BODY_ROTADD(x, y) asm volatile("{ .reg .u32 t; shf.l.wrap.b32 t, %0, %0, 7; add.u32 %0, t, %1; }" : "+r"(x) : "r"(y))

template <int MODE>
__global__ void __launch_bounds__(1024, 1) kern(uint32_t seed, uint32_t y, uint32_t z, uint32_t* out, long long* cyc) {
    uint32_t v[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) v[c] = seed + threadIdx.x * 7 + c;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            if (MODE == 0) { BODY_LOP3(v[c], y, z); }
            if (MODE == 1) { BODY_SHF(v[c]); }
            if (MODE == 2) { asm volatile("add.u32 %0, %0, %1;" : "+r"(v[c]) : "r"(v[(c + 1) % kChains])); }
            if (MODE == 3) { BODY_IMAD(v[c], y, z); }
            if (MODE == 4) { BODY_IMADHI(v[c], y, z); }
            if (MODE == 5) { BODY_PRMT(v[c], y); }
            if (MODE == 6) { BODY_ROTADD(v[c], y); }
            if (MODE == 7) { BODY_LOP3(v[c], y, z); BODY_ADDI(v[c]); }      // LOP3 + VIADD in one chain
            if (MODE == 8) { if (c & 1) BODY_LOP3(v[c], y, z); else BODY_IMAD(v[c], y, z); } // LOP3 + IMAD
            if (MODE == 9) { if (c & 1) BODY_LOP3(v[c], y, z); else BODY_IMADHI(v[c], y, z); }
            if (MODE == 10) { if (c & 1) BODY_SHF(v[c]); else BODY_IMAD(v[c], y, z); }
            if (MODE == 11) { BODY_ADD3(v[c], v[(c + 1) % kChains], y); }
            if (MODE == 12) { BODY_LOP3(v[c], y, z); BODY_ADD3(v[c], v[(c + 1) % kChains], y); }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc ^= v[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

static const char* kNames[] = {"LOP3", "SHF.L.W", "a+b (2-reg add)", "IMAD", "IMAD.HI", "PRMT",
                               "rotl+add (LEA.HI)", "LOP3;+imm chain", "LOP3+IMAD 50/50", "LOP3+IMAD.HI 50/50",
                               "SHF+IMAD 50/50", "a+b+c (IADD3)", "LOP3;a+b+c chain"};

template <int MODE>
static void run(int sms, uint32_t* out, long long* cyc, long long* hcyc) {
    kern<MODE><<<sms, 1024>>>(1u, 0x9e3779b9u, 0x7f4a7c15u, out, cyc);
    kern<MODE><<<sms, 1024>>>(1u, 0x9e3779b9u, 0x7f4a7c15u, out, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(hcyc, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < sms; ++i) mean += (double)hcyc[i];
    mean /= sms;
    const double ops = 1024.0 * kIters * kChains;  // instructions x lanes per CTA (= per SM)
    const double per = (MODE == 7 || MODE == 12) ? 2.0 : 1.0;  // two SASS ops per chain step
    printf("%-24s %7.2f lanes/clk/SM (%.0f cycles)\n", kNames[MODE], per * ops / mean, mean);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(uint32_t) * sms * 1024);
    cudaMalloc(&cyc, sizeof(long long) * sms);
    long long* hcyc = new long long[sms];
    printf("SMs=%d, 1024 threads/SM, %d chains x %d iters\n", sms, kChains, kIters);
    run<0>(sms, out, cyc, hcyc); run<1>(sms, out, cyc, hcyc); run<2>(sms, out, cyc, hcyc);
    run<3>(sms, out, cyc, hcyc); run<4>(sms, out, cyc, hcyc); run<5>(sms, out, cyc, hcyc);
    run<6>(sms, out, cyc, hcyc); run<7>(sms, out, cyc, hcyc); run<8>(sms, out, cyc, hcyc);
    run<9>(sms, out, cyc, hcyc); run<10>(sms, out, cyc, hcyc); run<11>(sms, out, cyc, hcyc);
    run<12>(sms, out, cyc, hcyc);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
    return 0;
}
