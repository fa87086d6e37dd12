// hb_algos.cuh -- SHA-1 / MD5 / SM3 compression, one message per lane-slot.
//
// Each function keeps the chaining state and the whole message schedule in
// registers (fully unrolled, constant indices only) and compiles to
// LOP3 (boolean functions), SHF.L.W / LEA.HI (rotates, rotate+add), IADD3 /
// IMAD / VIADD (adds) and PRMT (byte swaps).  Inputs are the 16 RAW
// little-endian words of a 64-byte block as loaded from memory; the
// big-endian algorithms byte-swap inside.
//
// compress_n<NB> runs NB independent messages (of one thread) round by round,
// interleaved in source order, so the scheduler can overlap their dependency
// chains (instruction-level parallelism on top of warp parallelism).
//
// Reference semantics followed (paths relative to the reference repo):
//   SHA-1  pkg/src/hetoc/crypto/sha1.py:21-37   (batch kernel batch.py:145-170)
//   MD5    pkg/src/hetoc/crypto/md5.py:32-54    (batch kernel batch.py:178-202)
//   SM3    pkg/src/hetoc/crypto/sm3.py:33-63    (batch kernel batch.py:225-260)
//   padding _pad sha1.py:14-18 / md5.py:25-29 / sm3.py:26-30, batch.py:128-138
#pragma once
#include <stdint.h>

namespace hb {

enum Alg : int { kSha1 = 0, kMd5 = 1, kSm3 = 2 };

__device__ __forceinline__ uint32_t rotl(uint32_t x, int n) { return __funnelshift_l(x, x, n); }
__device__ __forceinline__ uint32_t bswap(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// Boolean round functions; each lowers to one LOP3.
__device__ __forceinline__ uint32_t xor3(uint32_t x, uint32_t y, uint32_t z) { return x ^ y ^ z; }             // 0x96
__device__ __forceinline__ uint32_t ch(uint32_t x, uint32_t y, uint32_t z) { return z ^ (x & (y ^ z)); }       // 0xCA
__device__ __forceinline__ uint32_t maj(uint32_t x, uint32_t y, uint32_t z) { return (x & y) | (z & (x | y)); } // 0xE8

// ------------------------------------------------------- pipe balancing --
// On sm_100 LOP3 / SHF / PRMT / IADD3 / LEA.HI all issue to the ALU pipe (64
// lanes/clk/SM, tools/pipe_bench.cu), while IMAD runs on the FMA pipe at the
// same rate and VIADD (register + immediate) does not occupy the ALU pipe.
// ptxas lowers every hash round to ALU ops, so the kernels start out
// ALU-bound with the FMA pipe idle (ncu: ALU 92-97 %, FMA 5-17 %).
// Multiplying by an *opaque* 1 (a __constant__ word ptxas cannot fold)
// forces an addition onto the FMA pipe as IMAD; rotl_f does a rotate as IMAD +
// IMAD.HI (the latter is half rate, so it is used sparingly).  Which rounds use
// which form is a compile-time "variant" (A/B-measured on the B200).
__constant__ uint32_t c_opaque[33] = {
    1u, 2u, 4u, 8u, 16u, 32u, 64u, 128u, 256u, 512u, 1024u, 2048u, 4096u, 8192u, 16384u, 32768u, 65536u,
    1u << 17, 1u << 18, 1u << 19, 1u << 20, 1u << 21, 1u << 22, 1u << 23, 1u << 24, 1u << 25, 1u << 26,
    1u << 27, 1u << 28, 1u << 29, 1u << 30, 1u << 31, 1u};
__device__ __forceinline__ uint32_t add_f(uint32_t a, uint32_t b) { return a * c_opaque[32] + b; }   // IMAD
// A second, distinct opaque 1 (c_opaque[0]): ptxas may not factor x*one + y*one
// into (x + y)*one across the two, which would pull adds back onto the
// round's critical path.
__device__ __forceinline__ uint32_t add_g(uint32_t a, uint32_t b) { return a * c_opaque[0] + b; }    // IMAD
__device__ __forceinline__ uint32_t rotl_f(uint32_t x, int n) {                                       // IMAD.HI + IMAD
    return __umulhi(x, c_opaque[n]) + x * c_opaque[n];
}

// Variant ids (template parameter V of the compress functions).
constexpr int kVarPlain = 0;  // plain C arithmetic, ptxas' choice (ALU-heavy)
constexpr int kVarBal = 1;    // additions partly routed to IMAD
constexpr int kVarBal2 = 2;   // + more FMA-pipe work (algorithm specific, see below)
constexpr int kVarBal3 = 3;
constexpr int kNumVariants = 4;

template <int ALG, int V = -1> struct HashAlg;

// Default (tuned) variant per algorithm -- used by every kernel that does not
// take an explicit variant (generic / varlen / decimal).  Measured A/B on the
// B200 (profiles/variant_sweep_r1.txt): variant 1 is best for all three.
template <int ALG> struct DefaultVariant { static constexpr int value = kVarBal; };

// ------------------------------------------------------------------ SHA-1 --
// Variants: 1 = round adds e+W+K+f via IMAD/VIADD (then LEA.HI for +rotl(a,5));
// 2 = 1 + schedule rotl1 via IMAD/IMAD.HI on every expanded word;
// 3 = 1 + schedule rotl1 via IMAD/IMAD.HI on every other expanded word.
template <int V> struct HashAlg<kSha1, V> {
    static constexpr int kStateWords = 5;
    static constexpr int kDigestBytes = 20;
    static constexpr bool kBigEndian = true;
    static constexpr int kV = V < 0 ? DefaultVariant<kSha1>::value : V;

    __device__ __forceinline__ static void init(uint32_t s[5]) {   // sha1.py:5
        s[0] = 0x67452301u; s[1] = 0xEFCDAB89u; s[2] = 0x98BADCFEu; s[3] = 0x10325476u; s[4] = 0xC3D2E1F0u;
    }

    template <int NB>
    __device__ __forceinline__ static void compress_n(uint32_t (&s)[NB][5], const uint32_t (&raw)[NB][16]) {
        uint32_t w[NB][16], a[NB], b[NB], c[NB], d[NB], e[NB];
#pragma unroll
        for (int q = 0; q < NB; ++q) {
#pragma unroll
            for (int t = 0; t < 16; ++t) w[q][t] = bswap(raw[q][t]);  // sha1.py:22 (">16I")
            a[q] = s[q][0]; b[q] = s[q][1]; c[q] = s[q][2]; d[q] = s[q][3]; e[q] = s[q][4];
        }
#pragma unroll
        for (int t = 0; t < 80; ++t) {
#pragma unroll
            for (int q = 0; q < NB; ++q) {
                uint32_t wt;
                if (t < 16) {
                    wt = w[q][t];
                } else {                                              // batch.py:156-157 circular schedule
                    const uint32_t x = w[q][(t - 3) & 15] ^ w[q][(t - 8) & 15] ^ w[q][(t - 14) & 15] ^ w[q][t & 15];
                    const bool fma_rot = (kV == 2) || (kV == 3 && (t & 1));
                    wt = fma_rot ? rotl_f(x, 1) : rotl(x, 1);
                    w[q][t & 15] = wt;
                }
                uint32_t f, k;
                if (t < 20)      { f = ch(b[q], c[q], d[q]);   k = 0x5A827999u; }   // sha1.py:27-34
                else if (t < 40) { f = xor3(b[q], c[q], d[q]); k = 0x6ED9EBA1u; }
                else if (t < 60) { f = maj(b[q], c[q], d[q]);  k = 0x8F1BBCDCu; }
                else             { f = xor3(b[q], c[q], d[q]); k = 0xCA62C1D6u; }
                uint32_t tmp;                                         // sha1.py:35
                if (kV >= kVarBal) tmp = add_g(f, add_f(e[q], wt + k)) + rotl(a[q], 5);
                else tmp = rotl(a[q], 5) + f + e[q] + k + wt;
                e[q] = d[q]; d[q] = c[q]; c[q] = rotl(b[q], 30); b[q] = a[q]; a[q] = tmp;   // sha1.py:36
            }
        }
#pragma unroll
        for (int q = 0; q < NB; ++q) {                                // sha1.py:37
            s[q][0] += a[q]; s[q][1] += b[q]; s[q][2] += c[q]; s[q][3] += d[q]; s[q][4] += e[q];
        }
    }

    __device__ __forceinline__ static void digest_words(const uint32_t s[5], uint32_t o[5]) {
#pragma unroll
        for (int i = 0; i < 5; ++i) o[i] = bswap(s[i]);               // sha1.py:46 (">5I")
    }
};

// -------------------------------------------------------------------- MD5 --
// K[i] = floor(|sin(i+1)|*2^32) (md5.py:9), S (md5.py:11-16), g (md5.py:38-49).
__host__ __device__ constexpr uint32_t md5_k(int i) {
    constexpr uint32_t K[64] = {
        0xd76aa478, 0xe8c7b756, 0x242070db, 0xc1bdceee, 0xf57c0faf, 0x4787c62a, 0xa8304613, 0xfd469501,
        0x698098d8, 0x8b44f7af, 0xffff5bb1, 0x895cd7be, 0x6b901122, 0xfd987193, 0xa679438e, 0x49b40821,
        0xf61e2562, 0xc040b340, 0x265e5a51, 0xe9b6c7aa, 0xd62f105d, 0x02441453, 0xd8a1e681, 0xe7d3fbc8,
        0x21e1cde6, 0xc33707d6, 0xf4d50d87, 0x455a14ed, 0xa9e3e905, 0xfcefa3f8, 0x676f02d9, 0x8d2a4c8a,
        0xfffa3942, 0x8771f681, 0x6d9d6122, 0xfde5380c, 0xa4beea44, 0x4bdecfa9, 0xf6bb4b60, 0xbebfbc70,
        0x289b7ec6, 0xeaa127fa, 0xd4ef3085, 0x04881d05, 0xd9d4d039, 0xe6db99e5, 0x1fa27cf8, 0xc4ac5665,
        0xf4292244, 0x432aff97, 0xab9423a7, 0xfc93a039, 0x655b59c3, 0x8f0ccc92, 0xffeff47d, 0x85845dd1,
        0x6fa87e4f, 0xfe2ce6e0, 0xa3014314, 0x4e0811a1, 0xf7537e82, 0xbd3af235, 0x2ad7d2bb, 0xeb86d391};
    return K[i];
}
// The same K table in constant memory: an opaque operand keeps ptxas from
// splitting a + M + K into VIADD + IMAD.IADD, so variants 4 / 5 get one
// IADD3 R, R, c[..], R per round for the off-chain sum.
__constant__ uint32_t c_md5k[64] = {
    0xd76aa478, 0xe8c7b756, 0x242070db, 0xc1bdceee, 0xf57c0faf, 0x4787c62a, 0xa8304613, 0xfd469501,
    0x698098d8, 0x8b44f7af, 0xffff5bb1, 0x895cd7be, 0x6b901122, 0xfd987193, 0xa679438e, 0x49b40821,
    0xf61e2562, 0xc040b340, 0x265e5a51, 0xe9b6c7aa, 0xd62f105d, 0x02441453, 0xd8a1e681, 0xe7d3fbc8,
    0x21e1cde6, 0xc33707d6, 0xf4d50d87, 0x455a14ed, 0xa9e3e905, 0xfcefa3f8, 0x676f02d9, 0x8d2a4c8a,
    0xfffa3942, 0x8771f681, 0x6d9d6122, 0xfde5380c, 0xa4beea44, 0x4bdecfa9, 0xf6bb4b60, 0xbebfbc70,
    0x289b7ec6, 0xeaa127fa, 0xd4ef3085, 0x04881d05, 0xd9d4d039, 0xe6db99e5, 0x1fa27cf8, 0xc4ac5665,
    0xf4292244, 0x432aff97, 0xab9423a7, 0xfc93a039, 0x655b59c3, 0x8f0ccc92, 0xffeff47d, 0x85845dd1,
    0x6fa87e4f, 0xfe2ce6e0, 0xa3014314, 0x4e0811a1, 0xf7537e82, 0xbd3af235, 0x2ad7d2bb, 0xeb86d391};
__host__ __device__ constexpr int md5_s(int i) {
    constexpr int S[4][4] = {{7, 12, 17, 22}, {5, 9, 14, 20}, {4, 11, 16, 23}, {6, 10, 15, 21}};
    return S[i / 16][i % 4];
}
__host__ __device__ constexpr int md5_g(int i) {
    return i < 16 ? i : i < 32 ? (5 * i + 1) % 16 : i < 48 ? (3 * i + 5) % 16 : (7 * i) % 16;
}

// Variants: 1 = two of every three rounds add a+M(+K)+F through IMAD/VIADD,
// the third through IADD3 (balances ALU vs FMA issue); 2 = every round via IMAD;
// 3 = as 1 but written so K stays attached to M (3-op dependency chain).
template <int V> struct HashAlg<kMd5, V> {
    static constexpr int kStateWords = 4;
    static constexpr int kDigestBytes = 16;
    static constexpr bool kBigEndian = false;
    static constexpr int kV = V < 0 ? DefaultVariant<kMd5>::value : V;

    __device__ __forceinline__ static void init(uint32_t s[4]) {   // md5.py:6
        s[0] = 0x67452301u; s[1] = 0xEFCDAB89u; s[2] = 0x98BADCFEu; s[3] = 0x10325476u;
    }

    __device__ __forceinline__ static constexpr bool use_fma(int i) {
        return kV == kVarPlain ? false : kV == kVarBal2 ? true : (i % 3) != 2;
    }

    template <int NB>
    __device__ __forceinline__ static void compress_n(uint32_t (&st)[NB][4], const uint32_t (&m)[NB][16]) {
        uint32_t a[NB], b[NB], c[NB], d[NB];
#pragma unroll
        for (int q = 0; q < NB; ++q) { a[q] = st[q][0]; b[q] = st[q][1]; c[q] = st[q][2]; d[q] = st[q][3]; }
#pragma unroll
        for (int i = 0; i < 64; ++i) {                                // md5.py:35-53
#pragma unroll
            for (int q = 0; q < NB; ++q) {
                uint32_t f;
                if (i < 16)      f = ch(b[q], c[q], d[q]);            // (b&c)|(~b&d)
                else if (i < 32) f = ch(d[q], b[q], c[q]);            // (d&b)|(~d&c)
                else if (i < 48) f = xor3(b[q], c[q], d[q]);
                else             f = c[q] ^ (b[q] | ~d[q]);
                const uint32_t mg = m[q][md5_g(i)];
                // t = a + M[g] + K is off the critical path (a is four rounds
                // old); only f -> IMAD -> LEA.HI depends on the previous round.
                // Written so ptxas keeps K attached to M (it sinks immediate adds
                // to the end of an add chain otherwise, lengthening the chain).
                // Variant 1 (B200-measured best, profiles/variant_sweep_r1c.txt):
                // ptxas lowers it to IMAD.IADD(f+a) -> IMAD(x*1+M) -> VIADD(+K),
                // keeping two of the three adds off the ALU pipe.  Variant 3
                // keeps K attached to M (shorter dependency chain, 2 IMADs).
                uint32_t u;
                if (kV == kVarBal3) u = use_fma(i) ? add_g(f, add_f(a[q], mg + md5_k(i))) : add_g(f, a[q] + (mg + md5_k(i)));
                // 4: variant 3's chain; one round in three sums a + M + K in one IADD3 (ALU)
                // 5: every round does (fewest instructions: LOP3, IADD3, IMAD, LEA.HI)
                else if (kV == 4) u = (i % 3) == 2 ? add_g(f, a[q] + mg + c_md5k[i]) : add_g(f, add_f(a[q], mg + md5_k(i)));
                else if (kV == 5) u = add_g(f, a[q] + mg + c_md5k[i]);
                // 6 / 7: as 4 with one round in two / in four through the IADD3
                else if (kV == 6) u = (i % 2) == 1 ? add_g(f, a[q] + mg + c_md5k[i]) : add_g(f, add_f(a[q], mg + md5_k(i)));
                else if (kV == 7) u = (i % 4) == 3 ? add_g(f, a[q] + mg + c_md5k[i]) : add_g(f, add_f(a[q], mg + md5_k(i)));
                else if (use_fma(i)) u = add_f(f, add_f(a[q], mg) + md5_k(i));
                else u = a[q] + f + mg + md5_k(i);
                const uint32_t nb = b[q] + rotl(u, md5_s(i));         // one LEA.HI
                a[q] = d[q]; d[q] = c[q]; c[q] = b[q]; b[q] = nb;
            }
        }
#pragma unroll
        for (int q = 0; q < NB; ++q) {                                // md5.py:54
            st[q][0] += a[q]; st[q][1] += b[q]; st[q][2] += c[q]; st[q][3] += d[q];
        }
    }

    __device__ __forceinline__ static void digest_words(const uint32_t s[4], uint32_t o[4]) {
#pragma unroll
        for (int i = 0; i < 4; ++i) o[i] = s[i];                      // md5.py:63 ("<4I")
    }
};

// -------------------------------------------------------------------- SM3 --
// Variants: 1 = TT1/TT2/SS1 additions through IMAD/VIADD; 2 = 1 + rotl(b,9) and
// rotl(f,19) via IMAD/IMAD.HI; 3 = 1 + only rotl(b,9) via IMAD/IMAD.HI.
template <int V> struct HashAlg<kSm3, V> {
    static constexpr int kStateWords = 8;
    static constexpr int kDigestBytes = 32;
    static constexpr bool kBigEndian = true;
    static constexpr int kV = V < 0 ? DefaultVariant<kSm3>::value : V;

    __device__ __forceinline__ static void init(uint32_t s[8]) {   // sm3.py:5-8
        s[0] = 0x7380166Fu; s[1] = 0x4914B2B9u; s[2] = 0x172442D7u; s[3] = 0xDA8A0600u;
        s[4] = 0xA96F30BCu; s[5] = 0x163138AAu; s[6] = 0xE38DEE4Du; s[7] = 0xB0FB0E4Eu;
    }
    __device__ __forceinline__ static uint32_t p0(uint32_t x) { return xor3(x, rotl(x, 9), rotl(x, 17)); }   // sm3.py:18-19
    __device__ __forceinline__ static uint32_t p1(uint32_t x) { return xor3(x, rotl(x, 15), rotl(x, 23)); }  // sm3.py:22-23
    // T_j pre-rotated by j mod 32 (batch.py:209-214); folds to an immediate.
    __host__ __device__ static constexpr uint32_t tj(int j) {
        return (j % 32) == 0 ? (j < 16 ? 0x79CC4519u : 0x7A879D8Au)
                             : (((j < 16 ? 0x79CC4519u : 0x7A879D8Au) << (j % 32)) |
                                ((j < 16 ? 0x79CC4519u : 0x7A879D8Au) >> (32 - (j % 32))));
    }

    template <int NB>
    __device__ __forceinline__ static void compress_n(uint32_t (&s)[NB][8], const uint32_t (&raw)[NB][16]) {
        // 16-word circular window: round j needs W[j] and W[j+4]; W[j+4] is
        // expanded (sm3.py:35-40) just in time and overwrites W[j-12].
        uint32_t w[NB][16], a[NB], b[NB], c[NB], d[NB], e[NB], f[NB], g[NB], h[NB];
#pragma unroll
        for (int q = 0; q < NB; ++q) {
#pragma unroll
            for (int t = 0; t < 16; ++t) w[q][t] = bswap(raw[q][t]);  // sm3.py:34 (">16I")
            a[q] = s[q][0]; b[q] = s[q][1]; c[q] = s[q][2]; d[q] = s[q][3];
            e[q] = s[q][4]; f[q] = s[q][5]; g[q] = s[q][6]; h[q] = s[q][7];
        }
#pragma unroll
        for (int j = 0; j < 64; ++j) {
#pragma unroll
            for (int q = 0; q < NB; ++q) {
                const int k = j + 4;
                if (k >= 16) {
                    w[q][k & 15] = p1(xor3(w[q][(k - 16) & 15], w[q][(k - 9) & 15], rotl(w[q][(k - 3) & 15], 15)))
                                   ^ rotl(w[q][(k - 13) & 15], 7) ^ w[q][(k - 6) & 15];
                }
                const uint32_t wj = w[q][j & 15];
                const uint32_t wj2 = wj ^ w[q][k & 15];                // W'_j, sm3.py:41
                const uint32_t a12 = rotl(a[q], 12);
                uint32_t ss1;                                          // sm3.py:45
                if (kV >= kVarBal) ss1 = rotl(add_f(a12, e[q]) + tj(j), 7);
                else ss1 = rotl(a12 + e[q] + tj(j), 7);
                const uint32_t ss2 = ss1 ^ a12;                        // sm3.py:46
                uint32_t ff, gg;
                if (j < 16) { ff = xor3(a[q], b[q], c[q]); gg = xor3(e[q], f[q], g[q]); }   // sm3.py:47-52
                else        { ff = maj(a[q], b[q], c[q]);  gg = ch(e[q], f[q], g[q]); }
                uint32_t tt1, tt2;
                if (kV >= kVarBal) {
                    tt1 = add_g(ss2, add_f(ff, d[q]) + wj2);           // sm3.py:53
                    tt2 = add_g(ss1, add_f(gg, h[q]) + wj);            // sm3.py:54
                } else {
                    tt1 = ff + d[q] + ss2 + wj2;
                    tt2 = gg + h[q] + ss1 + wj;
                }
                const bool fb = kV == kVarBal2 || kV == kVarBal3;
                const bool ff19 = kV == kVarBal2;
                d[q] = c[q]; c[q] = fb ? rotl_f(b[q], 9) : rotl(b[q], 9); b[q] = a[q]; a[q] = tt1;       // sm3.py:55-58
                h[q] = g[q]; g[q] = ff19 ? rotl_f(f[q], 19) : rotl(f[q], 19); f[q] = e[q]; e[q] = p0(tt2);  // sm3.py:59-62
            }
        }
#pragma unroll
        for (int q = 0; q < NB; ++q) {                                 // sm3.py:63 (XOR feed-forward)
            s[q][0] ^= a[q]; s[q][1] ^= b[q]; s[q][2] ^= c[q]; s[q][3] ^= d[q];
            s[q][4] ^= e[q]; s[q][5] ^= f[q]; s[q][6] ^= g[q]; s[q][7] ^= h[q];
        }
    }

    __device__ __forceinline__ static void digest_words(const uint32_t s[8], uint32_t o[8]) {
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = bswap(s[i]);               // sm3.py:72 (">8I")
    }
};

// Single-message convenience wrapper.
template <int ALG, int V = -1>
__device__ __forceinline__ void compress1(uint32_t* st, const uint32_t* raw) {
    using H = HashAlg<ALG, V>;
    uint32_t s[1][H::kStateWords];
    uint32_t r[1][16];
#pragma unroll
    for (int i = 0; i < H::kStateWords; ++i) s[0][i] = st[i];
#pragma unroll
    for (int i = 0; i < 16; ++i) r[0][i] = raw[i];
    H::template compress_n<1>(s, r);
#pragma unroll
    for (int i = 0; i < H::kStateWords; ++i) st[i] = s[0][i];
}

// ------------------------------------------------- Merkle-Damgard padding --
// Finish NB messages of the SAME length whose final r (0 <= r < 64) data bytes
// sit in raw[q][] as little-endian words with every byte at position >= r
// already zero.  Appends 0x80, zero fill and the 64-bit bit length exactly as
// _pad does (sha1.py:14-18, md5.py:25-29, sm3.py:26-30; batch.py:133-136),
// compressing one or two blocks.  No dynamic register indexing: the byte
// position is applied through an unrolled select.
template <int ALG, int V, int NB>
__device__ __forceinline__ void md_finish_n(uint32_t (&st)[NB][HashAlg<ALG, V>::kStateWords], uint32_t (&raw)[NB][16],
                                            uint32_t r, uint64_t len_bytes) {
    using H = HashAlg<ALG, V>;
    const uint32_t pad = 0x80u << ((r & 3u) * 8u);
    const uint32_t pw = r >> 2;
    const uint64_t bits = len_bytes * 8ull;
    const uint32_t lo = (uint32_t)bits, hi = (uint32_t)(bits >> 32);
    const uint32_t l14 = H::kBigEndian ? bswap(hi) : lo;
    const uint32_t l15 = H::kBigEndian ? bswap(lo) : hi;
#pragma unroll
    for (int q = 0; q < NB; ++q) {
#pragma unroll
        for (int j = 0; j < 16; ++j) raw[q][j] |= (pw == (uint32_t)j) ? pad : 0u;
    }
    // One compress call site for the 1- or 2-block tail keeps the kernel's
    // instruction footprint small (SM3's unrolled compress is ~1.7k SASS).
    const int ntail = r < 56u ? 1 : 2;
#pragma unroll 1
    for (int k = 0; k < ntail; ++k) {
        if (k == ntail - 1) {
#pragma unroll
            for (int q = 0; q < NB; ++q) {
                if (k == 1) {
#pragma unroll
                    for (int j = 0; j < 14; ++j) raw[q][j] = 0u;
                }
                raw[q][14] = l14;
                raw[q][15] = l15;
            }
        }
        H::template compress_n<NB>(st, raw);
    }
}

template <int ALG, int V = -1>
__device__ __forceinline__ void md_finish(uint32_t* st, uint32_t* raw, uint32_t r, uint64_t len_bytes) {
    using H = HashAlg<ALG, V>;
    uint32_t s[1][H::kStateWords];
    uint32_t w[1][16];
#pragma unroll
    for (int i = 0; i < H::kStateWords; ++i) s[0][i] = st[i];
#pragma unroll
    for (int i = 0; i < 16; ++i) w[0][i] = raw[i];
    md_finish_n<ALG, V, 1>(s, w, r, len_bytes);
#pragma unroll
    for (int i = 0; i < H::kStateWords; ++i) st[i] = s[0][i];
}

// Keep bytes [0, r) of 16 little-endian words, zero the rest.
__device__ __forceinline__ void mask_tail(uint32_t raw[16], uint32_t r) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const uint32_t lo = 4u * j;
        uint32_t m;
        if (r >= lo + 4u) m = 0xFFFFFFFFu;
        else if (r <= lo) m = 0u;
        else m = (1u << ((r - lo) * 8u)) - 1u;
        raw[j] &= m;
    }
}

// Write a digest (kDigestBytes) with 4-byte stores (20-byte SHA-1 rows are
// only 4-byte aligned; MD5/SM3 rows are 16-byte aligned and use vector stores).
template <int ALG>
__device__ __forceinline__ void store_digest(uint8_t* out, const uint32_t* st) {
    using H = HashAlg<ALG>;
    uint32_t o[H::kStateWords];
    H::digest_words(st, o);
    if constexpr (ALG == kSha1) {
        uint32_t* p = reinterpret_cast<uint32_t*>(out);
#pragma unroll
        for (int i = 0; i < 5; ++i) p[i] = o[i];
    } else {
        uint4* p = reinterpret_cast<uint4*>(out);
#pragma unroll
        for (int i = 0; i < H::kStateWords / 4; ++i) p[i] = make_uint4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
    }
}

}  // namespace hb
