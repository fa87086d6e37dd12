// hb_algos.cuh -- SHA-1 / MD5 / SM3 compression for one message per thread.
//
// Each function keeps the chaining state and the whole message schedule in
// registers (fully unrolled, constant indices only) and compiles to
// LOP3 (boolean functions), SHF.L.W (rotates), IADD3/IMAD (adds) and PRMT
// (byte swaps).  Inputs are the 16 RAW little-endian words of a 64-byte
// block as loaded from memory; the big-endian algorithms byte-swap inside.
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

// x ^ y ^ z as one LOP3 (immLut 0x96); the compiler already fuses these, the
// explicit forms below keep the intent visible in the source.
__device__ __forceinline__ uint32_t xor3(uint32_t x, uint32_t y, uint32_t z) { return x ^ y ^ z; }
__device__ __forceinline__ uint32_t ch(uint32_t x, uint32_t y, uint32_t z) { return z ^ (x & (y ^ z)); }   // 0xCA
__device__ __forceinline__ uint32_t maj(uint32_t x, uint32_t y, uint32_t z) { return (x & y) | (z & (x | y)); } // 0xE8

template <int ALG> struct HashAlg;

// ------------------------------------------------------------------ SHA-1 --
template <> struct HashAlg<kSha1> {
    static constexpr int kStateWords = 5;
    static constexpr int kDigestBytes = 20;
    static constexpr bool kBigEndian = true;

    __device__ __forceinline__ static void init(uint32_t s[5]) {   // sha1.py:5
        s[0] = 0x67452301u; s[1] = 0xEFCDAB89u; s[2] = 0x98BADCFEu; s[3] = 0x10325476u; s[4] = 0xC3D2E1F0u;
    }

    __device__ __forceinline__ static void compress(uint32_t s[5], const uint32_t raw[16]) {
        uint32_t w[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) w[t] = bswap(raw[t]);            // sha1.py:22 (">16I")
        uint32_t a = s[0], b = s[1], c = s[2], d = s[3], e = s[4];
#pragma unroll
        for (int t = 0; t < 80; ++t) {
            uint32_t wt;
            if (t < 16) {
                wt = w[t];
            } else {                                                  // batch.py:156-157 circular schedule
                wt = rotl(w[(t - 3) & 15] ^ w[(t - 8) & 15] ^ w[(t - 14) & 15] ^ w[t & 15], 1);
                w[t & 15] = wt;
            }
            uint32_t f, k;
            if (t < 20)      { f = ch(b, c, d);   k = 0x5A827999u; }    // sha1.py:27-34
            else if (t < 40) { f = xor3(b, c, d); k = 0x6ED9EBA1u; }
            else if (t < 60) { f = maj(b, c, d);  k = 0x8F1BBCDCu; }
            else             { f = xor3(b, c, d); k = 0xCA62C1D6u; }
            const uint32_t tmp = rotl(a, 5) + f + e + k + wt;         // sha1.py:35
            e = d; d = c; c = rotl(b, 30); b = a; a = tmp;             // sha1.py:36
        }
        s[0] += a; s[1] += b; s[2] += c; s[3] += d; s[4] += e;         // sha1.py:37
    }

    __device__ __forceinline__ static void digest_words(const uint32_t s[5], uint32_t o[5]) {
#pragma unroll
        for (int i = 0; i < 5; ++i) o[i] = bswap(s[i]);               // sha1.py:46 (">5I")
    }
};

// -------------------------------------------------------------------- MD5 --
template <> struct HashAlg<kMd5> {
    static constexpr int kStateWords = 4;
    static constexpr int kDigestBytes = 16;
    static constexpr bool kBigEndian = false;

    __device__ __forceinline__ static void init(uint32_t s[4]) {   // md5.py:6
        s[0] = 0x67452301u; s[1] = 0xEFCDAB89u; s[2] = 0x98BADCFEu; s[3] = 0x10325476u;
    }

    // One step of md5.py:36-53: b' = b + rotl(a + f(b,c,d) + K[i] + m[g], S), with
    // the (a,b,c,d) <- (d,b',b,c) rename folded into the macro's argument order.
#define HB_MD5_F(x, y, z) (ch((x), (y), (z)))                  // i<16: (b&c)|(~b&d)
#define HB_MD5_G(x, y, z) (ch((z), (x), (y)))                  // i<32: (d&b)|(~d&c)
#define HB_MD5_H(x, y, z) (xor3((x), (y), (z)))                // i<48
#define HB_MD5_I(x, y, z) ((y) ^ ((x) | ~(z)))                 // i<64: c^(b|~d)
#define HB_MD5_STEP(FN, a, b, c, d, m, k, s) a = (b) + rotl((a) + FN((b), (c), (d)) + (m) + (k), (s))

    __device__ __forceinline__ static void compress(uint32_t st[4], const uint32_t m[16]) {
        uint32_t a = st[0], b = st[1], c = st[2], d = st[3];
        // K[i] = floor(|sin(i+1)|*2^32) (md5.py:9), S (md5.py:11-16), g (md5.py:38-49)
        HB_MD5_STEP(HB_MD5_F, a, b, c, d, m[0], 0xd76aa478u, 7);
        HB_MD5_STEP(HB_MD5_F, d, a, b, c, m[1], 0xe8c7b756u, 12);
        HB_MD5_STEP(HB_MD5_F, c, d, a, b, m[2], 0x242070dbu, 17);
        HB_MD5_STEP(HB_MD5_F, b, c, d, a, m[3], 0xc1bdceeeu, 22);
        HB_MD5_STEP(HB_MD5_F, a, b, c, d, m[4], 0xf57c0fafu, 7);
        HB_MD5_STEP(HB_MD5_F, d, a, b, c, m[5], 0x4787c62au, 12);
        HB_MD5_STEP(HB_MD5_F, c, d, a, b, m[6], 0xa8304613u, 17);
        HB_MD5_STEP(HB_MD5_F, b, c, d, a, m[7], 0xfd469501u, 22);
        HB_MD5_STEP(HB_MD5_F, a, b, c, d, m[8], 0x698098d8u, 7);
        HB_MD5_STEP(HB_MD5_F, d, a, b, c, m[9], 0x8b44f7afu, 12);
        HB_MD5_STEP(HB_MD5_F, c, d, a, b, m[10], 0xffff5bb1u, 17);
        HB_MD5_STEP(HB_MD5_F, b, c, d, a, m[11], 0x895cd7beu, 22);
        HB_MD5_STEP(HB_MD5_F, a, b, c, d, m[12], 0x6b901122u, 7);
        HB_MD5_STEP(HB_MD5_F, d, a, b, c, m[13], 0xfd987193u, 12);
        HB_MD5_STEP(HB_MD5_F, c, d, a, b, m[14], 0xa679438eu, 17);
        HB_MD5_STEP(HB_MD5_F, b, c, d, a, m[15], 0x49b40821u, 22);

        HB_MD5_STEP(HB_MD5_G, a, b, c, d, m[1], 0xf61e2562u, 5);
        HB_MD5_STEP(HB_MD5_G, d, a, b, c, m[6], 0xc040b340u, 9);
        HB_MD5_STEP(HB_MD5_G, c, d, a, b, m[11], 0x265e5a51u, 14);
        HB_MD5_STEP(HB_MD5_G, b, c, d, a, m[0], 0xe9b6c7aau, 20);
        HB_MD5_STEP(HB_MD5_G, a, b, c, d, m[5], 0xd62f105du, 5);
        HB_MD5_STEP(HB_MD5_G, d, a, b, c, m[10], 0x02441453u, 9);
        HB_MD5_STEP(HB_MD5_G, c, d, a, b, m[15], 0xd8a1e681u, 14);
        HB_MD5_STEP(HB_MD5_G, b, c, d, a, m[4], 0xe7d3fbc8u, 20);
        HB_MD5_STEP(HB_MD5_G, a, b, c, d, m[9], 0x21e1cde6u, 5);
        HB_MD5_STEP(HB_MD5_G, d, a, b, c, m[14], 0xc33707d6u, 9);
        HB_MD5_STEP(HB_MD5_G, c, d, a, b, m[3], 0xf4d50d87u, 14);
        HB_MD5_STEP(HB_MD5_G, b, c, d, a, m[8], 0x455a14edu, 20);
        HB_MD5_STEP(HB_MD5_G, a, b, c, d, m[13], 0xa9e3e905u, 5);
        HB_MD5_STEP(HB_MD5_G, d, a, b, c, m[2], 0xfcefa3f8u, 9);
        HB_MD5_STEP(HB_MD5_G, c, d, a, b, m[7], 0x676f02d9u, 14);
        HB_MD5_STEP(HB_MD5_G, b, c, d, a, m[12], 0x8d2a4c8au, 20);

        HB_MD5_STEP(HB_MD5_H, a, b, c, d, m[5], 0xfffa3942u, 4);
        HB_MD5_STEP(HB_MD5_H, d, a, b, c, m[8], 0x8771f681u, 11);
        HB_MD5_STEP(HB_MD5_H, c, d, a, b, m[11], 0x6d9d6122u, 16);
        HB_MD5_STEP(HB_MD5_H, b, c, d, a, m[14], 0xfde5380cu, 23);
        HB_MD5_STEP(HB_MD5_H, a, b, c, d, m[1], 0xa4beea44u, 4);
        HB_MD5_STEP(HB_MD5_H, d, a, b, c, m[4], 0x4bdecfa9u, 11);
        HB_MD5_STEP(HB_MD5_H, c, d, a, b, m[7], 0xf6bb4b60u, 16);
        HB_MD5_STEP(HB_MD5_H, b, c, d, a, m[10], 0xbebfbc70u, 23);
        HB_MD5_STEP(HB_MD5_H, a, b, c, d, m[13], 0x289b7ec6u, 4);
        HB_MD5_STEP(HB_MD5_H, d, a, b, c, m[0], 0xeaa127fau, 11);
        HB_MD5_STEP(HB_MD5_H, c, d, a, b, m[3], 0xd4ef3085u, 16);
        HB_MD5_STEP(HB_MD5_H, b, c, d, a, m[6], 0x04881d05u, 23);
        HB_MD5_STEP(HB_MD5_H, a, b, c, d, m[9], 0xd9d4d039u, 4);
        HB_MD5_STEP(HB_MD5_H, d, a, b, c, m[12], 0xe6db99e5u, 11);
        HB_MD5_STEP(HB_MD5_H, c, d, a, b, m[15], 0x1fa27cf8u, 16);
        HB_MD5_STEP(HB_MD5_H, b, c, d, a, m[2], 0xc4ac5665u, 23);

        HB_MD5_STEP(HB_MD5_I, a, b, c, d, m[0], 0xf4292244u, 6);
        HB_MD5_STEP(HB_MD5_I, d, a, b, c, m[7], 0x432aff97u, 10);
        HB_MD5_STEP(HB_MD5_I, c, d, a, b, m[14], 0xab9423a7u, 15);
        HB_MD5_STEP(HB_MD5_I, b, c, d, a, m[5], 0xfc93a039u, 21);
        HB_MD5_STEP(HB_MD5_I, a, b, c, d, m[12], 0x655b59c3u, 6);
        HB_MD5_STEP(HB_MD5_I, d, a, b, c, m[3], 0x8f0ccc92u, 10);
        HB_MD5_STEP(HB_MD5_I, c, d, a, b, m[10], 0xffeff47du, 15);
        HB_MD5_STEP(HB_MD5_I, b, c, d, a, m[1], 0x85845dd1u, 21);
        HB_MD5_STEP(HB_MD5_I, a, b, c, d, m[8], 0x6fa87e4fu, 6);
        HB_MD5_STEP(HB_MD5_I, d, a, b, c, m[15], 0xfe2ce6e0u, 10);
        HB_MD5_STEP(HB_MD5_I, c, d, a, b, m[6], 0xa3014314u, 15);
        HB_MD5_STEP(HB_MD5_I, b, c, d, a, m[13], 0x4e0811a1u, 21);
        HB_MD5_STEP(HB_MD5_I, a, b, c, d, m[4], 0xf7537e82u, 6);
        HB_MD5_STEP(HB_MD5_I, d, a, b, c, m[11], 0xbd3af235u, 10);
        HB_MD5_STEP(HB_MD5_I, c, d, a, b, m[2], 0x2ad7d2bbu, 15);
        HB_MD5_STEP(HB_MD5_I, b, c, d, a, m[9], 0xeb86d391u, 21);
        st[0] += a; st[1] += b; st[2] += c; st[3] += d;                // md5.py:54
    }
#undef HB_MD5_F
#undef HB_MD5_G
#undef HB_MD5_H
#undef HB_MD5_I
#undef HB_MD5_STEP

    __device__ __forceinline__ static void digest_words(const uint32_t s[4], uint32_t o[4]) {
#pragma unroll
        for (int i = 0; i < 4; ++i) o[i] = s[i];                      // md5.py:63 ("<4I")
    }
};

// -------------------------------------------------------------------- SM3 --
template <> struct HashAlg<kSm3> {
    static constexpr int kStateWords = 8;
    static constexpr int kDigestBytes = 32;
    static constexpr bool kBigEndian = true;

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

    __device__ __forceinline__ static void compress(uint32_t s[8], const uint32_t raw[16]) {
        // 16-word circular window: round j needs W[j] and W[j+4]; W[j+4] is
        // expanded (sm3.py:35-40) just in time and overwrites W[j-12].
        uint32_t w[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) w[t] = bswap(raw[t]);            // sm3.py:34 (">16I")
        uint32_t a = s[0], b = s[1], c = s[2], d = s[3], e = s[4], f = s[5], g = s[6], h = s[7];
#pragma unroll
        for (int j = 0; j < 64; ++j) {
            const int k = j + 4;
            if (k >= 16) {
                w[k & 15] = p1(xor3(w[(k - 16) & 15], w[(k - 9) & 15], rotl(w[(k - 3) & 15], 15)))
                            ^ rotl(w[(k - 13) & 15], 7) ^ w[(k - 6) & 15];
            }
            const uint32_t wj = w[j & 15];
            const uint32_t wj2 = wj ^ w[k & 15];                       // W'_j, sm3.py:41
            const uint32_t a12 = rotl(a, 12);
            const uint32_t ss1 = rotl(a12 + e + tj(j), 7);             // sm3.py:45
            const uint32_t ss2 = ss1 ^ a12;                            // sm3.py:46
            uint32_t ff, gg;
            if (j < 16) { ff = xor3(a, b, c); gg = xor3(e, f, g); }    // sm3.py:47-52
            else        { ff = maj(a, b, c);  gg = ch(e, f, g); }
            const uint32_t tt1 = ff + d + ss2 + wj2;                   // sm3.py:53
            const uint32_t tt2 = gg + h + ss1 + wj;                    // sm3.py:54
            d = c; c = rotl(b, 9); b = a; a = tt1;                     // sm3.py:55-58
            h = g; g = rotl(f, 19); f = e; e = p0(tt2);                // sm3.py:59-62
        }
        s[0] ^= a; s[1] ^= b; s[2] ^= c; s[3] ^= d;                    // sm3.py:63 (XOR feed-forward)
        s[4] ^= e; s[5] ^= f; s[6] ^= g; s[7] ^= h;
    }

    __device__ __forceinline__ static void digest_words(const uint32_t s[8], uint32_t o[8]) {
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = bswap(s[i]);               // sm3.py:72 (">8I")
    }
};

// ------------------------------------------------- Merkle-Damgard padding --
// Finish a message whose final r (0 <= r < 64) data bytes sit in raw[] as
// little-endian words with every byte at position >= r already zero.  Appends
// 0x80, zero fill and the 64-bit bit length exactly as _pad does
// (sha1.py:14-18, md5.py:25-29, sm3.py:26-30; batch.py:133-136), compressing
// one or two blocks.  No dynamic register indexing: the byte position is
// applied through an unrolled select.
template <int ALG>
__device__ __forceinline__ void md_finish(uint32_t st[], uint32_t raw[16], uint32_t r, uint64_t len_bytes) {
    using H = HashAlg<ALG>;
    const uint32_t pad = 0x80u << ((r & 3u) * 8u);
    const uint32_t pw = r >> 2;
#pragma unroll
    for (int j = 0; j < 16; ++j) raw[j] |= (pw == (uint32_t)j) ? pad : 0u;
    const uint64_t bits = len_bytes * 8ull;
    const uint32_t lo = (uint32_t)bits, hi = (uint32_t)(bits >> 32);
    const uint32_t l14 = H::kBigEndian ? bswap(hi) : lo;
    const uint32_t l15 = H::kBigEndian ? bswap(lo) : hi;
    // One compress call site for the 1- or 2-block tail keeps the kernel's
    // instruction footprint small (SM3's unrolled compress is ~1.7k SASS).
    const int ntail = r < 56u ? 1 : 2;
#pragma unroll 1
    for (int k = 0; k < ntail; ++k) {
        if (k == ntail - 1) {
            if (k == 1) {
#pragma unroll
                for (int j = 0; j < 14; ++j) raw[j] = 0u;
            }
            raw[14] = l14;
            raw[15] = l15;
        }
        H::compress(st, raw);
    }
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
__device__ __forceinline__ void store_digest(uint8_t* out, const uint32_t st[]) {
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
