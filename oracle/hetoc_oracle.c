/*
 * hetoc_oracle.c -- CPU restatement of the reference hash path.
 *
 * TEST INFRASTRUCTURE ONLY (see hetoc_oracle.h): the checker and the CPU
 * baseline, never the product.  Straight scalar C that follows the reference's
 * scalar modules line by line; no SIMD, no SHA-NI, so that it reads as the
 * reference algorithm.
 */
#include "hetoc_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

static inline uint32_t rotl32(uint32_t x, unsigned n) {
    n &= 31u; /* sm3.py:13-15 reduces the amount mod 32 */
    return n ? (x << n) | (x >> (32u - n)) : x;
}
static inline uint32_t load_be32(const uint8_t *p) {
    return ((uint32_t)p[0] << 24) | ((uint32_t)p[1] << 16) | ((uint32_t)p[2] << 8) | p[3];
}
static inline uint32_t load_le32(const uint8_t *p) {
    return ((uint32_t)p[3] << 24) | ((uint32_t)p[2] << 16) | ((uint32_t)p[1] << 8) | p[0];
}
static inline void store_be32(uint8_t *p, uint32_t v) {
    p[0] = (uint8_t)(v >> 24); p[1] = (uint8_t)(v >> 16); p[2] = (uint8_t)(v >> 8); p[3] = (uint8_t)v;
}
static inline void store_le32(uint8_t *p, uint32_t v) {
    p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); p[2] = (uint8_t)(v >> 16); p[3] = (uint8_t)(v >> 24);
}

/* ---------------------------------------------------------------- SHA-1 -- */
/* _compress, pkg/src/hetoc/crypto/sha1.py:21-37 */
static void sha1_compress(uint32_t st[5], const uint8_t *block) {
    uint32_t w[80];
    for (int t = 0; t < 16; t++) w[t] = load_be32(block + 4 * t); /* sha1.py:22 */
    for (int t = 16; t < 80; t++)                                   /* sha1.py:23-24 */
        w[t] = rotl32(w[t - 3] ^ w[t - 8] ^ w[t - 14] ^ w[t - 16], 1);
    uint32_t a = st[0], b = st[1], c = st[2], d = st[3], e = st[4];
    for (int t = 0; t < 80; t++) { /* sha1.py:26-36 */
        uint32_t f, k;
        if (t < 20) { f = (b & c) | (~b & d); k = 0x5A827999u; }
        else if (t < 40) { f = b ^ c ^ d; k = 0x6ED9EBA1u; }
        else if (t < 60) { f = (b & c) | (b & d) | (c & d); k = 0x8F1BBCDCu; }
        else { f = b ^ c ^ d; k = 0xCA62C1D6u; }
        uint32_t tmp = rotl32(a, 5) + f + e + k + w[t];
        e = d; d = c; c = rotl32(b, 30); b = a; a = tmp;
    }
    st[0] += a; st[1] += b; st[2] += c; st[3] += d; st[4] += e; /* sha1.py:37 */
}

/* ------------------------------------------------------------------ MD5 -- */
/* K[i] = floor(|sin(i+1)| * 2^32), pkg/src/hetoc/crypto/md5.py:9 (tabulated) */
static const uint32_t MD5_K[64] = {
    0xd76aa478, 0xe8c7b756, 0x242070db, 0xc1bdceee, 0xf57c0faf, 0x4787c62a, 0xa8304613, 0xfd469501,
    0x698098d8, 0x8b44f7af, 0xffff5bb1, 0x895cd7be, 0x6b901122, 0xfd987193, 0xa679438e, 0x49b40821,
    0xf61e2562, 0xc040b340, 0x265e5a51, 0xe9b6c7aa, 0xd62f105d, 0x02441453, 0xd8a1e681, 0xe7d3fbc8,
    0x21e1cde6, 0xc33707d6, 0xf4d50d87, 0x455a14ed, 0xa9e3e905, 0xfcefa3f8, 0x676f02d9, 0x8d2a4c8a,
    0xfffa3942, 0x8771f681, 0x6d9d6122, 0xfde5380c, 0xa4beea44, 0x4bdecfa9, 0xf6bb4b60, 0xbebfbc70,
    0x289b7ec6, 0xeaa127fa, 0xd4ef3085, 0x04881d05, 0xd9d4d039, 0xe6db99e5, 0x1fa27cf8, 0xc4ac5665,
    0xf4292244, 0x432aff97, 0xab9423a7, 0xfc93a039, 0x655b59c3, 0x8f0ccc92, 0xffeff47d, 0x85845dd1,
    0x6fa87e4f, 0xfe2ce6e0, 0xa3014314, 0x4e0811a1, 0xf7537e82, 0xbd3af235, 0x2ad7d2bb, 0xeb86d391};
/* S table, pkg/src/hetoc/crypto/md5.py:11-16 */
static const unsigned MD5_S[4][4] = {{7, 12, 17, 22}, {5, 9, 14, 20}, {4, 11, 16, 23}, {6, 10, 15, 21}};

/* _compress, pkg/src/hetoc/crypto/md5.py:32-54 */
static void md5_compress(uint32_t st[4], const uint8_t *block) {
    uint32_t m[16];
    for (int i = 0; i < 16; i++) m[i] = load_le32(block + 4 * i); /* md5.py:33 */
    uint32_t a = st[0], b = st[1], c = st[2], d = st[3];
    for (int i = 0; i < 64; i++) {
        uint32_t f; int g;
        if (i < 16) { f = (b & c) | (~b & d); g = i; }
        else if (i < 32) { f = (d & b) | (~d & c); g = (5 * i + 1) % 16; }
        else if (i < 48) { f = b ^ c ^ d; g = (3 * i + 5) % 16; }
        else { f = c ^ (b | ~d); g = (7 * i) % 16; }
        uint32_t tmp = d;
        d = c;
        c = b;
        uint32_t rot = a + f + MD5_K[i] + m[g];
        b = b + rotl32(rot, MD5_S[i / 16][i % 4]);
        a = tmp;
    }
    st[0] += a; st[1] += b; st[2] += c; st[3] += d; /* md5.py:54 */
}

/* ------------------------------------------------------------------ SM3 -- */
static inline uint32_t sm3_p0(uint32_t x) { return x ^ rotl32(x, 9) ^ rotl32(x, 17); }  /* sm3.py:18-19 */
static inline uint32_t sm3_p1(uint32_t x) { return x ^ rotl32(x, 15) ^ rotl32(x, 23); } /* sm3.py:22-23 */

/* _compress, pkg/src/hetoc/crypto/sm3.py:33-63 */
static void sm3_compress(uint32_t st[8], const uint8_t *block) {
    uint32_t w[68], w2[64];
    for (int j = 0; j < 16; j++) w[j] = load_be32(block + 4 * j); /* sm3.py:34 */
    for (int j = 16; j < 68; j++)                                 /* sm3.py:35-40 */
        w[j] = sm3_p1(w[j - 16] ^ w[j - 9] ^ rotl32(w[j - 3], 15)) ^ rotl32(w[j - 13], 7) ^ w[j - 6];
    for (int j = 0; j < 64; j++) w2[j] = w[j] ^ w[j + 4]; /* sm3.py:41 */
    uint32_t a = st[0], b = st[1], c = st[2], d = st[3], e = st[4], f = st[5], g = st[6], h = st[7];
    for (int j = 0; j < 64; j++) { /* sm3.py:43-62 */
        uint32_t t = j < 16 ? 0x79CC4519u : 0x7A879D8Au;
        uint32_t ss1 = rotl32(rotl32(a, 12) + e + rotl32(t, (unsigned)j), 7);
        uint32_t ss2 = ss1 ^ rotl32(a, 12);
        uint32_t ff, gg;
        if (j < 16) { ff = a ^ b ^ c; gg = e ^ f ^ g; }
        else { ff = (a & b) | (a & c) | (b & c); gg = (e & f) | (~e & g); }
        uint32_t tt1 = ff + d + ss2 + w2[j];
        uint32_t tt2 = gg + h + ss1 + w[j];
        d = c;
        c = rotl32(b, 9);
        b = a;
        a = tt1;
        h = g;
        g = rotl32(f, 19);
        f = e;
        e = sm3_p0(tt2);
    }
    st[0] ^= a; st[1] ^= b; st[2] ^= c; st[3] ^= d; /* sm3.py:63: XOR feed-forward */
    st[4] ^= e; st[5] ^= f; st[6] ^= g; st[7] ^= h;
}

/* ------------------------------------------------- Merkle-Damgard driver -- */
/* _pad (sha1.py:14-18, md5.py:25-29, sm3.py:26-30) + the block loop of
 * sha1()/md5()/sm3() (sha1.py:40-46, md5.py:57-63, sm3.py:66-72).  Full data
 * blocks are compressed straight from the message; the padded tail (1 or 2
 * blocks) is built exactly as _pad builds it: 0x80, zeros to 56 mod 64, then
 * the 64-bit bit length (big-endian for SHA-1/SM3, little-endian for MD5).  */
typedef void (*compress_fn)(uint32_t *, const uint8_t *);

static void md_hash(const uint8_t *msg, uint64_t len, uint32_t *st, compress_fn fn, int len_be) {
    uint64_t nfull = len / 64;
    for (uint64_t b = 0; b < nfull; b++) fn(st, msg + 64 * b);
    uint8_t tail[128];
    uint64_t r = len - 64 * nfull;
    memset(tail, 0, sizeof tail);
    if (r) memcpy(tail, msg + 64 * nfull, (size_t)r);
    tail[r] = 0x80;
    uint64_t tlen = (r + 1 + 8 <= 64) ? 64 : 128; /* (56 - len%64) % 64 zeros */
    uint64_t bitlen = len * 8u;                      /* md5.py:26 masks to 64 bits */
    for (int i = 0; i < 8; i++) {
        int shift = len_be ? 8 * (7 - i) : 8 * i;
        tail[tlen - 8 + i] = (uint8_t)(bitlen >> shift);
    }
    fn(st, tail);
    if (tlen == 128) fn(st, tail + 64);
}

static void sha1_c(uint32_t *s, const uint8_t *b) { sha1_compress(s, b); }
static void md5_c(uint32_t *s, const uint8_t *b) { md5_compress(s, b); }
static void sm3_c(uint32_t *s, const uint8_t *b) { sm3_compress(s, b); }

void orc_sha1(const uint8_t *msg, uint64_t len, uint8_t out[20]) {
    uint32_t st[5] = {0x67452301u, 0xEFCDAB89u, 0x98BADCFEu, 0x10325476u, 0xC3D2E1F0u}; /* sha1.py:5 */
    md_hash(msg, len, st, sha1_c, 1);
    for (int i = 0; i < 5; i++) store_be32(out + 4 * i, st[i]); /* sha1.py:46 */
}

void orc_md5(const uint8_t *msg, uint64_t len, uint8_t out[16]) {
    uint32_t st[4] = {0x67452301u, 0xEFCDAB89u, 0x98BADCFEu, 0x10325476u}; /* md5.py:6 */
    md_hash(msg, len, st, md5_c, 0);
    for (int i = 0; i < 4; i++) store_le32(out + 4 * i, st[i]); /* md5.py:63 */
}

void orc_sm3(const uint8_t *msg, uint64_t len, uint8_t out[32]) {
    uint32_t st[8] = {0x7380166Fu, 0x4914B2B9u, 0x172442D7u, 0xDA8A0600u,
                      0xA96F30BCu, 0x163138AAu, 0xE38DEE4Du, 0xB0FB0E4Eu}; /* sm3.py:5-8 */
    md_hash(msg, len, st, sm3_c, 1);
    for (int i = 0; i < 8; i++) store_be32(out + 4 * i, st[i]); /* sm3.py:72 */
}

int orc_digest_len(int alg) {
    switch (alg) {
    case ORC_SHA1: return 20;
    case ORC_MD5: return 16;
    case ORC_SM3: return 32;
    default: return -1;
    }
}

int orc_digest(int alg, const uint8_t *msg, uint64_t len, uint8_t *out) {
    switch (alg) { /* batch.py:102-109 */
    case ORC_SHA1: orc_sha1(msg, len, out); return 0;
    case ORC_MD5: orc_md5(msg, len, out); return 0;
    case ORC_SM3: orc_sm3(msg, len, out); return 0;
    default: return -1;
    }
}

/* ------------------------------------------------------------- batches -- */
typedef struct {
    int alg;
    const uint8_t *data;
    const uint64_t *offsets; /* NULL => fixed width */
    uint64_t msg_len;
    uint64_t lo, hi;
    uint8_t *out;
} orc_job;

static void *orc_run(void *p) {
    orc_job *j = (orc_job *)p;
    int dlen = orc_digest_len(j->alg);
    for (uint64_t i = j->lo; i < j->hi; i++) {
        const uint8_t *m;
        uint64_t len;
        if (j->offsets) { m = j->data + j->offsets[i]; len = j->offsets[i + 1] - j->offsets[i]; }
        else { m = j->data + i * j->msg_len; len = j->msg_len; }
        orc_digest(j->alg, m, len, j->out + i * (uint64_t)dlen);
    }
    return NULL;
}

static int orc_batch(int alg, const uint8_t *data, const uint64_t *offsets, uint64_t n,
                     uint64_t msg_len, uint8_t *out, int nthreads) {
    if (orc_digest_len(alg) < 0) return -1;
    if (nthreads < 1) return -2;
    if ((uint64_t)nthreads > n) nthreads = n ? (int)n : 1;
    orc_job *jobs = (orc_job *)calloc((size_t)nthreads, sizeof(orc_job));
    pthread_t *tid = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    if (!jobs || !tid) { free(jobs); free(tid); return -3; }
    for (int k = 0; k < nthreads; k++) { /* np.linspace bounds, batch.py:305 */
        jobs[k].alg = alg; jobs[k].data = data; jobs[k].offsets = offsets; jobs[k].msg_len = msg_len;
        jobs[k].lo = (uint64_t)((double)n * k / nthreads);
        jobs[k].hi = (k == nthreads - 1) ? n : (uint64_t)((double)n * (k + 1) / nthreads);
        jobs[k].out = out;
    }
    if (nthreads == 1) orc_run(&jobs[0]);
    else {
        for (int k = 0; k < nthreads; k++) pthread_create(&tid[k], NULL, orc_run, &jobs[k]);
        for (int k = 0; k < nthreads; k++) pthread_join(tid[k], NULL);
    }
    free(jobs); free(tid);
    return 0;
}

int orc_batch_fixed(int alg, const uint8_t *data, uint64_t n, uint64_t msg_len, uint8_t *out, int nthreads) {
    return orc_batch(alg, data, NULL, n, msg_len, out, nthreads);
}

int orc_batch_varlen(int alg, const uint8_t *data, const uint64_t *offsets, uint64_t n, uint8_t *out, int nthreads) {
    return orc_batch(alg, data, offsets, n, 0, out, nthreads);
}

/* ------------------------------------------------------ synthetic data -- */
/* splitmix64 finaliser over the global 64-bit word index; must match
 * hb_fill_random_dev in paper_2407_09333_b200/csrc/hb_kernels.cu.           */
static inline uint64_t mix64(uint64_t seed, uint64_t idx) {
    uint64_t z = (idx + 1u) * 0x9E3779B97F4A7C15ull + seed * 0xD1B54A32D192ED03ull;
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27; z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

void orc_fill_random(uint8_t *buf, uint64_t nbytes, uint64_t seed, uint64_t byte_offset) {
    uint64_t w0 = byte_offset / 8;
    for (uint64_t i = 0; i < nbytes; i += 8) {
        uint64_t v = mix64(seed, w0 + i / 8);
        for (uint64_t k = 0; k < 8 && i + k < nbytes; k++) buf[i + k] = (uint8_t)(v >> (8 * k));
    }
}

/* gen_messages, pkg/src/hetoc/crypto/batch.py:86-99 */
int orc_gen_decimal(uint64_t start, uint64_t count, int width, uint8_t *out) {
    if (width <= 0) return -1;
    for (uint64_t i = 0; i < count; i++) {
        uint64_t v = start + i;
        for (int pos = width - 1; pos >= 0; pos--) {
            out[i * (uint64_t)width + (uint64_t)pos] = (uint8_t)('0' + v % 10);
            v /= 10;
        }
    }
    return 0;
}
