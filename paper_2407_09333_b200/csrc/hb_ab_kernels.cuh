// hb_ab_kernels.cuh -- the A/B arms of the round-1 measurements (compiled only
// with -DHB_AB; included by hb_kernels.cuh inside namespace hb).  None of them
// ships in the default library: each lost to the tuned default in an
// interleaved B200 A/B run recorded under profiles/:
//   k_fixed_tma<..>   per-warp TMA rings (lane 0 issues)   profiles/variant_sweep_r1*.txt
//   k_varlen32        256-bit loads, 8 alignment classes    profiles/ab_varlen_r1g.txt, _r1h.txt
//   k_varlen_bulk     per-lane cp.async.bulk (TMA engine)   profiles/ab_varlen_r1e.txt
//   k_varlen_coop     warp-cooperative cp.async staging     profiles/ab_varlen_r1.txt, _r1b.txt
#pragma once
// Round-2 varlen arms that lost to the shipped kernels (interleaved B200 A/B,
// profiles/r2/): two messages per thread (k_varlen16x2, ab_varlen_r2i.txt),
// the uniform-finish loops with predicated windows for every algorithm
// (k_varlen16u, k_varlen16f; ab_varlen_r2q.txt), the FMA-pipe realignment
// (k_varlen16m, ab_varlen_r2ae.txt) and the two-block carry loop (k_varlen16c,
// ab_varlen_r2ab.txt).  They build on the shipped helpers of hb_kernels.cuh.
// The rest of one message from full block b0 on: full blocks b0 .. len/64-1,
// then the tail and padding (md_finish), digest stored.  `st` holds the state
// after blocks 0 .. b0-1.
template <int ALG, bool EDGE>
__device__ __forceinline__ void varlen16_rest(const uint4* w16, uintptr_t a, uint64_t len, uintptr_t dend,
                                              uint64_t b0, uint32_t* st, uint8_t* dout) {
    const uint32_t q = (uint32_t)(a >> 2) & 3u, sh = (uint32_t)(a & 3u) * 8u;
    const bool misaligned = (a & 15u) != 0;
    uint32_t c[20];
    uint32_t raw[16];
    const uint64_t nfull = len >> 6;
    for (uint64_t b = b0; b < nfull; ++b) {
        load_full_window(w16 + 4 * b, misaligned, c, EDGE, dend);
        realign16(c, q, sh, raw);
        compress1<ALG>(st, raw);
    }
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

// Two messages per thread: sorted neighbours 2t and 2t+1 (same alignment
// class and block count, or adjacent counts, after the q-major windowed
// sort) compress together while both have full blocks left -- two
// independent round chains interleaved in one instruction stream, for the
// dependency stalls that dominate the one-message kernel (ncu: 43 % `wait`).
// Leftover full blocks and the 1-2 finishing blocks run per message.
template <int ALG>
__global__ void __launch_bounds__(128)
k_varlen16x2(const uint8_t* __restrict__ data, const uint8_t* data_end, const uint64_t* __restrict__ offsets,
             uint64_t offset_base, const uint32_t* __restrict__ perm, uint64_t n, uint8_t* __restrict__ out) {
    using H = HashAlg<ALG>;
    const uint64_t k0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2u;
    if (k0 >= n) return;
    const bool two = k0 + 1 < n;
    const uint64_t i0 = perm ? (uint64_t)perm[k0] : k0;
    const uint64_t i1 = two ? (perm ? (uint64_t)perm[k0 + 1] : k0 + 1) : i0;
    const uint64_t len0 = offsets[i0 + 1] - offsets[i0], len1 = offsets[i1 + 1] - offsets[i1];
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(data + (offsets[i0] - offset_base));
    const uintptr_t a1 = reinterpret_cast<uintptr_t>(data + (offsets[i1] - offset_base));
    const uint4* w0 = reinterpret_cast<const uint4*>(a0 & ~uintptr_t(15));
    const uint4* w1 = reinterpret_cast<const uint4*>(a1 & ~uintptr_t(15));
    const uintptr_t dend = reinterpret_cast<uintptr_t>(data_end);
    if (((a0 + len0 + 15u) & ~uintptr_t(15)) > dend || ((a1 + len1 + 15u) & ~uintptr_t(15)) > dend) {
        // a message whose last granule straddles the end of the data: bounded loads, one at a time
        varlen16_message<ALG, 0, true>(w0, a0, len0, dend, out + i0 * H::kDigestBytes);
        if (two) varlen16_message<ALG, 0, true>(w1, a1, len1, dend, out + i1 * H::kDigestBytes);
        return;
    }
    const uint32_t q0 = (uint32_t)(a0 >> 2) & 3u, sh0 = (uint32_t)(a0 & 3u) * 8u;
    const uint32_t q1 = (uint32_t)(a1 >> 2) & 3u, sh1 = (uint32_t)(a1 & 3u) * 8u;
    const bool mis0 = (a0 & 15u) != 0, mis1 = (a1 & 15u) != 0;
    uint32_t st[2][H::kStateWords];
    H::init(st[0]);
    H::init(st[1]);
    const uint64_t nf0 = len0 >> 6, nf1 = len1 >> 6;
    const uint64_t nmin = nf0 < nf1 ? nf0 : nf1;
    uint32_t c0[20], c1[20], raw[2][16];
    for (uint64_t b = 0; b < nmin; ++b) {
        load_full_window(w0 + 4 * b, mis0, c0);
        load_full_window(w1 + 4 * b, mis1, c1);
        realign16(c0, q0, sh0, raw[0]);
        realign16(c1, q1, sh1, raw[1]);
        H::template compress_n<2>(st, raw);
    }
    varlen16_rest<ALG, false>(w0, a0, len0, dend, nmin, st[0], out + i0 * H::kDigestBytes);
    if (two) varlen16_rest<ALG, false>(w1, a1, len1, dend, nmin, st[1], out + i1 * H::kDigestBytes);
}

// -------------------------------------------------------------------------
// Variable-length kernel with a warp-uniform block loop.  After the length
// sort a warp's 32 messages share their block count nb = (len+8)/64 + 1,
// but not whether the final data bytes and the padding need one block or
// two (r = len % 64 >= 56 needs two): k_varlen16 runs the full-block loop to
// len/64 and then md_finish's 1-2 compressions, so a warp with both kinds of
// lanes executes nb + 1 compressions.  Here every lane runs exactly nb:
// blocks 0 .. nb-3 are full data blocks for every lane, and the last two go
// through one branch-free tail body (bytes past the message masked to zero,
// 0x80 where the message ends, the bit length in the last block) -- one
// compress call site per loop, no divergence when nb is warp-uniform.
// V: round variant (1 = the tuned ALU/FMA balance, 2 = every addition on the
// FMA pipe: the realignment's funnel shifts load the ALU pipe here).
// -------------------------------------------------------------------------
template <int ALG, int V, bool EDGE>
__device__ __forceinline__ void varlen16u_message(const uint4* w16, uintptr_t a, uint64_t len, uintptr_t dend,
                                                  uint8_t* dout) {
    using H = HashAlg<ALG, V>;
    const uint32_t q = (uint32_t)(a >> 2) & 3u, sh = (uint32_t)(a & 3u) * 8u;
    const bool misaligned = (a & 15u) != 0;
    uint32_t st[1][H::kStateWords];
    H::init(st[0]);
    uint32_t c[20];
    uint32_t raw[1][16];
    const uint64_t nb = (len + 8u) / 64u + 1u;
    const uint64_t nmain = nb >= 2u ? nb - 2u : 0u;  // every lane: full data blocks
    for (uint64_t b = 0; b < nmain; ++b) {
        load_full_window(w16 + 4 * b, misaligned, c, EDGE, dend);
        realign16(c, q, sh, raw[0]);
        H::template compress_n<1>(st, raw);
    }
    const uint64_t bits = len * 8ull;
    const uint32_t l14 = H::kBigEndian ? bswap((uint32_t)(bits >> 32)) : (uint32_t)bits;
    const uint32_t l15 = H::kBigEndian ? bswap((uint32_t)bits) : (uint32_t)(bits >> 32);
    const uintptr_t mend = a + len;
#pragma unroll 1
    for (uint64_t k = nmain; k < nb; ++k) {
        const uint4* src = w16 + 4 * k;
#pragma unroll
        for (int kk = 0; kk < 5; ++kk) {  // the chunks that overlap the message's bytes of block k
            uint4 v = make_uint4(0, 0, 0, 0);
            if (reinterpret_cast<uintptr_t>(src + kk) < mend) v = ld16_edge(src + kk, EDGE, dend);
            c[4 * kk] = v.x; c[4 * kk + 1] = v.y; c[4 * kk + 2] = v.z; c[4 * kk + 3] = v.w;
        }
        realign16(c, q, sh, raw[0]);
        const int64_t rem = (int64_t)len - 64 * (int64_t)k;  // message bytes from this block's start
        if (rem < 64) {
            const uint32_t r = rem > 0 ? (uint32_t)rem : 0u;
            mask_tail(raw[0], r);
            const uint32_t pad = rem >= 0 ? 0x80u << ((r & 3u) * 8u) : 0u, pw = r >> 2;
#pragma unroll
            for (int j = 0; j < 16; ++j) raw[0][j] |= (pw == (uint32_t)j) ? pad : 0u;
        }
        if (k == nb - 1u) { raw[0][14] = l14; raw[0][15] = l15; }
        H::template compress_n<1>(st, raw);
    }
    store_digest<ALG>(dout, st[0]);
}

template <int ALG, int V>
__global__ void __launch_bounds__(128)
k_varlen16u(const uint8_t* __restrict__ data, const uint8_t* data_end, const uint64_t* __restrict__ offsets,
            uint64_t offset_base, const uint32_t* __restrict__ perm, uint64_t n, uint8_t* __restrict__ out) {
    using H = HashAlg<ALG>;
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint64_t i = perm ? (uint64_t)perm[t] : t;
    const uint64_t start = offsets[i] - offset_base;
    const uint64_t len = offsets[i + 1] - offsets[i];
    const uintptr_t a = reinterpret_cast<uintptr_t>(data + start);
    const uint4* w16 = reinterpret_cast<const uint4*>(a & ~uintptr_t(15));
    const uintptr_t dend = reinterpret_cast<uintptr_t>(data_end);
    if (((a + len + 15u) & ~uintptr_t(15)) > dend)
        varlen16u_message<ALG, V, true>(w16, a, len, dend, out + i * H::kDigestBytes);
    else
        varlen16u_message<ALG, V, false>(w16, a, len, dend, out + i * H::kDigestBytes);
}

// -------------------------------------------------------------------------
// Realignment on the FMA pipe (ALU-bound SHA-1 / SM3).  The funnel shifts of
// realign16 are ALU-pipe ops, 16 per block, on top of an ALU pipe the
// compression already keeps ~95 % busy.  Here the window is based at the
// granule holding byte a-1, so the shift s = 8 * ((a-1) % 4) + 8 lies in
// 8..32 and never is 0, and word j = (c[j+q+1]:c[j+q]) >> s =
// umulhi(c[j+q], m) + c[j+q+1] * m with m = 2^(32-s): one IMAD.HI (with the
// addend) and one IMAD, both FMA-pipe.  The word class q = ((a-1) >> 2) % 4
// must be warp-uniform, so the length sort keys on a-1 (bias shifted by one).
// -------------------------------------------------------------------------
__device__ __forceinline__ void realign16m(const uint32_t (&c)[20], uint32_t q, uint32_t m, uint32_t (&raw)[16]) {
#define HB_RM(Q) \
    _Pragma("unroll") for (int j = 0; j < 16; ++j) raw[j] = __umulhi(c[j + Q], m) + c[j + Q + 1] * m;
    switch (q) {
    case 0: HB_RM(0) break;
    case 1: HB_RM(1) break;
    case 2: HB_RM(2) break;
    default: HB_RM(3) break;
    }
#undef HB_RM
}

template <int ALG>
__global__ void __launch_bounds__(128)
k_varlen16m(const uint8_t* __restrict__ data, const uint8_t* data_end, const uint64_t* __restrict__ offsets,
            uint64_t offset_base, const uint32_t* __restrict__ perm, uint64_t n, uint8_t* __restrict__ out) {
    using H = HashAlg<ALG>;
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint64_t i = perm ? (uint64_t)perm[t] : t;
    const uint64_t start = offsets[i] - offset_base;
    const uint64_t len = offsets[i + 1] - offsets[i];
    const uintptr_t a = reinterpret_cast<uintptr_t>(data + start);
    const uintptr_t dend = reinterpret_cast<uintptr_t>(data_end);
    uint8_t* dout = out + i * H::kDigestBytes;
    const uintptr_t wb = (a - 1u) & ~uintptr_t(15);
    if (wb < reinterpret_cast<uintptr_t>(data) || ((a + len + 15u) & ~uintptr_t(15)) > dend || (len >> 38)) {
        // a message at the very start (its window would begin before the data) or at the end
        varlen16_message<ALG, 0, true>(reinterpret_cast<const uint4*>(a & ~uintptr_t(15)), a, len, dend, dout);
        return;
    }
    const uint4* w = reinterpret_cast<const uint4*>(wb);
    const uint32_t q = (uint32_t)((a - 1u) >> 2) & 3u;
    // m = 2^(32 - s), s = 8 ((a-1) % 4) + 8, read from constant memory: a shift
    // ptxas can see is a power of two would be strength-reduced back to SHF
    const uint32_t m = c_opaque[24u - 8u * ((uint32_t)(a - 1u) & 3u)];
    const uint32_t nfull = (uint32_t)(len >> 6);
    uint32_t st[H::kStateWords];
    H::init(st);
    uint32_t c[20], raw[16];
    for (uint32_t b = 0; b < nfull; ++b) {
        const uint4* src = w + 4 * (uint64_t)b;
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const uint4 v = __ldg(src + k);
            c[4 * k] = v.x; c[4 * k + 1] = v.y; c[4 * k + 2] = v.z; c[4 * k + 3] = v.w;
        }
        realign16m(c, q, m, raw);
        compress1<ALG>(st, raw);
    }
    const uint32_t r = (uint32_t)(len & 63u);
    const uintptr_t tail_end = a + len;
    const uint4* src = w + 4 * (uint64_t)nfull;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const uint4 v = ld16_pred(src + k, reinterpret_cast<uintptr_t>(src + k) < tail_end);
        c[4 * k] = v.x; c[4 * k + 1] = v.y; c[4 * k + 2] = v.z; c[4 * k + 3] = v.w;
    }
    realign16m(c, q, m, raw);
    mask_tail(raw, r);
    md_finish<ALG>(st, raw, r, len);
    store_digest<ALG>(dout, st);
}

// -------------------------------------------------------------------------
// Lean loop unrolled by two with the shared granule carried: window b+1's
// first granule is window b's fifth, so after the first window every block
// loads four granules instead of five (-20 % L1 wavefronts), and the loop
// bookkeeping and the realignment switch's branches are paid once per two
// blocks.  The carry is a register renaming in the unrolled body (cA[16..19]
// becomes cB[0..3] and back), not a copy.  Every window's fifth granule is
// loaded (a 16-byte-aligned message does not use it for its own block), so a
// message whose last granule ends within 16 bytes of the data end takes the
// bounded path.  L2 policies as in k_varlen16l<.., HINT>.
// -------------------------------------------------------------------------
__device__ __forceinline__ void load_granules_1to4(const uint4* src, uint32_t (&c)[20]) {
#pragma unroll
    for (int k = 1; k < 5; ++k) {
        const uint4 v = __ldg(src + k);
        c[4 * k] = v.x; c[4 * k + 1] = v.y; c[4 * k + 2] = v.z; c[4 * k + 3] = v.w;
    }
}

template <int ALG>
__global__ void __launch_bounds__(128)
k_varlen16c(const uint8_t* __restrict__ data, const uint8_t* data_end, const uint64_t* __restrict__ offsets,
            uint64_t offset_base, const uint32_t* __restrict__ perm, uint64_t n, uint8_t* __restrict__ out) {
    using H = HashAlg<ALG>;
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint64_t i = perm ? (uint64_t)perm[t] : t;
    const uint64_t start = offsets[i] - offset_base;
    const uint64_t len = offsets[i + 1] - offsets[i];
    const uintptr_t a = reinterpret_cast<uintptr_t>(data + start);
    const uint4* w16 = reinterpret_cast<const uint4*>(a & ~uintptr_t(15));
    const uintptr_t dend = reinterpret_cast<uintptr_t>(data_end);
    uint8_t* dout = out + i * H::kDigestBytes;
    if (((a + len + 15u) & ~uintptr_t(15)) + 16u > dend || (len >> 38)) {  // near the data end, or > 2^32 blocks
        varlen16_message<ALG, 1, true>(w16, a, len, dend, dout);
        return;
    }
    const uint32_t q = (uint32_t)(a >> 2) & 3u, sh = (uint32_t)(a & 3u) * 8u;
    const uint32_t nfull = (uint32_t)(len >> 6);
    uint32_t st[H::kStateWords];
    H::init(st);
    uint32_t cA[20], cB[20], raw[16];
    if (nfull) load_window5_hint(w16, 1u, cA, policy_evict_last());
    uint32_t b = 0;
    for (; b + 2 <= nfull; b += 2) {
        realign16(cA, q, sh, raw);
        cB[0] = cA[16]; cB[1] = cA[17]; cB[2] = cA[18]; cB[3] = cA[19];
        load_granules_1to4(w16 + 4 * (b + 1), cB);  // block b+1 is full
        compress1<ALG>(st, raw);
        realign16(cB, q, sh, raw);
        if (b + 2 < nfull) {
            cA[0] = cB[16]; cA[1] = cB[17]; cA[2] = cB[18]; cA[3] = cB[19];
            load_granules_1to4(w16 + 4 * (b + 2), cA);
        }
        compress1<ALG>(st, raw);
    }
    if (b < nfull) {  // an odd block count: the last full block's window is in cA
        realign16(cA, q, sh, raw);
        compress1<ALG>(st, raw);
    }
    const uint32_t r = (uint32_t)(len & 63u);
    const uintptr_t tail_end = a + len;
    const uint4* src = w16 + 4 * (uint64_t)nfull;
    uint32_t c[20];
    const uint64_t pol_tail = policy_evict_first();
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const uint4 v = ld16_pred_hint(src + k, reinterpret_cast<uintptr_t>(src + k) < tail_end, pol_tail);
        c[4 * k] = v.x; c[4 * k + 1] = v.y; c[4 * k + 2] = v.z; c[4 * k + 3] = v.w;
    }
    realign16(c, q, sh, raw);
    mask_tail(raw, r);
    md_finish<ALG>(st, raw, r, len);
    store_digest<ALG>(dout, st);
}

// -------------------------------------------------------------------------
// Lean block loop with a uniform finish.  A message of block count nb (data
// + 0x80 + length) needs nb compressions, but k_varlen16(l) runs its full-
// block loop to len/64 and then md_finish's one or two: a lane whose last
// r = len % 64 bytes are >= 56 has one full block fewer and one tail block
// more, so a warp holding both kinds (nearly every warp: P(r >= 56) = 1/8 per
// lane) executes nb + 1 compressions.  Here every lane runs nb - 1 loop
// iterations -- the r >= 56 lanes' partial block, with its 0x80, is the last
// one, masked in place (a branch taken once per message) -- and then one
// final block: the remaining data, 0x80 (r < 56) and the bit length.  The
// window after the last full block is loaded with per-granule predicates
// (never past the message's last granule).
// -------------------------------------------------------------------------
__device__ __forceinline__ void load_window_tail(const uint4* src, uintptr_t tail_end, uint32_t (&c)[20]) {
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const uint4 v = ld16_pred(src + k, reinterpret_cast<uintptr_t>(src + k) < tail_end);
        c[4 * k] = v.x; c[4 * k + 1] = v.y; c[4 * k + 2] = v.z; c[4 * k + 3] = v.w;
    }
}

template <int ALG>
__global__ void __launch_bounds__(128)
k_varlen16f(const uint8_t* __restrict__ data, const uint8_t* data_end, const uint64_t* __restrict__ offsets,
            uint64_t offset_base, const uint32_t* __restrict__ perm, uint64_t n, uint8_t* __restrict__ out) {
    using H = HashAlg<ALG>;
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint64_t i = perm ? (uint64_t)perm[t] : t;
    const uint64_t start = offsets[i] - offset_base;
    const uint64_t len = offsets[i + 1] - offsets[i];
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
    const uint32_t nfull = (uint32_t)(len >> 6), r = (uint32_t)(len & 63u);
    const uint32_t nmain = nfull + (r >= 56u ? 1u : 0u);  // every block but the final one
    const uint32_t pad = 0x80u << ((r & 3u) * 8u), pw = r >> 2;
    const uintptr_t tail_end = a + len;
    uint32_t st[H::kStateWords];
    H::init(st);
    uint32_t c[20], raw[16];
    if (nfull) load_window5(w16, mis, c);
    else load_window_tail(w16, tail_end, c);
    for (uint32_t b = 0; b < nmain; ++b) {
        realign16(c, q, sh, raw);
        if (b + 1 < nfull) load_window5(w16 + 4 * (b + 1), mis, c);
        else load_window_tail(w16 + 4 * (b + 1), tail_end, c);
        if (b == nfull) {  // r >= 56: the partial data block carries the 0x80
            mask_tail(raw, r);
#pragma unroll
            for (int j = 0; j < 16; ++j) raw[j] |= (pw == (uint32_t)j) ? pad : 0u;
        }
        compress1<ALG>(st, raw);
    }
    // final block: r < 56 -> the last r data bytes, 0x80 and the length; r >= 56 -> zeros and the length
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

template <int ALG, int V, int NB, int STAGES, int W = kTmaWarps>
__global__ void __launch_bounds__(W * 32, (TmaOcc<ALG, NB, STAGES, W>::kMinCtas))
k_fixed_tma(const __grid_constant__ CUtensorMap tmap, uint32_t n, uint32_t msg_len, uint8_t* __restrict__ out) {
    using H = HashAlg<ALG, V>;
    using C = TmaCfg<NB, STAGES, W>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t row0 = (blockIdx.x * W + warp) * C::kRows;
    if (row0 >= n) return;  // warp-uniform

    // 1024-align the ring (the swizzle pattern is a function of address bits 7:8).
    const uint32_t base_s = smem_u32(smem_raw);
    uint8_t* ring = smem_raw + (((base_s + 1023u) & ~1023u) - base_s);
    uint8_t* wring = ring + warp * (STAGES * C::kStageBytes);
    uint64_t* bars = reinterpret_cast<uint64_t*>(ring + W * STAGES * C::kStageBytes) + warp * STAGES;

    const uint32_t nload = (msg_len + 63u) >> 6;  // blocks holding message bytes
    if (lane == 0) {
        prefetch_tmap(&tmap);
#pragma unroll
        for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
        const uint32_t pro = nload < (uint32_t)STAGES ? nload : (uint32_t)STAGES;
        for (uint32_t b = 0; b < pro; ++b) {
            mbar_arrive_expect_tx(&bars[b], C::kStageBytes);
            tma_load_2d(wring + b * C::kStageBytes, &tmap, &bars[b], (int)(b * 64u), (int)row0);
        }
    }
    __syncwarp();

    uint32_t st[NB][H::kStateWords];
#pragma unroll
    for (int q = 0; q < NB; ++q) H::init(st[q]);
    // SWIZZLE_64B: the 16-byte chunk index is XORed with address bits 7:8, i.e.
    // (row >> 1) & 3; rows lane and lane+32q share it.
    const uint32_t swz = (lane >> 1) & 3u;
    uint32_t stage = 0, phase = 0;
    uint32_t raw[NB][16];
    // Shared-memory byte offsets of this lane's four 16-byte chunks in stage 0;
    // a stage adds a warp-uniform base, so each read is LDS.128 [R + UR].
    uint32_t choff[NB][4];
#pragma unroll
    for (int q = 0; q < NB; ++q)
#pragma unroll
        for (uint32_t c = 0; c < 4; ++c) choff[q][c] = smem_u32(wring) + (lane + 32u * q) * 64u + ((c ^ swz) << 4);
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
    for (uint32_t b = 0; b < nfull; ++b) {
        mbar_wait_parity(&bars[stage], phase);
        read_stage(stage);
        H::template compress_n<NB>(st, raw);
        __syncwarp();  // every lane has consumed this stage (its registers fed compress)
        if (lane == 0 && b + STAGES < nload) {
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&bars[stage], C::kStageBytes);
            tma_load_2d(wring + stage * C::kStageBytes, &tmap, &bars[stage], (int)((b + STAGES) * 64u), (int)row0);
        }
        if (++stage == (uint32_t)STAGES) { stage = 0; phase ^= 1u; }
    }
    const uint32_t r = msg_len & 63u;
    if (r) {  // partial data block: TMA zero-filled the columns >= msg_len
        mbar_wait_parity(&bars[stage], phase);
        read_stage(stage);
    } else {  // padding-only final block (0x80, zeros, length)
#pragma unroll
        for (int q = 0; q < NB; ++q)
#pragma unroll
            for (int j = 0; j < 16; ++j) raw[q][j] = 0u;
    }
    md_finish_n<ALG, V, NB>(st, raw, r, msg_len);
#pragma unroll
    for (int q = 0; q < NB; ++q) {
        const uint32_t row = row0 + lane + 32u * q;
        if (row < n) store_digest<ALG>(out + (uint64_t)row * H::kDigestBytes, st[q]);
    }
}

// -------------------------------------------------------------------------
// Variable-length kernel, 256-bit loads (LDG.E.ENL2.256, sm_100).
//
// The 16-byte kernel is bound by the L1 data pipe: each LDG.128 of a warp
// touches 32 scattered lines (one wavefront each), 4-5 per block.  A 256-bit
// load moves the same line traffic in half the instructions, so each block
// costs 2-3 wavefronts per lane instead of 4-5.  The message's 32-aligned
// 96-byte window around block b is realigned by a word select over
// q = (address >> 2) mod 8 (warp-uniform: the sort key uses 8 alignment
// classes) and one funnel shift.  Loads never cross `data_end`: a chunk that
// would (only possible for the batch's last message) is read word by word.
// -------------------------------------------------------------------------
__device__ __forceinline__ void ld256_nc(const uint32_t* p, uint32_t* w) {
    asm volatile("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                 : "l"(p));
}

// 32-byte chunk at p (32-aligned): bytes < lim are read, the rest are zero
// (lim = min(message end, data_end) is only binding in the tail; full blocks
// pass lim = data_end).
__device__ __forceinline__ void load_chunk32(const uint8_t* p, uintptr_t lim, uint32_t* w) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    if (a + 32u <= lim) {
        ld256_nc(reinterpret_cast<const uint32_t*>(p), w);
    } else {
#pragma unroll
        for (int k = 0; k < 8; ++k)
            w[k] = (a + 4u * k < lim) ? __ldg(reinterpret_cast<const uint32_t*>(p) + k) : 0u;
    }
}

__device__ __forceinline__ void realign32(const uint32_t (&c)[24], uint32_t q, uint32_t sh, uint32_t (&raw)[16]) {
#define HB_RA(Q)                                                                    \
    _Pragma("unroll") for (int j = 0; j < 16; ++j) raw[j] = __funnelshift_r(c[j + Q], c[j + Q + 1], sh);
    switch (q) {
    case 0: HB_RA(0) break;
    case 1: HB_RA(1) break;
    case 2: HB_RA(2) break;
    case 3: HB_RA(3) break;
    case 4: HB_RA(4) break;
    case 5: HB_RA(5) break;
    case 6: HB_RA(6) break;
    default: HB_RA(7) break;
    }
#undef HB_RA
}

template <int ALG, int PF = 0>
__global__ void __launch_bounds__(128)
k_varlen32(const uint8_t* __restrict__ data, const uint8_t* data_end, const uint64_t* __restrict__ offsets,
           uint64_t offset_base, const uint32_t* __restrict__ perm, uint64_t n, uint8_t* __restrict__ out) {
    using H = HashAlg<ALG>;
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint64_t i = perm ? (uint64_t)perm[t] : t;
    const uint64_t start = offsets[i] - offset_base;
    const uint64_t len = offsets[i + 1] - offsets[i];
    const uintptr_t a = reinterpret_cast<uintptr_t>(data + start);
    const uint8_t* w32 = reinterpret_cast<const uint8_t*>(a & ~uintptr_t(31));
    const uint32_t q = (uint32_t)(a >> 2) & 7u, sh = (uint32_t)(a & 3u) * 8u;
    const bool misaligned = (a & 31u) != 0;
    const uintptr_t dend = reinterpret_cast<uintptr_t>(data_end);
    uint32_t st[H::kStateWords];
    H::init(st);
    uint32_t c[24];
    uint32_t raw[16];
    const uint64_t nfull = len >> 6;
    auto load_win = [&](uint64_t b) {
        const uint8_t* src = w32 + 64 * b;
        load_chunk32(src, dend, c);
        load_chunk32(src + 32, dend, c + 8);
        if (misaligned) {
            load_chunk32(src + 64, dend, c + 16);
        } else {
#pragma unroll
            for (int k = 16; k < 24; ++k) c[k] = 0u;
        }
    };
    if (PF) {  // software pipelining: block b+1's window loads in flight during b's compression
        if (nfull) load_win(0);
        for (uint64_t b = 0; b < nfull; ++b) {
            realign32(c, q, sh, raw);
            if (b + 1 < nfull) load_win(b + 1);
            compress1<ALG>(st, raw);
        }
    } else {
        for (uint64_t b = 0; b < nfull; ++b) {
            load_win(b);
            realign32(c, q, sh, raw);
            compress1<ALG>(st, raw);
        }
    }
    // tail: the r = len % 64 remaining bytes (chunks overlapping [p, p + r) only)
    const uint32_t r = (uint32_t)(len & 63u);
    const uintptr_t mend = a + len;
    const uintptr_t lim = mend < dend ? mend : dend;
    const uint8_t* src = w32 + 64 * nfull;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        if (reinterpret_cast<uintptr_t>(src + 32 * k) < mend) {
            load_chunk32(src + 32 * k, lim, c + 8 * k);
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) c[8 * k + j] = 0u;
        }
    }
    realign32(c, q, sh, raw);
    mask_tail(raw, r);
    md_finish<ALG>(st, raw, r, len);
    store_digest<ALG>(out + i * H::kDigestBytes, st);
}

// -------------------------------------------------------------------------
// Variable-length kernel, per-lane bulk copies (TMA engine).
//
// The per-thread kernel is bound by the L1 data pipe (ncu: LSU wavefronts at
// 85 % of peak): every LDG.128 of a warp touches 32 scattered lines.  Here
// each lane asks the TMA engine for its own message's 16-aligned window of
// block b (<= 80 bytes, clipped at the message's last 16-byte chunk) with one
// cp.async.bulk into its slot of a per-warp STAGES-deep ring; completion is
// counted on the stage's mbarrier (32 arrivals + tx bytes).  Lanes then read
// their slot with LDS.128 (conflict-free at an 80-byte stride), realign,
// apply padding in registers and compress.  Opt-in ($HB_VARLEN_BULK): on the
// B200 the TMA engine does not keep up with 32 tiny (<= 80 B) copies per warp
// step -- 3.9-4.2 vs 2.06 ms for MD5 at configs[3] (profiles/ab_varlen_r1e.txt).
// -------------------------------------------------------------------------
template <int ALG, int STAGES, int MINB = 1>
__global__ void __launch_bounds__(128, MINB)
k_varlen_bulk(const uint8_t* __restrict__ data, const uint64_t* __restrict__ offsets, uint64_t offset_base,
              const uint32_t* __restrict__ perm, uint64_t n, uint8_t* __restrict__ out) {
    using H = HashAlg<ALG>;
    constexpr int kWarps = 4, kSlot = 80, kStage = 32 * kSlot;
    __shared__ __align__(128) uint8_t ring[kWarps][STAGES][kStage];
    __shared__ __align__(8) uint64_t bars[kWarps][STAGES];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t wbase = ((uint64_t)blockIdx.x * kWarps + warp) * 32u;
    if (wbase >= n) return;  // warp-uniform
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < STAGES; ++k) mbar_init(&bars[warp][k], 32);
        fence_mbar_init();
    }
    __syncwarp();
    const uint64_t t = wbase + lane;
    const bool live = t < n;
    uint64_t i = 0, len = 0;
    uintptr_t a = reinterpret_cast<uintptr_t>(data);
    if (live) {
        i = perm ? (uint64_t)perm[t] : t;
        a = reinterpret_cast<uintptr_t>(data + (offsets[i] - offset_base));
        len = offsets[i + 1] - offsets[i];
    }
    const uint32_t nb = live ? (uint32_t)((len + 8u) / 64u + 1u) : 0u;  // blocks incl. padding
    const uint32_t nfull = (uint32_t)(len >> 6);
    const uint32_t nbmax = __reduce_max_sync(0xFFFFFFFFu, nb);
    const uintptr_t w16 = a & ~uintptr_t(15);
    const uintptr_t end16 = (a + len + 15u) & ~uintptr_t(15);  // message bytes live in [w16, end16)
    const uint32_t slot = smem_u32(&ring[warp][0][0]) + lane * kSlot;
    auto issue = [&](uint32_t b) {
        const uint32_t s = b % STAGES;
        const uintptr_t ws = w16 + 64u * (uintptr_t)b;
        // only blocks holding message bytes are fetched (b <= nfull); at most 80 bytes
        const uint32_t bytes = (b > nfull || ws >= end16) ? 0u
                               : (end16 - ws >= 80u ? 80u : (uint32_t)(end16 - ws));
        mbar_arrive_expect_tx(&bars[warp][s], bytes);
        if (bytes) bulk_copy_g2s(slot + s * kStage, reinterpret_cast<const void*>(ws), bytes, &bars[warp][s]);
    };
#pragma unroll
    for (int k = 0; k < STAGES - 1; ++k)
        if ((uint32_t)k < nbmax) issue(k);

    const uint32_t q = (uint32_t)(a >> 2) & 3u, sh = (uint32_t)(a & 3u) * 8u;
    const uint32_t r = (uint32_t)(len & 63u);
    const uint64_t bits = len * 8ull;
    const uint32_t l14 = H::kBigEndian ? bswap((uint32_t)(bits >> 32)) : (uint32_t)bits;
    const uint32_t l15 = H::kBigEndian ? bswap((uint32_t)bits) : (uint32_t)(bits >> 32);
    uint32_t st[H::kStateWords];
    H::init(st);
    for (uint32_t b = 0; b < nbmax; ++b) {
        if (b + STAGES - 1 < nbmax) {
            fence_proxy_async_smem();  // this lane's generic reads of the stage happened before (syncwarp below)
            issue(b + STAGES - 1);
        }
        const uint32_t s = b % STAGES;
        mbar_wait_parity(&bars[warp][s], (b / STAGES) & 1u);
        uint32_t c[20];
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            uint32_t x, y, z, w;
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(x), "=r"(y), "=r"(z), "=r"(w)
                         : "r"(slot + s * kStage + 16u * k)
                         : "memory");
            c[4 * k] = x; c[4 * k + 1] = y; c[4 * k + 2] = z; c[4 * k + 3] = w;
        }
        __syncwarp();  // every lane has read stage s before it is refilled
        if (b < nb) {
            uint32_t raw[16];
            realign16(c, q, sh, raw);
            if (b >= nfull) {  // the last one or two blocks: keep bytes [0, r) (none after), 0x80, length
                mask_tail(raw, b == nfull ? r : 0u);
                const uint32_t pad = b == nfull ? 0x80u << ((r & 3u) * 8u) : 0u, pw = r >> 2;
#pragma unroll
                for (int j = 0; j < 16; ++j) raw[j] |= (pw == (uint32_t)j) ? pad : 0u;
                if (b == nb - 1u) { raw[14] = l14; raw[15] = l15; }
            }
            compress1<ALG>(st, raw);
        }
    }
    if (live) store_digest<ALG>(out + i * H::kDigestBytes, st);
}

// -------------------------------------------------------------------------
// Variable-length kernel, warp-cooperative staging (the default).
//
// A warp owns 32 messages (after the length sort: equal block counts and the
// same word alignment).  Per 64-byte step every message needs the 80-byte
// 16-aligned window around its block: 32 x 5 = 160 16-byte chunks.  Lane l
// copies chunks c = l + 32j (j < 5) -- message c/5, chunk c%5 -- with
// cp.async (zero-filled past the message end), so five consecutive lanes
// fetch one message's 80 contiguous bytes: each warp instruction touches ~7
// messages instead of 32 (per-thread LDG.128 touches 32 lines per
// instruction and the L1 tag stage, not HBM, was the limit for MD5).  Chunks
// land in a STAGES-deep per-warp ring (slot m at m*80: conflict-free
// LDS.128 reads); the owner lane realigns its window (word select + funnel
// shift) and compresses.  Padding is applied in registers on the last one
// or two blocks (bytes past the end arrive as zeros), so there is one
// compress call site and the loop runs to the warp's largest block count.
// -------------------------------------------------------------------------
constexpr int kVcWarps = 4;
constexpr int kVcSlot = 80;                   // bytes per message per stage
constexpr int kVcWarpStage = 32 * kVcSlot;    // 2,560 bytes

// STAGES-deep ring (smem 10 KiB per stage per CTA), MINB CTAs/SM register
// target, PF = L2 prefetch size of the cp.async copies.
template <int ALG, int STAGES = 4, int MINB = 5, int PF = 256>
__global__ void __launch_bounds__(kVcWarps * 32, MINB)
k_varlen_coop(const uint8_t* __restrict__ data, const uint64_t* __restrict__ offsets, uint64_t offset_base,
              const uint32_t* __restrict__ perm, uint64_t n, uint8_t* __restrict__ out) {
    using H = HashAlg<ALG>;
    __shared__ __align__(128) uint8_t ring[kVcWarps][STAGES][kVcWarpStage];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t wbase = ((uint64_t)blockIdx.x * kVcWarps + warp) * 32u;
    if (wbase >= n) return;  // warp-uniform
    const uint64_t t = wbase + lane;
    const bool live = t < n;
    uint64_t i = 0, len = 0;
    uintptr_t a = reinterpret_cast<uintptr_t>(data);
    if (live) {
        i = perm ? (uint64_t)perm[t] : t;
        a = reinterpret_cast<uintptr_t>(data + (offsets[i] - offset_base));
        len = offsets[i + 1] - offsets[i];
    }
    const uint32_t nb = live ? (uint32_t)((len + 8u) / 64u + 1u) : 0u;   // blocks incl. padding
    const uint32_t nfull = (uint32_t)(len >> 6);
    const uint32_t nbmax = __reduce_max_sync(0xFFFFFFFFu, nb);

    // This lane's five copy slots: source message m = c/5, chunk k = c%5.
    uintptr_t src0[5];
    int64_t avail0[5];  // bytes of the chunk inside the message at step 0 (minus 64 per step)
#pragma unroll
    for (int j = 0; j < 5; ++j) {
        const uint32_t c = lane + 32u * j, m = c / 5u, k = c % 5u;
        const uintptr_t am = __shfl_sync(0xFFFFFFFFu, a, m);
        const uint64_t lm = __shfl_sync(0xFFFFFFFFu, len, m);
        src0[j] = (am & ~uintptr_t(15)) + 16u * k;
        const bool need = (k < 4u) || (am & 15u);  // chunk 4 only for a misaligned window
        avail0[j] = (need && lm) ? (int64_t)lm + (int64_t)(am & 15u) - 16 * (int64_t)k : INT64_MIN / 2;
    }
    uint8_t* wring = &ring[warp][0][0];
    const uint32_t sring = smem_u32(wring);
    auto issue = [&](uint32_t b) {
        const uint32_t sdst = sring + (b % STAGES) * kVcWarpStage;
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            const int64_t av = avail0[j] - 64 * (int64_t)b;
            const uint32_t sz = av <= 0 ? 0u : av >= 16 ? 16u : (uint32_t)av;
            const uintptr_t src = sz ? src0[j] + 64u * (uintptr_t)b : reinterpret_cast<uintptr_t>(data);
            cp_async16_zfill<PF>(sdst + 16u * (lane + 32u * j), reinterpret_cast<const void*>(src), sz);
        }
    };
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if ((uint32_t)s < nbmax) issue(s);
        cp_async_commit();
    }

    const uint32_t q = (uint32_t)(a >> 2) & 3u, sh = (uint32_t)(a & 3u) * 8u;
    const uint32_t r = (uint32_t)(len & 63u);
    const uint64_t bits = len * 8ull;
    const uint32_t l14 = H::kBigEndian ? bswap((uint32_t)(bits >> 32)) : (uint32_t)bits;
    const uint32_t l15 = H::kBigEndian ? bswap((uint32_t)bits) : (uint32_t)(bits >> 32);
    uint32_t st[H::kStateWords];
    H::init(st);
    const uint32_t slot = smem_u32(wring) + lane * kVcSlot;
    for (uint32_t b = 0; b < nbmax; ++b) {
        if (b + STAGES - 1 < nbmax) issue(b + STAGES - 1);
        cp_async_commit();
        cp_async_wait<STAGES - 1>();  // this lane's copies of step b have landed
        __syncwarp();                    // ... and every other lane's
        uint32_t c[20];
        const uint32_t sbase = slot + (b % STAGES) * kVcWarpStage;
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            uint32_t x, y, z, w;
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(x), "=r"(y), "=r"(z), "=r"(w)
                         : "r"(sbase + 16u * k)
                         : "memory");
            c[4 * k] = x; c[4 * k + 1] = y; c[4 * k + 2] = z; c[4 * k + 3] = w;
        }
        __syncwarp();  // the stage may be refilled from the next iteration on
        if (b < nb) {
            uint32_t raw[16];
            realign16(c, q, sh, raw);
            if (b >= nfull) {  // the final one or two blocks: 0x80, zero fill, bit length
                if (b == nfull) {
                    const uint32_t pad = 0x80u << ((r & 3u) * 8u), pw = r >> 2;
#pragma unroll
                    for (int j = 0; j < 16; ++j) raw[j] |= (pw == (uint32_t)j) ? pad : 0u;
                }
                if (b == nb - 1u) { raw[14] = l14; raw[15] = l15; }
            }
            compress1<ALG>(st, raw);
        }
    }
    if (live) store_digest<ALG>(out + i * H::kDigestBytes, st);
}

// =========================================================================
// A/B launchers (-DHB_AB only): every arm of profiles/ab_*_r1*.txt and
// profiles/variant_sweep_r1*.txt, selected through the Tuning A/B fields.
// =========================================================================
enum TmaCfgId { kCfg1x3 = 0, kCfg2x2 = 1, kCfg2x3 = 2, kCfgWs2 = 3, kCfgWs3 = 4, kCfg1x2 = 5, kCfgWs2x2 = 6,
                kCfgWs3x2 = 7, kCfgWs3u = 8, kCfgWs3x2u = 9, kCfgWs3n = 10,
                // single-warp CTAs (per-warp ring, W = 1) with NB messages per thread: a
                // mid-size batch (2^16 messages, 3.46 warps per scheduler at NB = 1) as
                // <= 1 warp per scheduler carrying NB independent round chains
                kCfgW1x1 = 11, kCfgW1x2 = 12, kCfgW1x4 = 13, kCfgW1x4s2 = 14, kCfgW1x2p = 15, kCfgWs3v6 = 16, kCfgW1x2s4 = 17,
                kCfgW1x2s2 = 18, kCfgW1x3 = 19, kCfgW1x4p = 20 };

template <int ALG, int V, int NB, int STAGES, int W = kTmaWarps>
static cudaError_t launch_fixed_tma_alg(const uint8_t* d_msgs, uint32_t n, uint32_t L, uint8_t* d_out,
                                        cudaStream_t stream) {
    using C = TmaCfg<NB, STAGES, W>;
    CUtensorMap map;
    cudaError_t e = encode_rows_map(&map, d_msgs, n, L, (uint32_t)C::kRows, 256);
    if (e != cudaSuccess) return e;
    static std::atomic<uint64_t> attr_done{0};
    e = set_smem_attr_once(attr_done, [] {
        return cudaFuncSetAttribute(k_fixed_tma<ALG, V, NB, STAGES, W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    C::kSmem);
    });
    if (e != cudaSuccess) return e;
    const uint32_t rows_per_cta = W * C::kRows;
    note_launch(reinterpret_cast<const void*>(k_fixed_tma<ALG, V, NB, STAGES, W>), true);
    k_fixed_tma<ALG, V, NB, STAGES, W><<<(n + rows_per_cta - 1) / rows_per_cta, W * 32, C::kSmem, stream>>>(
        map, n, L, d_out);
    return cudaGetLastError();
}

template <int ALG>
static cudaError_t launch_tma_ab(const uint8_t* src, uint32_t n, uint32_t L, uint8_t* dst, cudaStream_t s) {
    const int cfg = tuning().tma_cfg >= 0 ? tuning().tma_cfg : (ALG == kSha1 ? kCfgWs3x2 : kCfgWs3);
    const int v = tuning().variant >= 0 ? tuning().variant : kVarBal;
    switch (cfg) {
    case kCfg1x2: return v == 0 ? launch_fixed_tma_alg<ALG, 0, 1, 2>(src, n, L, dst, s)
                                : launch_fixed_tma_alg<ALG, 1, 1, 2>(src, n, L, dst, s);
    case kCfgWs2: return v == 0 ? launch_fixed_tma_ws<ALG, 0, 1, 2>(src, n, L, dst, s)
                                : launch_fixed_tma_ws<ALG, 1, 1, 2>(src, n, L, dst, s);
    case kCfgWs3:
        if constexpr (ALG == kMd5) {
            if (v == 4) return launch_fixed_tma_ws<ALG, 4, 1, 3>(src, n, L, dst, s);
            if (v == 5) return launch_fixed_tma_ws<ALG, 5, 1, 3>(src, n, L, dst, s);
            if (v == 6) return launch_fixed_tma_ws<ALG, 6, 1, 3>(src, n, L, dst, s);
            if (v == 7) return launch_fixed_tma_ws<ALG, 7, 1, 3>(src, n, L, dst, s);
        }
        switch (v) {
        case 0: return launch_fixed_tma_ws<ALG, 0, 1, 3>(src, n, L, dst, s);
        case 2: return launch_fixed_tma_ws<ALG, 2, 1, 3>(src, n, L, dst, s);
        case 3: return launch_fixed_tma_ws<ALG, 3, 1, 3>(src, n, L, dst, s);
        default: return launch_fixed_tma_ws<ALG, 1, 1, 3>(src, n, L, dst, s);
        }
    case kCfgW1x1: return v == 3 ? launch_fixed_tma_alg<ALG, 3, 1, 3, 1>(src, n, L, dst, s)
                                 : launch_fixed_tma_alg<ALG, 1, 1, 3, 1>(src, n, L, dst, s);
    case kCfgW1x2:
        if constexpr (ALG == kMd5)
            if (v == 4) return launch_fixed_tma_alg<ALG, 4, 2, 3, 1>(src, n, L, dst, s);
        return v == 3 ? launch_fixed_tma_alg<ALG, 3, 2, 3, 1>(src, n, L, dst, s)
                                 : launch_fixed_tma_alg<ALG, 1, 2, 3, 1>(src, n, L, dst, s);
    case kCfgW1x4:
        if constexpr (ALG == kMd5)
            if (v == 5) return launch_fixed_tma_alg<ALG, 5, 4, 3, 1>(src, n, L, dst, s);
        return v == 3 ? launch_fixed_tma_alg<ALG, 3, 4, 3, 1>(src, n, L, dst, s)
                      : launch_fixed_tma_alg<ALG, 1, 4, 3, 1>(src, n, L, dst, s);
    case kCfgW1x4s2: return launch_fixed_tma_alg<ALG, 1, 4, 2, 1>(src, n, L, dst, s);
    case kCfgW1x2p:  // the shipping single-warp kernel (PDL, early loads) at the selected variant
        if constexpr (ALG == kMd5) {
            if (v == 4) return launch_fixed_tma_w1<ALG, 4, 2, 3>(src, n, L, dst, s);
            if (v == 6) return launch_fixed_tma_w1<ALG, 6, 2, 3>(src, n, L, dst, s);
        }
        return launch_fixed_tma_w1<ALG, 1, 2, 3>(src, n, L, dst, s);
    case kCfgW1x2s2:  // shipping single-warp kernel, 2 stages (more CTAs per SM) / 3 messages per thread
        if constexpr (ALG == kMd5) return launch_fixed_tma_w1<ALG, 6, 2, 2>(src, n, L, dst, s);
        return launch_fixed_tma_w1<ALG, 1, 2, 2>(src, n, L, dst, s);
    case kCfgW1x3:
        if constexpr (ALG == kMd5) return launch_fixed_tma_w1<ALG, 6, 3, 3>(src, n, L, dst, s);
        return launch_fixed_tma_w1<ALG, 1, 3, 3>(src, n, L, dst, s);
    case kCfgW1x4p:  // shipping single-warp kernel, 4 messages per thread
        if constexpr (ALG == kMd5) return launch_fixed_tma_w1<ALG, 6, 4, 3>(src, n, L, dst, s);
        return launch_fixed_tma_w1<ALG, 1, 4, 3>(src, n, L, dst, s);
    case kCfgW1x2s4:
        if constexpr (ALG == kMd5) return launch_fixed_tma_w1<ALG, 4, 2, 4>(src, n, L, dst, s);
        return launch_fixed_tma_w1<ALG, 1, 2, 4>(src, n, L, dst, s);
    case kCfgWs3v6:
        if constexpr (ALG == kMd5) return launch_fixed_tma_ws<ALG, 6, 1, 3>(src, n, L, dst, s);
        return launch_fixed_tma_ws<ALG, 1, 1, 3>(src, n, L, dst, s);
    case kCfgWs3u: return launch_fixed_tma_ws<ALG, kVarBal, 1, 3, true>(src, n, L, dst, s);
    case kCfgWs3n: return launch_fixed_tma_ws<ALG, kVarBal, 1, 3, false, false>(src, n, L, dst, s);
    case kCfgWs3x2u: return launch_fixed_tma_ws<ALG, kVarBal, 2, 3, true>(src, n, L, dst, s);
    case kCfgWs2x2: return v == 3 ? launch_fixed_tma_ws<ALG, 3, 2, 2>(src, n, L, dst, s)
                                  : launch_fixed_tma_ws<ALG, 1, 2, 2>(src, n, L, dst, s);
    case kCfgWs3x2: return v == 3 ? launch_fixed_tma_ws<ALG, 3, 2, 3>(src, n, L, dst, s)
                                  : launch_fixed_tma_ws<ALG, 1, 2, 3>(src, n, L, dst, s);
    case kCfg2x2:
        switch (v) {
        case 0: return launch_fixed_tma_alg<ALG, 0, 2, 2>(src, n, L, dst, s);
        case 2: return launch_fixed_tma_alg<ALG, 2, 2, 2>(src, n, L, dst, s);
        default: return launch_fixed_tma_alg<ALG, 1, 2, 2>(src, n, L, dst, s);
        }
    case kCfg2x3:
        switch (v) {
        case 0: return launch_fixed_tma_alg<ALG, 0, 2, 3>(src, n, L, dst, s);
        case 2: return launch_fixed_tma_alg<ALG, 2, 2, 3>(src, n, L, dst, s);
        default: return launch_fixed_tma_alg<ALG, 1, 2, 3>(src, n, L, dst, s);
        }
    default:
        switch (v) {
        case 0: return launch_fixed_tma_alg<ALG, 0, 1, 3>(src, n, L, dst, s);
        case 2: return launch_fixed_tma_alg<ALG, 2, 1, 3>(src, n, L, dst, s);
        case 3: return launch_fixed_tma_alg<ALG, 3, 1, 3>(src, n, L, dst, s);
        default: return launch_fixed_tma_alg<ALG, 1, 1, 3>(src, n, L, dst, s);
        }
    }
}

// Compile-time-width kernel arms: plain rounds ($HB_CONST_VARIANT=0) and the
// CTA size ($HB_SMALL_CTA: fewer threads per CTA spread a small batch over
// more SMs).
template <int ALG, int L>
static void launch_small_one_ab(const uint8_t* d_msgs, uint64_t n, uint8_t* d_out, cudaStream_t s) {
    const Tuning& T = tuning();
    const unsigned b = T.small_cta >= 128 ? 128u : T.small_cta >= 64 ? 64u : 32u;
    const bool pair = T.small_pair_all || (ALG == kMd5 && n >= (1ull << 20) && L <= 32 && T.small_pair);
    if (T.const_variant == 0)
        launch_pdl(k_fixed_small<ALG, L, kVarPlain>, (unsigned)((n + b - 1) / b), b, s, d_msgs, n, d_out, 0u);
    else if (T.const_variant == 3)
        launch_pdl(k_fixed_small<ALG, L, kVarBal3>, (unsigned)((n + b - 1) / b), b, s, d_msgs, n, d_out, 0u);
    else if (T.const_variant == 4)
        launch_pdl(k_fixed_small<ALG, L, ALG == kMd5 ? 4 : kVarBal3>, (unsigned)((n + b - 1) / b), b, s, d_msgs, n, d_out, 0u);
    else if (pair)
        launch_pdl(k_fixed_small<ALG, L, kVarBal, 2>, (unsigned)(((n + 1) / 2 + b - 1) / b), b, s, d_msgs, n, d_out, 0u);
    else
        launch_pdl(k_fixed_small<ALG, L, kVarBal>, (unsigned)((n + b - 1) / b), b, s, d_msgs, n, d_out, 0u);
}

template <int ALG>
static cudaError_t launch_small_ab(const uint8_t* d_msgs, uint64_t n, uint64_t L, uint8_t* d_out, cudaStream_t s) {
    switch (L) {
    case 16: launch_small_one_ab<ALG, 16>(d_msgs, n, d_out, s); break;
    case 32: launch_small_one_ab<ALG, 32>(d_msgs, n, d_out, s); break;
    case 48: launch_small_one_ab<ALG, 48>(d_msgs, n, d_out, s); break;
    case 64: launch_small_one_ab<ALG, 64>(d_msgs, n, d_out, s); break;
    case 128: launch_small_one_ab<ALG, 128>(d_msgs, n, d_out, s); break;
    default: launch_plain(k_fixed_direct<ALG>, (unsigned)((n + 127) / 128), 128, s, d_msgs, n, (uint32_t)L, d_out);
    }
    return cudaGetLastError();
}

static bool varlen_ab_selected(uint32_t flags) {
    const Tuning& T = tuning();
    return (flags & (HB_FLAG_VARLEN_WORDS | HB_FLAG_VARLEN_COOP)) || T.varlen_bulk || T.varlen_prefetch ||
           T.varlen_ld == 32 || T.varlen_kernel >= 0;
}

template <int ALG>
static cudaError_t launch_varlen_ab(const uint8_t* d_data, uint64_t data_bytes, const uint64_t* d_offsets,
                                    uint64_t offset_base, uint64_t n, uint8_t* d_out, void* d_scratch,
                                    cudaStream_t stream, uint32_t flags) {
    const Tuning& T = tuning();
    const bool special = (flags & (HB_FLAG_VARLEN_WORDS | HB_FLAG_VARLEN_COOP)) || T.varlen_bulk;
    const bool wide = !special && T.varlen_ld == 32;
    const uint32_t* perm = nullptr;
    const int qcls = wide ? (int)T.varlen_q : 4;
    // k_varlen16m groups warps by the word class of byte a-1: sort on a bias one lower
    const uint64_t sort_base = T.varlen_kernel == 52 ? offset_base + 1 : offset_base;
    cudaError_t e = launch_varlen_sort(ALG, d_data, d_offsets, sort_base, n, d_scratch, stream, flags, &perm,
                                       qcls == 4 ? 4 : 8);
    if (e != cudaSuccess) return e;
    const unsigned grid = (unsigned)((n + 127) / 128);
    if (wide) {
        if (T.varlen_prefetch)
            launch_plain(k_varlen32<ALG, 1>, grid, 128, stream, d_data, d_data + data_bytes, d_offsets, offset_base,
                         perm, n, d_out);
        else
            launch_plain(k_varlen32<ALG>, grid, 128, stream, d_data, d_data + data_bytes, d_offsets, offset_base,
                         perm, n, d_out);
    } else if (flags & HB_FLAG_VARLEN_WORDS) {
        launch_plain(k_generic<ALG, true>, grid, 128, stream, d_data, d_data + data_bytes, d_offsets, offset_base,
                     perm, (uint64_t)0, n, d_out);
    } else if ((flags & HB_FLAG_VARLEN_COOP) && data_bytes < (1ull << 37)) {
        constexpr int T32 = kVcWarps * 32;
        const unsigned gg = (unsigned)((n + T32 - 1) / T32);
        const int stages = T.vc_stages > 0 ? T.vc_stages : (ALG == kMd5 ? 3 : 4);
        if (stages == 3) launch_plain(k_varlen_coop<ALG, 3, 7, 256>, gg, T32, stream, d_data, d_offsets, offset_base, perm, n, d_out);
        else if (stages == 2) launch_plain(k_varlen_coop<ALG, 2, 8, 256>, gg, T32, stream, d_data, d_offsets, offset_base, perm, n, d_out);
        else if (T.vc_pf == 128) launch_plain(k_varlen_coop<ALG, 4, 5, 128>, gg, T32, stream, d_data, d_offsets, offset_base, perm, n, d_out);
        else if (T.vc_pf == 0) launch_plain(k_varlen_coop<ALG, 4, 5, 0>, gg, T32, stream, d_data, d_offsets, offset_base, perm, n, d_out);
        else launch_plain(k_varlen_coop<ALG, 4, 5, 256>, gg, T32, stream, d_data, d_offsets, offset_base, perm, n, d_out);
    } else if (T.varlen_bulk) {
        switch (T.varlen_bulk) {  // ring depth x register cap
        case 2: launch_plain(k_varlen_bulk<ALG, 2, 1>, grid, 128, stream, d_data, d_offsets, offset_base, perm, n, d_out); break;
        case 4: launch_plain(k_varlen_bulk<ALG, 3, 6>, grid, 128, stream, d_data, d_offsets, offset_base, perm, n, d_out); break;
        case 5: launch_plain(k_varlen_bulk<ALG, 2, 8>, grid, 128, stream, d_data, d_offsets, offset_base, perm, n, d_out); break;
        default: launch_plain(k_varlen_bulk<ALG, 3, 1>, grid, 128, stream, d_data, d_offsets, offset_base, perm, n, d_out); break;
        }
    } else if (T.varlen_kernel >= 20) {  // load-hint arms: 20 + 3*LD + PF (PF 0 | 1; 25 / 28: carry, LD 0 / 1)
        const unsigned blk = T.small_cta >= 128 ? 128u : 64u;  // $HB_SMALL_CTA=64: 64-thread CTAs
        const unsigned g2 = (unsigned)((n + blk - 1) / blk);
        switch (T.varlen_kernel) {
        case 23: launch_plain(k_varlen16<ALG, 0, 1>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        case 24: launch_plain(k_varlen16<ALG, 1, 1>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        case 26: launch_plain(k_varlen16<ALG, 0, 2>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        case 27: launch_plain(k_varlen16<ALG, 1, 2>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        case 21: launch_plain(k_varlen16<ALG, 1, 0>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        case 25: launch_plain(k_varlen16<ALG, 5, 0>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        // register caps: 29 / 30 = pipelined kernel at >= 8 / 9 CTAs per SM, 31 = plain kernel at 10
        case 29: launch_plain(k_varlen16<ALG, 1, 0, 8>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        case 30: launch_plain(k_varlen16<ALG, 1, 0, 9>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        case 31: launch_plain(k_varlen16<ALG, 0, 0, 10>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        case 32: launch_plain(k_varlen16<ALG, 3, 0>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        case 33: launch_plain(k_varlen16x2<ALG>, (unsigned)(((n + 1) / 2 + blk - 1) / blk), blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        case 28: launch_plain(k_varlen16<ALG, 5, 1>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        // lean block loop: 40 = one loop (runtime realignment switch), 41 = one loop per alignment class
        case 40: launch_plain(k_varlen16l<ALG, false>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        case 41: launch_plain(k_varlen16l<ALG, true>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        // ... with MD5 round variant 4 / 6 / 7 (one round in three / two / four sums a + M + K in one IADD3)
        case 42: launch_plain(k_varlen16l<ALG, false, ALG == kMd5 ? 4 : -1>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        case 43: launch_plain(k_varlen16l<ALG, true, ALG == kMd5 ? 4 : -1>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        case 44: launch_plain(k_varlen16l<ALG, true, ALG == kMd5 ? 6 : -1>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        case 45: launch_plain(k_varlen16l<ALG, true, ALG == kMd5 ? 7 : -1>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        // 46: per-class loops + variant 4 + L2 policies (first window evict_last, tail evict_first); 47: runtime switch + L2 policies
        case 46: launch_plain(k_varlen16l<ALG, true, ALG == kMd5 ? 4 : -1, true>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        case 47: launch_plain(k_varlen16l<ALG, false, -1, true>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        // lean loop, uniform finish (nb compressions per warp, not nb + 1)
        case 48: launch_plain(k_varlen16f<ALG>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        case 49: launch_plain(k_varlen16g<ALG>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        case 50: launch_plain(k_varlen16g<ALG, true>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        // lean loop unrolled by two, fifth granule carried (4 loads per block), L2 policies
        case 51: launch_plain(k_varlen16c<ALG>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        // realignment on the FMA pipe (IMAD.HI + IMAD instead of funnel shifts), sort keyed on a-1
        case 52: launch_plain(k_varlen16m<ALG>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        // the shipping MD5 loop (runtime alignment switch + L2 policies) at MD5 round variants 3 / 4 / 5 / 6
        case 53: launch_plain(k_varlen16l<ALG, false, ALG == kMd5 ? 3 : -1, true>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        case 54: launch_plain(k_varlen16l<ALG, false, ALG == kMd5 ? 4 : -1, true>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        case 55: launch_plain(k_varlen16l<ALG, false, ALG == kMd5 ? 5 : -1, true>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        case 56: launch_plain(k_varlen16l<ALG, false, ALG == kMd5 ? 6 : -1, true>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        default: launch_plain(k_varlen16<ALG, 0, 0>, g2, blk, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        }
    } else if (T.varlen_kernel >= 10) {  // prefetch-instruction arms of the per-thread kernel (PF = kernel - 10)
        switch (T.varlen_kernel - 10) {
        case 2: launch_plain(k_varlen16<ALG, 2>, grid, 128, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        case 3: launch_plain(k_varlen16<ALG, 3>, grid, 128, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        default: launch_plain(k_varlen16<ALG, 4>, grid, 128, stream, d_data, d_data + data_bytes, d_offsets, offset_base, perm, n, d_out); break;
        }
    } else if (T.varlen_kernel == 0) {  // the per-thread kernel with md_finish tails
        launch_plain(k_varlen16<ALG, 0>, grid, 128, stream, d_data, d_data + data_bytes, d_offsets, offset_base,
                     perm, n, d_out);
    } else if (T.varlen_kernel == 2) {  // uniform block loop, every addition on the FMA pipe
        launch_plain(k_varlen16u<ALG, kVarBal2>, grid, 128, stream, d_data, d_data + data_bytes, d_offsets,
                     offset_base, perm, n, d_out);
    } else if (T.varlen_kernel == 1) {  // uniform block loop, tuned variant
        launch_plain(k_varlen16u<ALG, kVarBal>, grid, 128, stream, d_data, d_data + data_bytes, d_offsets,
                     offset_base, perm, n, d_out);
    } else if (T.varlen_prefetch) {
        launch_plain(k_varlen16<ALG, 1>, grid, 128, stream, d_data, d_data + data_bytes, d_offsets, offset_base,
                     perm, n, d_out);
    } else {
        launch_plain(k_varlen16<ALG, 0>, grid, 128, stream, d_data, d_data + data_bytes, d_offsets, offset_base,
                     perm, n, d_out);
    }
    return cudaGetLastError();
}

// Decimal arms: $HB_DEC_PAIR, $HB_FMA_DIGITS=0 (IMAD.HI + SHF digits),
// $HB_CONST_VARIANT = 1 | 3, $HB_DEC_RUN=0.
template <int ALG, int W>
static void dec_launch_ab(uint64_t start, uint64_t count, uint8_t* d_out, cudaStream_t s) {
    const Tuning& T = tuning();
    const unsigned grid = (unsigned)((count + 127) / 128);
    if constexpr (W >= 2 && W <= 10) {
        if (T.dec_run && (start + count) / 10u < (1ull << 30) - 1) {
            const uint64_t threads = (start + count + 9u) / 10u - start / 10u;
            const unsigned g = (unsigned)((threads + 127) / 128);
            if (T.const_variant == 3)
                launch_plain(k_decimal_run<ALG, W, kVarBal3>, g, 128, s, start, count, d_out);
            else if (T.const_variant == 4 && ALG == kMd5)
                launch_plain(k_decimal_run<ALG, W, ALG == kMd5 ? 4 : kVarBal, true>, g, 128, s, start, count, d_out);
            else if (T.dec_pair >= 0 ? T.dec_pair : ALG == kMd5)
                launch_plain(k_decimal_run<ALG, W, kVarBal, true>, g, 128, s, start, count, d_out);
            else
                launch_plain(k_decimal_run<ALG, W, kVarBal>, g, 128, s, start, count, d_out);
            return;
        }
    }
    if (!T.fma_digits)
        launch_plain(k_decimal<ALG, W, kVarBal, false>, grid, 128, s, start, count, d_out);
    else if ((T.const_variant >= 0 ? T.const_variant : (ALG == kSha1 ? 3 : 1)) == 3)
        launch_plain(k_decimal<ALG, W, kVarBal3, true>, grid, 128, s, start, count, d_out);
    else
        launch_plain(k_decimal<ALG, W, kVarBal, true>, grid, 128, s, start, count, d_out);
}
