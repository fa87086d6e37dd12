// hb_internal.h -- launcher interface between the kernel TU (hb_kernels.cu)
// and the host engine / C ABI (hb_engine.cu).  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hb {

// ------------------------------------------------------------------ tuning --
// Every knob of the engine and the kernel dispatch, parsed ONCE from the
// environment (first use, or hb_tuning_reload()).  Launch paths read these
// fields; none calls getenv.  Defaults are the B200-measured best (DESIGN.md
// §4).  The fields under "A/B" only have an effect in a -DHB_AB build, which
// also instantiates the losing kernel arms they select.
struct Tuning {
    // engine (hb_engine.cu)
    uint64_t chunk_bytes = 256ull << 20;        // $HB_CHUNK_BYTES: sub-batch (chunk) input bytes
    uint64_t pipe_min_out = 4ull << 20;         // $HB_PIPE_MIN_OUT: digest bytes from which a shard is pipelined
    uint64_t pipe_chunks = 4;                   // $HB_PIPE_CHUNKS
    uint64_t min_chunk_bytes = 8ull << 20;      // $HB_MIN_CHUNK_BYTES
    uint64_t memcpy_threads = 0;                // $HB_MEMCPY_THREADS (0 = auto)
    bool bind_numa = true;                      // $HB_BIND_NUMA=0 disables worker NUMA pinning
    uint64_t multi_gpu_min_bytes = 32ull << 20; // $HB_MULTI_GPU_MIN_BYTES: smaller default-GPU calls use one GPU
    uint64_t device_reserve = 2ull << 30;       // $HB_DEVICE_RESERVE: HBM left free when sizing the chunk ring
    // kernels (hb_kernels.cuh)
    bool pdl = true;                            // $HB_PDL
    uint64_t small_n = 1ull << 18;              // $HB_SMALL_N: below it, one message per thread in TMA tiles
    uint64_t chain_n = 1ull << 16;              // $HB_CHAIN_N: MD5 TMA batches below it: 4+1-warp tile, variant 6
    bool late_wait = true;                      // $HB_LATE_WAIT: INPUT_READY launches wait only before their stores
    uint32_t trigger_wave_pct = 100;            // $HB_TRIGGER_WAVE_PCT: early release if the grid fits this share of the slots
    uint64_t md5_nb3_n = 1ull << 22;            // $HB_MD5_NB3_N: from it, three messages per thread in the single-warp tile
    bool varlen_pf = true;                      // $HB_VARLEN_PF: MD5 varlen, software-pipelined per-thread kernel
    bool sort_qmajor = true;                    // $HB_SORT_QMAJOR: windowed sort key (q, block count), else (block count, q)
    uint64_t direct_max_len = 128;              // $HB_DIRECT_MAX_L: rows up to it use the per-thread-load kernels
    bool small_pair = true;                     // $HB_SMALL_PAIR: MD5 <= 32 B rows, two per thread at >= 2^20
    bool dec_run = true;                        // $HB_DEC_RUN: runs-of-ten decimal kernel
    uint64_t zc_max_bytes = 256u << 10;         // $HB_ZERO_COPY_MAX: single-GPU untimed calls up to it read host memory directly (0 = off)
    bool small_poll = true;                     // $HB_SMALL_POLL: hb_digest_small polls its mapped slot, else syncs the stream
    int varlen_sort = -1;                       // $HB_VARLEN_SORT: -1 per algorithm, 0 global, 1 window
    // A/B (-DHB_AB)
    int tma_cfg = -1;                           // $HB_TMA_CFG
    int variant = -1;                           // $HB_VARIANT
    uint32_t tma_l2 = 256;                      // $HB_TMA_L2
    uint32_t tma_evict_first = 0;               // $HB_TMA_EVICT_FIRST
    bool small_kernel = true;                   // $HB_NO_SMALL_KERNEL
    bool small_kernel_ab = false;               // $HB_CONST_VARIANT=0 / $HB_SMALL_CTA set
    int const_variant = -1;                     // $HB_CONST_VARIANT
    uint32_t small_cta = 128;                   // $HB_SMALL_CTA
    bool small_pair_all = false;                // $HB_SMALL_PAIR_ALL: two rows per thread at every width / count
    bool input_ready = false;                   // $HB_INPUT_READY: treat every fixed-width launch as HB_FLAG_INPUT_READY
    bool dec_ab = false;                        // any of $HB_DEC_PAIR / $HB_FMA_DIGITS / $HB_CONST_VARIANT set
    int dec_pair = -1;                          // $HB_DEC_PAIR
    bool fma_digits = true;                     // $HB_FMA_DIGITS
    uint32_t sort_window = 8192;                // $HB_SORT_WINDOW
    uint32_t varlen_ld = 16;                    // $HB_VARLEN_LD
    uint32_t varlen_q = 8;                      // $HB_VARLEN_Q
    uint32_t varlen_prefetch = 0;               // $HB_VARLEN_PREFETCH
    uint32_t varlen_bulk = 0;                   // $HB_VARLEN_BULK
    int varlen_kernel = -1;                     // $HB_VARLEN_KERNEL: 0 k_varlen16, 1 / 2 k_varlen16u variant 1 / 2
    int vc_stages = -1;                         // $HB_VC_STAGES
    uint32_t vc_pf = 256;                       // $HB_VC_PF
};
const Tuning& tuning();
void tuning_reload();
bool built_with_ab();

// Launch bookkeeping: a process-wide count (bench.py reports gpu_launches
// from it) and, per calling thread, the last hash kernel launched (its symbol
// is resolved by hb_last_kernel_name, so reports name the kernel that ran).
void note_launch(const void* kernel, bool hash_kernel);
void note_launches(uint64_t k);
const void* last_hash_kernel();
void set_last_hash_kernel(const void* kernel);  // propagate a worker thread's launch to the caller

// Fixed-width messages already resident on the current device.
//   d_msgs: n*msg_len bytes (row i at i*msg_len), d_out: n*dlen bytes.
// Picks the TMA-staged kernel when msg_len % 16 == 0 and d_msgs is 16-byte
// aligned (unless HB_FLAG_NO_TMA), else the generic unaligned-load kernel.
cudaError_t launch_fixed(int alg, const uint8_t* d_msgs, uint64_t n, uint64_t msg_len, uint8_t* d_out,
                         cudaStream_t stream, uint32_t flags);

// Length/alignment-bucket permutation used by launch_varlen (*perm_out = null
// when not sorting: HB_FLAG_NO_SORT, small n or no scratch).
cudaError_t launch_varlen_sort(int alg, const uint8_t* d_data, const uint64_t* d_offsets, uint64_t offset_base,
                               uint64_t n, void* d_scratch, cudaStream_t stream, uint32_t flags,
                               const uint32_t** perm_out, int qclasses = 4);

// Scratch bytes launch_varlen needs for n messages (length-bucket sort).
uint64_t varlen_scratch_bytes(uint64_t n);

// Variable-length messages: message i = d_data[d_offsets[i]-offset_base, d_offsets[i+1]-offset_base).
// d_scratch must hold varlen_scratch_bytes(n) bytes (may be null when
// HB_FLAG_NO_SORT is set or n is small).
cudaError_t launch_varlen(int alg, const uint8_t* d_data, uint64_t data_bytes, const uint64_t* d_offsets,
                          uint64_t offset_base, uint64_t n, uint8_t* d_out, void* d_scratch, cudaStream_t stream,
                          uint32_t flags);

// One message of len <= HB_DIGEST_SMALL_MAX host bytes, passed by value in
// the launch; the digest is stored at `out` (device-visible, e.g. mapped
// pinned host memory) and then, when seq != 0, the u32 seq at out + 48
// (release, system scope).
cudaError_t launch_digest_small(int alg, const uint8_t* msg, uint64_t len, uint8_t* out, uint32_t seq,
                                cudaStream_t stream);

// Counter-based synthetic bytes (same stream as oracle/orc_fill_random).
cudaError_t launch_fill_random(uint8_t* d_buf, uint64_t nbytes, uint64_t seed, uint64_t byte_offset,
                               cudaStream_t stream);

// gen_messages(start, count, width) digests computed with the messages
// generated in registers (no message bytes in HBM at all).
cudaError_t launch_decimal(int alg, uint64_t start, uint64_t count, int width, uint8_t* d_out, cudaStream_t stream);

// Materialise gen_messages bytes on the device (count*width bytes).
cudaError_t launch_gen_decimal(uint64_t start, uint64_t count, int width, uint8_t* d_out, cudaStream_t stream);

const char* tma_error();

}  // namespace hb
