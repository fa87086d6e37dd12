/*
 * hetoc_b200.h -- C ABI of the B200-native batched-hash engine.
 *
 * Plain pointers and sizes only (no torch / CUDA types in the signatures;
 * `stream` is an opaque cudaStream_t passed as void*).  Every entry point
 * returns an hb_status; on failure hb_last_error() (thread-local) says why.
 * The Python package paper_2407_09333_b200.crypto binds these with ctypes,
 * mirroring the reference API (hetoc.crypto); INTEGRATION.md shows the
 * binding.
 *
 * Which reference interface each entry point replaces (paths relative to the
 * reference repo root):
 *
 *   hb_hash_fixed     batch_digest(alg, data)            pkg/src/hetoc/crypto/batch.py:274-290
 *                     (+ the hyper staging contract of _emit_dev_launch,
 *                      pkg/src/hetoc/passes/lower_hyper_for.py:279-368, the
 *                      message-range split partition_range,
 *                      pkg/src/hetoc/passes/partition.py:17-31, and the
 *                      capacity sub-batching of _run_group,
 *                      pkg/src/hetoc/runtime/executor.py:603-699)
 *   hb_hash_varlen    digest(alg, msg) mapped over an offsets array
 *                     (pkg/src/hetoc/crypto/batch.py:102-109; the reference has
 *                      no variable-length batch layout)
 *   hb_hash_fixed_dev _CHUNK_FN[alg](rows) on device-resident rows
 *                     pkg/src/hetoc/crypto/batch.py:263 / dev.launch body,
 *                     pkg/src/hetoc/runtime/executor.py:562-599
 *   hb_hash_decimal   hash_batch(alg, gen_messages(start, count, width))
 *                     pkg/src/hetoc/crypto/batch.py:86-99, :293-316
 *   hb_hash_fixed_split hash_batch lowered with hyper.for duty ratios over GPUs
 *                     (lower_loop pkg/src/hetoc/passes/lower_hyper_for.py:207-254)
 *   hb_partition_range partition_range  pkg/src/hetoc/passes/partition.py:17-31
 *   hb_device_count / hb_device_info   detect_hardware
 *                     pkg/src/hetoc/runtime/devices.py:169-184
 *   hb_digest_len     DIGEST_LEN         pkg/src/hetoc/crypto/batch.py:23
 */
#ifndef HETOC_B200_H
#define HETOC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HB_ABI_VERSION 3

typedef enum {
    HB_OK = 0,
    HB_ERR_ALG = 1,      /* unknown algorithm          -> UnknownAlgorithmError */
    HB_ERR_INVAL = 2,    /* bad argument               -> ValueError            */
    HB_ERR_CUDA = 3,     /* CUDA runtime/driver error  -> RuntimeError          */
    HB_ERR_NOMEM = 4,    /* device or pinned allocation failed                  */
    HB_ERR_NODEV = 5     /* no CUDA device / bad device ordinal                 */
} hb_status;

typedef enum { HB_SHA1 = 0, HB_MD5 = 1, HB_SM3 = 2 } hb_alg;

/* flags */
#define HB_FLAG_NO_TMA   0x1u  /* fixed width: direct-load kernel instead of TMA staging */
#define HB_FLAG_NO_SORT  0x2u  /* varlen: skip the length-bucket sort                    */
#define HB_FLAG_SYNC_H2D 0x4u  /* engine: no copy/compute overlap (diagnostics)          */
/* fixed width, hb_hash_fixed_dev: the caller guarantees the message bytes are
 * not written by the kernel that immediately precedes this launch on the
 * stream (e.g. they were copied in, or written earlier and synchronised).
 * The hash kernel then starts -- reading and hashing its messages -- while
 * that kernel is still running (programmatic dependent launch): consecutive
 * batches overlap; only the digest stores wait until it completes.  (The engine's own chunks follow their H2D copy, which a
 * dependent launch never overlaps, so it does not need it.)
 * varlen, hb_hash_varlen_dev (MD5's windowed length sort): the same guarantee
 * for `offsets` -- the sort then starts while the preceding varlen hash
 * kernel drains (that kernel releases it once every thread has read its
 * permutation entry, so the scratch may be the same); the hash kernel itself
 * still starts only after the sort completes.                               */
#define HB_FLAG_INPUT_READY 0x40u
/* A/B kernel arms: honoured only by a library built with -DHB_AB
 * (hb_built_with_ab() == 1); the default build returns HB_ERR_CUDA with
 * hb_last_error() saying so for VARLEN_WORDS / VARLEN_COOP.                 */
#define HB_FLAG_VARLEN_WORDS 0x8u /* varlen: per-thread 32-bit-load kernel (A/B baseline)       */
#define HB_FLAG_VARLEN_COOP_OFF 0x10u /* varlen: per-thread 128-bit-load kernel (the default;
                                         kept so callers can pin it explicitly)                 */
#define HB_FLAG_VARLEN_COOP 0x20u     /* varlen: warp-cooperative cp.async staging kernel      */

typedef struct {
    double total_ms;       /* host wall time of the call                              */
    double kernel_ms;      /* max over GPUs of the union of hash-kernel busy intervals */
    double h2d_ms;         /* max over GPUs of the union of H2D busy intervals         */
    double d2h_ms;         /* max over GPUs of the union of D2H busy intervals         */
    uint64_t h2d_bytes;    /* total bytes copied host -> device                       */
    uint64_t d2h_bytes;    /* total bytes copied device -> host                       */
    uint64_t chunks;       /* sub-batches (chunks) executed over all GPUs             */
    uint64_t launches;     /* kernels launched by this call                           */
    uint64_t shards;       /* GPUs that received a non-empty message range           */
    uint64_t device_mask;  /* bit d set: GPU d ran a shard                            */
} hb_timing;

/* One stage of one chunk on one GPU (hb_last_timeline): stage 0 = H2D,
 * 1 = hash kernel(s), 2 = D2H; times in ms from that GPU's first event of
 * the call (device clock, CUDA events).                                     */
typedef struct {
    int32_t dev;
    int32_t stage;
    uint64_t chunk;
    double t0_ms, t1_ms;
} hb_span;

typedef struct {
    int ordinal;
    int sm_count;
    int cc_major, cc_minor;
    uint64_t total_mem;
    uint64_t free_mem;
    int pci_bus_id;
    int clock_khz;
    char name[96];
} hb_device_info_t;

/* ---- introspection ---------------------------------------------------- */
int hb_abi_version(void);
const char *hb_last_error(void);          /* thread-local message of the last failure */
int hb_digest_len(int alg);               /* 20 / 16 / 32, or -1                      */
int hb_device_count(int *n);
int hb_device_info(int ordinal, hb_device_info_t *info);
uint64_t hb_launch_count(void);           /* kernels launched by this process so far   */

/* ---- host-buffer engine (staging + sharding + chunked streaming) ------- */
/* Hash n fixed-width messages (row i = msgs[i*msg_len, (i+1)*msg_len)) into
 * out[i*dlen, (i+1)*dlen).  [0,n) is split over gpus[0..n_gpus) with
 * partition_range's cumulative round-half-up rule and equal ratios; each GPU
 * streams its slice through a ring of pinned/device chunk buffers (H2D, kernel,
 * D2H overlapped on separate streams).  Host buffers may be pageable or
 * pinned (pinned is copied directly).  gpus == NULL / n_gpus == 0 means "all
 * devices" for calls staging >= $HB_MULTI_GPU_MIN_BYTES (32 MiB); smaller
 * calls run on ONE GPU chosen per calling thread (round-robin over threads).
 * Single-GPU calls run on the calling thread; multi-GPU calls hand their
 * shards to persistent per-GPU worker threads (NUMA-bound to their GPU).
 * t may be NULL (then no per-stage CUDA events are recorded, which saves
 * ~30 us per call on small batches).  msg_len 0 hashes empty messages.
 * Each GPU stages through kSlots = 3 chunk buffers whose size is capped by
 * that GPU's budget (free HBM at first use minus $HB_DEVICE_RESERVE, 2 GiB):
 * hb_engine_budget reports it.  An untimed (t == NULL) single-GPU call of at
 * most $HB_ZERO_COPY_MAX (256 KiB) message bytes and 128 KiB of digests skips
 * the ring: the batch is copied into a mapped pinned buffer that the kernel
 * reads over PCIe, and the digests are stored straight into mapped memory. */
int hb_hash_fixed(int alg, const uint8_t *msgs, uint64_t n, uint64_t msg_len, uint8_t *out,
                  const int *gpus, int n_gpus, uint32_t flags, hb_timing *t);

/* Same with explicit duty ratios per GPU -- the hyper.for device bindings
 * (lower_loop + partition_range, pkg/src/hetoc/passes/lower_hyper_for.py:207-254):
 * ratios[i] in [0,1] summing to 1 (+-1e-9, pkg/src/hetoc/hir/verify.py:245-260);
 * gpu i gets messages [b_i, b_{i+1}) by the cumulative round-half-up rule.
 * Output is bit-identical for every ratio vector.             */
int hb_hash_fixed_split(int alg, const uint8_t *msgs, uint64_t n, uint64_t msg_len, uint8_t *out,
                        const int *gpus, const double *ratios, int n_gpus, uint32_t flags, hb_timing *t);

/* Variable-length: message i = data[offsets[i], offsets[i+1]); offsets has n+1
 * non-decreasing entries, offsets[0] may be non-zero.                        */
int hb_hash_varlen(int alg, const uint8_t *data, const uint64_t *offsets, uint64_t n, uint8_t *out,
                   const int *gpus, int n_gpus, uint32_t flags, hb_timing *t);

/* One message (digest, pkg/src/hetoc/crypto/batch.py:102-109), len <=
 * HB_DIGEST_SMALL_MAX bytes, synchronously: the bytes are passed inside the
 * kernel launch and the digest is written to mapped pinned host memory, so a
 * call is one launch + one stream synchronise (no staging copies).  gpu < 0
 * picks the calling thread's default GPU as hb_hash_varlen does for a small
 * call.  Thread-safe; HB_ERR_INVAL for longer messages (use hb_hash_varlen). */
#define HB_DIGEST_SMALL_MAX 4096u
int hb_digest_small(int alg, const uint8_t *msg, uint64_t len, uint8_t *out, int gpu);

/* Paper workload (gen_messages): digests of the zero-padded decimal strings
 * of start .. start+count-1, width bytes each, generated on the GPU.
 * HB_ERR_INVAL unless start + count <= 10^width and does not wrap 2^64.    */
int hb_hash_decimal(int alg, uint64_t start, uint64_t count, int width, uint8_t *out,
                    const int *gpus, int n_gpus, uint32_t flags, hb_timing *t);

/* ---- device-resident (kernel-only) entry points ------------------------ */
/* All pointers are device pointers on `gpu`; work is enqueued on `stream`
 * (d_out rows are written with 16-byte stores for MD5 / SM3 and 4-byte
 * stores for SHA-1: d_out must be 16- / 4-byte aligned).
 * (NULL = legacy default stream) and NOT synchronised.  Fixed-width kernels
 * are launched with programmatic stream serialization (PDL): one may be
 * scheduled while the previous kernel on the stream drains, but it waits for
 * that kernel's completion (griddepcontrol.wait) before touching global
 * memory, so stream order holds as for a normal launch ($HB_PDL=0 disables). */
int hb_hash_fixed_dev(int alg, int gpu, const void *d_msgs, uint64_t n, uint64_t msg_len, void *d_out,
                      void *stream, uint32_t flags);
/* d_data must be readable up to round_up(address of the last byte + 1, 16)
 * (16-byte granular loads; cudaMalloc / torch allocations satisfy this).
 * d_scratch: hb_varlen_scratch_bytes(n) bytes, or NULL (unsorted).          */
int hb_hash_varlen_dev(int alg, int gpu, const void *d_data, uint64_t data_bytes, const uint64_t *d_offsets,
                       uint64_t offset_base, uint64_t n, void *d_out, void *d_scratch, void *stream,
                       uint32_t flags);
uint64_t hb_varlen_scratch_bytes(uint64_t n);
int hb_hash_decimal_dev(int alg, int gpu, uint64_t start, uint64_t count, int width, void *d_out, void *stream);

/* Synthetic message bytes: the counter-based generator (seed, byte_offset
 * multiple of 8) shared with the CPU oracle.  d_buf 8-byte aligned.          */
int hb_fill_random_dev(int gpu, void *d_buf, uint64_t nbytes, uint64_t seed, uint64_t byte_offset, void *stream);
/* gen_messages bytes on the device (count*width bytes).                     */
int hb_gen_decimal_dev(int gpu, uint64_t start, uint64_t count, int width, void *d_out, void *stream);

/* ---- staging memory ---------------------------------------------------- */
void *hb_alloc_pinned(uint64_t bytes);   /* page-locked, portable; NULL on failure */
int hb_free_pinned(void *p);
int hb_sync_device(int gpu);
/* Release every cached per-GPU context (streams, chunk buffers).            */
int hb_shutdown(void);

/* ---- peer-mapped digest buffers: the fused device-side gather ---------- */
/* north_star: "NCCL is needed only for an optional device-side gather".  The
 * fused form needs no collective at all: the root exports its (n, dlen)
 * digest buffer, every rank maps it (cudaIpcOpenMemHandle; peer access over
 * NVLink 5 / NVSwitch between GPUs) and passes root_ptr + s_i*dlen as d_out
 * of hb_hash_*_dev -- the hash kernels' own digest stores are the gather (the
 * copy-out rule dst_off = s*dlen of _emit_dev_launch,
 * pkg/src/hetoc/passes/lower_hyper_for.py:316).                              */
#define HB_IPC_HANDLE_BYTES 64
/* handle of the allocation holding d_ptr (64 bytes) + d_ptr's byte offset in it */
int hb_ipc_handle(const void *d_ptr, uint8_t *handle_out, uint64_t *offset_out);
int hb_ipc_open(int gpu, const uint8_t *handle, void **d_ptr_out);     /* map it: base; add the offset */
int hb_ipc_close(int gpu, void *d_ptr);

/* ---- engine introspection and tuning ----------------------------------- */
/* Re-read the $HB_* tuning environment (parsed once at first use otherwise).
 * Not synchronised with concurrent hash calls.                              */
int hb_tuning_reload(void);
int hb_built_with_ab(void);               /* 1 if the A/B kernel arms are compiled in */
/* Demangled name of the last hash kernel launched for the calling thread
 * (directly by *_dev, or by the engine for its last call).                  */
int hb_last_kernel_name(char *buf, int cap);
/* Stage spans of the calling thread's last call that passed an hb_timing:
 * copies min(count, cap) spans into out (may be NULL), returns count.       */
int hb_last_timeline(hb_span *out, int cap);
/* Per-GPU chunk-ring budget (bytes) and the largest input chunk it allows.  */
int hb_engine_budget(int gpu, uint64_t *budget, uint64_t *chunk_cap);

/* ---- task splitting ---------------------------------------------------- */
/* partition_range(lb, ub, ratios[0..k)): writes k+1 bounds.                 */
int hb_partition_range(int64_t lb, int64_t ub, const double *ratios, int k, int64_t *bounds_out);

#ifdef __cplusplus
}
#endif
#endif /* HETOC_B200_H */
