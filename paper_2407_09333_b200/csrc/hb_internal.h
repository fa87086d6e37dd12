// hb_internal.h -- launcher interface between the kernel TU (hb_kernels.cu)
// and the host engine / C ABI (hb_engine.cu).  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hb {

// Launch-count bookkeeping (bench.py reports gpu_launches from this).
void note_launches(uint64_t k);

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
