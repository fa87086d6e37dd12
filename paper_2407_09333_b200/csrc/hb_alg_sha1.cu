// hb_alg_sha1.cu -- SHA1 instantiation of the hash kernels (hb_kernels.cuh).
#include "hb_kernels.cuh"

namespace hb {

cudaError_t launch_fixed_sha1(const uint8_t* d_msgs, uint64_t n, uint64_t L, uint8_t* d_out, cudaStream_t s,
                            uint32_t flags) {
    return launch_fixed_alg<kSha1>(d_msgs, n, L, d_out, s, flags);
}

cudaError_t launch_varlen_sha1(const uint8_t* d_data, uint64_t data_bytes, const uint64_t* d_offsets,
                             uint64_t offset_base, uint64_t n, uint8_t* d_out, void* d_scratch, cudaStream_t s,
                             uint32_t flags) {
    return launch_varlen_alg<kSha1>(d_data, data_bytes, d_offsets, offset_base, n, d_out, d_scratch, s, flags);
}

cudaError_t launch_decimal_sha1(uint64_t start, uint64_t count, int width, uint8_t* d_out, cudaStream_t s) {
    return launch_decimal_alg<kSha1>(start, count, width, d_out, s);
}

}  // namespace hb
