// Ahead-of-time utility kernels (kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace pyrit_b200 {

cudaError_t launch_fill(std::uint64_t seed, std::uint64_t frag, std::uint8_t* dst, std::uint64_t begin,
                        std::uint64_t len, std::uint64_t valid, cudaStream_t stream);
cudaError_t launch_digest(const std::uint8_t* src, std::uint64_t len, std::uint64_t word_offset,
                          std::uint64_t* out, cudaStream_t stream);

// Generic bit-matrix kernel (kernels.cu): all in kernel parameters.
constexpr std::uint32_t kGenericMaxPtrs = 256;     // inputs + outputs
constexpr std::uint32_t kGenericMaxMasks = 12288;  // e * w rows x k inputs
struct GenericArgs {
    std::uint64_t S, off, nwords, nb, ibp, obp, sq, sr; // as the direct kernel (4-byte words)
    std::uint32_t k, e, w, pad;
    const std::uint8_t* ptr[kGenericMaxPtrs];  // k inputs, then e outputs
    std::uint16_t mask[kGenericMaxMasks];      // mask[(i*w + b)*k + j]: strips of input j in output i strip b
};
cudaError_t launch_generic(const GenericArgs& args, unsigned blocks, cudaStream_t stream);

} // namespace pyrit_b200
