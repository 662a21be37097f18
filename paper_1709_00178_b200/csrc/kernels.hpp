// Ahead-of-time utility kernels (kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace pyrit_b200 {

cudaError_t launch_fill(std::uint64_t seed, std::uint64_t frag, std::uint8_t* dst, std::uint64_t begin,
                        std::uint64_t len, std::uint64_t valid, cudaStream_t stream);
cudaError_t launch_digest(const std::uint8_t* src, std::uint64_t len, std::uint64_t word_offset,
                          std::uint64_t* out, cudaStream_t stream);

} // namespace pyrit_b200
