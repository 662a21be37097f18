// Dispatch of the runtime-matrix ring kernel (K2 of SURVEY.md section 8) over the
// ring geometries with an ahead-of-time instance: the reference's field presets
// (field.hpp:103-132) and BASELINE's GF(2^8) in R_{2,17}.  The kernel itself is
// ring_rt.cuh; each geometry is its own translation unit (ring_rt_w*_n*.cu).
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.hpp"

namespace pyrit_b200 {

#define PYRIT_RT_FIELDS(X) X(4, 5, 0x1Fu) X(6, 9, 0x49u) X(8, 17, 0x139u) X(10, 11, 0x7FFu) X(12, 13, 0x1FFFu)

#define PYRIT_RT_DECL(W, N, P)                                                     \
    cudaError_t launch_ring_rt_w##W##_n##N(const RtArgs& a, const RtLaunch& l); \
    cudaError_t warm_ring_rt_w##W##_n##N();
PYRIT_RT_FIELDS(PYRIT_RT_DECL)
#undef PYRIT_RT_DECL

bool rt_supported(std::uint32_t w, std::uint32_t n, std::uint32_t modulus) {
#define PYRIT_RT_HAS(W, N, P) if (w == W && n == N && modulus == P) return true;
    PYRIT_RT_FIELDS(PYRIT_RT_HAS)
#undef PYRIT_RT_HAS
    return false;
}

cudaError_t launch_ring_rt(const RtArgs& a, const RtLaunch& l) {
#define PYRIT_RT_GO(W, N, P) if (l.w == W && l.n == N && l.modulus == P) return launch_ring_rt_w##W##_n##N(a, l);
    PYRIT_RT_FIELDS(PYRIT_RT_GO)
#undef PYRIT_RT_GO
    return cudaErrorInvalidValue;
}

cudaError_t warm_ring_rt() {
    cudaError_t first = cudaSuccess;
#define PYRIT_RT_WARM(W, N, P)                                \
    {                                                         \
        const cudaError_t e = warm_ring_rt_w##W##_n##N();      \
        if (first == cudaSuccess) first = e;                  \
    }
    PYRIT_RT_FIELDS(PYRIT_RT_WARM)
#undef PYRIT_RT_WARM
    return first;
}

} // namespace pyrit_b200
