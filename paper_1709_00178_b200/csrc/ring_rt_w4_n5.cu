// The runtime-matrix ring kernel's instances for GF(2^4) in R_{2,5} (see ring_rt.cuh).
#include "ring_rt.cuh"

namespace pyrit_b200 {

cudaError_t launch_ring_rt_w4_n5(const RtArgs& a, const RtLaunch& l) { return rt_detail::launch_wn<4, 5, 0x1Fu>(a, l); }

// load this geometry's module now (cudaFuncGetAttributes on one instance)
cudaError_t warm_ring_rt_w4_n5() {
    cudaFuncAttributes fa;
    return cudaFuncGetAttributes(&fa, rt_detail::ring_rt_kernel<4, 5, 0x1Fu, 1, 1, 2, false, false, false>);
}

} // namespace pyrit_b200
