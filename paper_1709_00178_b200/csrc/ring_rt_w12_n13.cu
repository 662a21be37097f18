// The runtime-matrix ring kernel's instances for GF(2^12) in R_{2,13} (see ring_rt.cuh).
#include "ring_rt.cuh"

namespace pyrit_b200 {

cudaError_t launch_ring_rt_w12_n13(const RtArgs& a, const RtLaunch& l) { return rt_detail::launch_wn<12, 13, 0x1FFFu>(a, l); }

// load this geometry's module now (cudaFuncGetAttributes on one instance)
cudaError_t warm_ring_rt_w12_n13() {
    cudaFuncAttributes fa;
    return cudaFuncGetAttributes(&fa, rt_detail::ring_rt_kernel<12, 13, 0x1FFFu, 1, 1, 2, false, false, false>);
}

} // namespace pyrit_b200
