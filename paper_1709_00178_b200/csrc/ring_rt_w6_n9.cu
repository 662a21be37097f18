// The runtime-matrix ring kernel's instances for GF(2^6) in R_{2,9} (see ring_rt.cuh).
#include "ring_rt.cuh"

namespace pyrit_b200 {

cudaError_t launch_ring_rt_w6_n9(const RtArgs& a, const RtLaunch& l) { return rt_detail::launch_wn<6, 9, 0x49u>(a, l); }

// load this geometry's module now (cudaFuncGetAttributes on one instance)
cudaError_t warm_ring_rt_w6_n9() {
    cudaFuncAttributes fa;
    return cudaFuncGetAttributes(&fa, rt_detail::ring_rt_kernel<6, 9, 0x49u, 1, 1, 2, false, false, false>);
}

} // namespace pyrit_b200
