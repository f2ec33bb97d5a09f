// qsim_tma_f32.cu -- FP32-mode instances (NEXT-4), single and multi GPU (qsim_tma_impl.cuh; dispatched by qsim_tma.cu)
#include "qsim_tma_impl.cuh"

namespace qk {
cudaError_t tma_setup_f32() {
    cudaError_t e = setup_tma_kernels_v<float2, 0>();
    if (e == cudaSuccess) e = setup_tma_kernels_v<float2, 1>();
    return e == cudaSuccess ? setup_tma_kernels_v<float2, 2>() : e;
}
cudaError_t tma_launch_f32(const CUtensorMap &tm, const CUtensorMap &sm, const PassParams &P, int grid, cudaStream_t s) {
    return P.multi == 2 ? launch_tma_pass_v<float2, 2>(tm, sm, P, grid, s)
           : P.multi ? launch_tma_pass_v<float2, 1>(tm, sm, P, grid, s)
                     : launch_tma_pass_v<float2, 0>(tm, sm, P, grid, s);
}
}  // namespace qk
