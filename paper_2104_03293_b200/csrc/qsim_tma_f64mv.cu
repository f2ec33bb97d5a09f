// qsim_tma_f64mv.cu -- FP64 multi-GPU instances (MV 1: top-bit swap schedules, MV 2: low-bit swap) (qsim_tma_impl.cuh; dispatched by qsim_tma.cu)
#include "qsim_tma_impl.cuh"

namespace qk {
cudaError_t tma_setup_f64mv() {
    cudaError_t e = setup_tma_kernels_v<double2, 1>();
    return e == cudaSuccess ? setup_tma_kernels_v<double2, 2>() : e;
}
cudaError_t tma_launch_f64mv(const CUtensorMap &tm, const CUtensorMap &sm, const PassParams &P, int grid, cudaStream_t s) {
    return P.multi == 2 ? launch_tma_pass_v<double2, 2>(tm, sm, P, grid, s) : launch_tma_pass_v<double2, 1>(tm, sm, P, grid, s);
}
}  // namespace qk
