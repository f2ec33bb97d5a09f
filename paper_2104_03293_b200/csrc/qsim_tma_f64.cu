// qsim_tma_f64.cu -- FP64 single-GPU instances of the tile-pass kernels (qsim_tma_impl.cuh; dispatched by qsim_tma.cu)
#include "qsim_tma_impl.cuh"

namespace qk {
cudaError_t tma_setup_f64() { return setup_tma_kernels_v<double2, 0>(); }
cudaError_t tma_launch_f64(const CUtensorMap &tm, const CUtensorMap &sm, const PassParams &P, int grid, cudaStream_t s) {
    return launch_tma_pass_v<double2, 0>(tm, sm, P, grid, s);
}
}  // namespace qk
