// qsim_tma.cu -- dispatch of the TMA tile-pass kernels (qsim_tma_impl.cuh) to the translation
// units that hold their instances (compiled in parallel).
#include <cuda.h>

#include "qsim_device.h"
#include "qsim_tma_impl.cuh"

namespace qk {

cudaError_t tma_setup_f64();
cudaError_t tma_setup_f64mv();
cudaError_t tma_setup_f32();
cudaError_t tma_setup_pw();
cudaError_t tma_launch_f64(const CUtensorMap &tm, const CUtensorMap &sm, const PassParams &P, int grid, cudaStream_t s);
cudaError_t tma_launch_f64mv(const CUtensorMap &tm, const CUtensorMap &sm, const PassParams &P, int grid, cudaStream_t s);
cudaError_t tma_launch_f32(const CUtensorMap &tm, const CUtensorMap &sm, const PassParams &P, int grid, cudaStream_t s);
cudaError_t tma_launch_pw(const CUtensorMap &tm, const PassParams &P, int grid, cudaStream_t s);

size_t tma_smem_bytes() { return TmaSmem::total; }

cudaError_t setup_tma_kernels() {
    cudaError_t e = tma_setup_pw();
    if (e == cudaSuccess) e = tma_setup_f64();
    if (e == cudaSuccess) e = tma_setup_f64mv();
    if (e == cudaSuccess) e = tma_setup_f32();
    return e;
}

// multi-GPU handles (P.multi) launch the MV instances for every pass: 1 = top-bit swap
// schedules, 2 = the low-bit swap schedule (run frame V); P.pw selects a per-warp turning kernel
cudaError_t launch_tma_pass(const CUtensorMap &tm, const CUtensorMap &sm, const PassParams &P, int grid,
                            cudaStream_t s) {
    if (P.pw) return tma_launch_pw(tm, P, grid, s);  // tm: the SWIZZLE_128B map of the run set (in place)
    if (P.f32) return tma_launch_f32(tm, sm, P, grid, s);
    return P.multi ? tma_launch_f64mv(tm, sm, P, grid, s) : tma_launch_f64(tm, sm, P, grid, s);
}

}  // namespace qk
