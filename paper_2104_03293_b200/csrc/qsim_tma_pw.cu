// qsim_tma_pw.cu -- the per-warp turning-run kernels (qsim_tma_impl.cuh; dispatched by qsim_tma.cu)
#include "qsim_tma_impl.cuh"

namespace qk {

// the per-warp turning kernels: attributes and launch (P.pw = 1 | (NP == 5) << 1 | M1 << 2)
static cudaError_t setup_pw_kernels() {
    cudaError_t e = cudaSuccess;
    for (auto k : {tma_turn_pw_kernel<3, 0>, tma_turn_pw_kernel<5, 0>, tma_turn_pw_kernel<5, 1>, tma_turn_pw_kernel<5, 2>,
                   tma_turn_pw_kernel<5, 3>})
        if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PwSmem::total);
    return e;
}
static cudaError_t launch_pw(const CUtensorMap &tm, const PassParams &P, int grid, cudaStream_t s) {
    if (P.f32 || P.mv || P.multi == 2 || P.kind != K_TURN_RUN || P.gmix || P.reduce) return cudaErrorInvalidValue;
    const int np5 = (P.pw >> 1) & 1, m1 = (P.pw >> 2) & 3;
    const size_t sh = PwSmem::total;
    const dim3 b(TMA_NG * 128);
    switch (np5 * 4 + m1) {
        case 0: tma_turn_pw_kernel<3, 0><<<grid, b, sh, s>>>(tm, P); break;
        case 4: tma_turn_pw_kernel<5, 0><<<grid, b, sh, s>>>(tm, P); break;
        case 5: tma_turn_pw_kernel<5, 1><<<grid, b, sh, s>>>(tm, P); break;
        case 6: tma_turn_pw_kernel<5, 2><<<grid, b, sh, s>>>(tm, P); break;
        case 7: tma_turn_pw_kernel<5, 3><<<grid, b, sh, s>>>(tm, P); break;
        default: return cudaErrorInvalidValue;  // 9-bit runs only occur with three sets (no arrivals-only mix1)
    }
    return cudaGetLastError();
}

cudaError_t tma_setup_pw() { return setup_pw_kernels(); }
cudaError_t tma_launch_pw(const CUtensorMap &tm, const PassParams &P, int grid, cudaStream_t s) {
    return launch_pw(tm, P, grid, s);
}
}  // namespace qk
