// qsim_tma_pw.cu -- the per-warp turning-run kernels (qsim_tma_impl.cuh; dispatched by qsim_tma.cu)
#include "qsim_tma_impl.cuh"

namespace qk {

// the per-warp turning kernels: attributes and launch (P.pw = 1 | M1 << 2 | NP << 4)
static cudaError_t setup_pw_kernels() {
    cudaError_t e = cudaSuccess;
    for (auto k : {tma_turn_pw_kernel<3, 0>, tma_turn_pw_kernel<4, 0>, tma_turn_pw_kernel<5, 0>, tma_turn_pw_kernel<6, 0>,
                   tma_turn_pw_kernel<7, 0>, tma_turn_pw_kernel<8, 0>, tma_turn_pw_kernel<9, 0>, tma_turn_pw_kernel<10, 0>,
                   tma_turn_pw_kernel<11, 0>, tma_turn_pw_kernel<5, 1>, tma_turn_pw_kernel<5, 2>, tma_turn_pw_kernel<5, 3>})
        if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PwSmem::total);
    return e;
}
static cudaError_t launch_pw(const CUtensorMap &tm, const PassParams &P, int grid, cudaStream_t s) {
    if (P.f32 || P.mv || P.multi == 2 || P.kind != K_TURN_RUN || P.gmix || P.reduce) return cudaErrorInvalidValue;
    const int np = (P.pw >> 4) & 15, m1 = (P.pw >> 2) & 3;
    const size_t sh = PwSmem::total;
    const dim3 b(TMA_NG * 128);
    switch (np * 4 + m1) {
        case 12: tma_turn_pw_kernel<3, 0><<<grid, b, sh, s>>>(tm, P); break;
        case 16: tma_turn_pw_kernel<4, 0><<<grid, b, sh, s>>>(tm, P); break;
        case 20: tma_turn_pw_kernel<5, 0><<<grid, b, sh, s>>>(tm, P); break;
        case 21: tma_turn_pw_kernel<5, 1><<<grid, b, sh, s>>>(tm, P); break;
        case 22: tma_turn_pw_kernel<5, 2><<<grid, b, sh, s>>>(tm, P); break;
        case 23: tma_turn_pw_kernel<5, 3><<<grid, b, sh, s>>>(tm, P); break;
        case 24: tma_turn_pw_kernel<6, 0><<<grid, b, sh, s>>>(tm, P); break;
        case 28: tma_turn_pw_kernel<7, 0><<<grid, b, sh, s>>>(tm, P); break;
        case 32: tma_turn_pw_kernel<8, 0><<<grid, b, sh, s>>>(tm, P); break;
        case 36: tma_turn_pw_kernel<9, 0><<<grid, b, sh, s>>>(tm, P); break;
        case 40: tma_turn_pw_kernel<10, 0><<<grid, b, sh, s>>>(tm, P); break;
        case 44: tma_turn_pw_kernel<11, 0><<<grid, b, sh, s>>>(tm, P); break;
        default: return cudaErrorInvalidValue;  // arrivals-only mix1 occurs on 7-bit runs (>= 4 sets) only
    }
    return cudaGetLastError();
}

cudaError_t tma_setup_pw() { return setup_pw_kernels(); }
cudaError_t tma_launch_pw(const CUtensorMap &tm, const PassParams &P, int grid, cudaStream_t s) {
    return launch_pw(tm, P, grid, s);
}
}  // namespace qk
