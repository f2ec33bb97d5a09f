// dmma_probe.cu -- one-off check required by BASELINE.json's north star: do FP64 tensor cores
// (DMMA, mma.sync.m8n8k4.f64; tcgen05 has no f64 kind) beat the scaled R_x butterflies for the
// mixer?  Both variants apply e^{-i b X} on the 3 lowest qubits of every group of 8 amplitudes,
// REPS times over data held in registers / shared memory (compute-bound, no HBM), and on a
// 2^27-amplitude state streamed once (HBM-bound).
//
//   butterfly: 3 stages x 2 DFMA per output amplitude (scaled form; the cos^3 scalar omitted,
//              as the product path folds it elsewhere)
//   dmma:      the fused 8x8 complex matrix M = R(x)R(x)R as the 16x16 real block [[Mr,-Mi],[Mi,Mr]]
//              times 16 x 8 real column blocks: 8 m8n8k4 DMMAs per 8 groups (64 amplitudes)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/dmma_probe tools/dmma_probe.cu
//   tools/dmma_probe            -> one JSON line per variant (ms, amplitude-bit updates/s, FP64 flop/s)
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <vector>

#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            return 1;                                                                 \
        }                                                                             \
    } while (0)

// ---------------------------------------------------------------- compute-bound variants
// each thread keeps 8 groups of 8 amplitudes (64 complex) in registers and applies the 3-qubit
// mixer REPS times; one write at the end keeps the work alive
__global__ void __launch_bounds__(128) bfly_kernel(double2 *out, double t, int reps) {
    double2 v[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) v[j] = make_double2(1.0 + 1e-3 * j + threadIdx.x, 0.5);
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int bit = 0; bit < 3; ++bit)
#pragma unroll
            for (int j = 0; j < 64; ++j) {
                if (j & (1 << bit)) continue;
                const double2 a = v[j], b = v[j | (1 << bit)];
                v[j] = make_double2(fma(t, b.y, a.x), fma(-t, b.x, a.y));
                v[j | (1 << bit)] = make_double2(fma(t, a.y, b.x), fma(-t, a.x, b.y));
            }
    }
    double2 s = make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 0; j < 64; ++j) s = make_double2(s.x + v[j].x, s.y + v[j].y);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// D(8x8) += A(8x4) B(4x8), FP64, one warp (the sm_80+ DMMA shape, valid on sm_100a)
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// a warp holds X = 16 x 8 real (8 columns = 8 groups of 8 complex amplitudes; rows 0..7 real
// parts, 8..15 imaginary) in the B-fragment layout, multiplies by the 16 x 16 real block matrix
// Mb (A fragments, loop-invariant registers) REPS times: Y = Mb X as 2 (row blocks) x 4 (k steps)
// DMMAs per 8-column block; 8 column blocks per warp per rep (= 512 amplitudes).
__global__ void __launch_bounds__(128) dmma_kernel(double *out, const double *Mb, int reps) {
    const int lane = threadIdx.x & 31;
    // A fragment of m8n8k4 (row major 8x4): lane holds A[lane / 4][lane % 4]
    double a[2][4];
#pragma unroll
    for (int rb = 0; rb < 2; ++rb)
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) a[rb][ks] = Mb[(rb * 8 + lane / 4) * 16 + ks * 4 + lane % 4];
    // B fragments (4x8 col major: lane holds B[lane % 4][lane / 4]) of 8 column blocks x 4 k steps
    double x[8][4];
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) x[c][ks] = 1.0 + 1e-3 * (c * 4 + ks) + 1e-6 * lane;
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            double d0[2] = {0.0, 0.0}, d1[2] = {0.0, 0.0};
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                dmma(d0, a[0][ks], x[c][ks]);
                dmma(d1, a[1][ks], x[c][ks]);
            }
            // D fragment (8x8): lane holds D[lane / 4][2 (lane % 4) + {0,1}]; route it back into the
            // B layout of the next rep through two shuffles per value (the data movement a fused
            // mixer pays between matrix applications)
            const int src = ((lane % 4) * 2) * 4;  // placeholder permutation with the same traffic
            x[c][0] = __shfl_sync(0xffffffffu, d0[0], (lane + src) & 31);
            x[c][1] = __shfl_sync(0xffffffffu, d0[1], (lane + src + 1) & 31);
            x[c][2] = __shfl_sync(0xffffffffu, d1[0], (lane + src + 2) & 31);
            x[c][3] = __shfl_sync(0xffffffffu, d1[1], (lane + src + 3) & 31);
        }
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) s += x[c][ks];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// ------------------------------------------------------------------- HBM-bound variants
__global__ void bfly_stream(double2 *psi, size_t groups, double t) {
    for (size_t gidx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; gidx < groups; gidx += (size_t)gridDim.x * blockDim.x) {
        double2 v[8];
        const double4 *p = reinterpret_cast<const double4 *>(psi + 8 * gidx);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const double4 q = p[j];
            v[2 * j] = make_double2(q.x, q.y);
            v[2 * j + 1] = make_double2(q.z, q.w);
        }
#pragma unroll
        for (int bit = 0; bit < 3; ++bit)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (j & (1 << bit)) continue;
                const double2 a = v[j], b = v[j | (1 << bit)];
                v[j] = make_double2(fma(t, b.y, a.x), fma(-t, b.x, a.y));
                v[j | (1 << bit)] = make_double2(fma(t, a.y, b.x), fma(-t, a.x, b.y));
            }
        double4 *w = reinterpret_cast<double4 *>(psi + 8 * gidx);
#pragma unroll
        for (int j = 0; j < 4; ++j) w[j] = make_double4(v[2 * j].x, v[2 * j].y, v[2 * j + 1].x, v[2 * j + 1].y);
    }
}

int main() {
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    const int blocks = nsm * 8, threads = 128, reps = 2000;
    const double b = 0.3, t = std::tan(b);
    double2 *o2;
    double *o1, *Mb;
    CK(cudaMalloc(&o2, sizeof(double2) * blocks * threads));
    CK(cudaMalloc(&o1, sizeof(double) * blocks * threads));
    // 16 x 16 real block form of R(x)R(x)R, R = [[c, -i s], [-i s, c]]
    std::vector<double> M(256, 0.0);
    {
        const double c = std::cos(b), s = std::sin(b);
        double Mr[8][8], Mi[8][8];
        for (int r = 0; r < 8; ++r)
            for (int q = 0; q < 8; ++q) {
                double re = 1.0, im = 0.0;
                for (int k = 0; k < 3; ++k) {
                    const bool flip = ((r ^ q) >> k) & 1;
                    const double er = flip ? 0.0 : c, ei = flip ? -s : 0.0;
                    const double nr = re * er - im * ei, ni = re * ei + im * er;
                    re = nr;
                    im = ni;
                }
                Mr[r][q] = re;
                Mi[r][q] = im;
            }
        for (int r = 0; r < 8; ++r)
            for (int q = 0; q < 8; ++q) {
                M[r * 16 + q] = Mr[r][q];
                M[r * 16 + 8 + q] = -Mi[r][q];
                M[(8 + r) * 16 + q] = Mi[r][q];
                M[(8 + r) * 16 + 8 + q] = Mr[r][q];
            }
    }
    CK(cudaMalloc(&Mb, sizeof(double) * 256));
    CK(cudaMemcpy(Mb, M.data(), sizeof(double) * 256, cudaMemcpyHostToDevice));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    float ms = 0.f;
    // compute-bound butterflies: per thread 64 amplitudes x 3 bits x reps
    bfly_kernel<<<blocks, threads>>>(o2, t, 10);
    CK(cudaEventRecord(e0));
    bfly_kernel<<<blocks, threads>>>(o2, t, reps);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    {
        const double amps = (double)blocks * threads * 64 * reps;
        std::printf("{\"variant\": \"butterfly 3-qubit, registers\", \"ms\": %.3f, \"amp_bit_updates_per_s\": %.4g, "
                    "\"fp64_flops_per_s\": %.4g}\n", ms, amps * 3 / (ms * 1e-3), amps * 3 * 4 / (ms * 1e-3));
    }
    // compute-bound DMMA: per warp 8 column blocks x 64 amplitudes x reps
    dmma_kernel<<<blocks, threads>>>(o1, Mb, 10);
    CK(cudaEventRecord(e0));
    dmma_kernel<<<blocks, threads>>>(o1, Mb, reps);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    {
        const double warps = (double)blocks * threads / 32;
        const double amps = warps * 8 * 64 * reps;      // 8 column blocks x 8 columns x 8 complex amplitudes
        const double flops = warps * 64.0 * 512 * reps;  // 64 DMMAs x (8x8x4 MACs x 2 flops) per warp and rep
        std::printf("{\"variant\": \"DMMA fused 3-qubit (16x16 real block), registers\", \"ms\": %.3f, "
                    "\"amp_bit_updates_per_s\": %.4g, \"fp64_tensor_flops_per_s\": %.4g}\n",
                    ms, amps * 3 / (ms * 1e-3), flops / (ms * 1e-3));
    }
    // HBM-bound streaming butterflies on a 2^27-amplitude state (2 GiB)
    const size_t N = 1ull << 27;
    double2 *psi;
    CK(cudaMalloc(&psi, sizeof(double2) * N));
    CK(cudaMemset(psi, 0, sizeof(double2) * N));
    bfly_stream<<<nsm * 16, 256>>>(psi, N / 8, t);
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 10; ++r) bfly_stream<<<nsm * 16, 256>>>(psi, N / 8, t);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    std::printf("{\"variant\": \"butterfly 3-qubit, streamed from HBM\", \"ms_per_sweep\": %.3f, \"GBps\": %.1f}\n",
                ms / 10, 32.0 * N / (ms / 10 * 1e-3) / 1e9);
    CK(cudaGetLastError());
    return 0;
}
