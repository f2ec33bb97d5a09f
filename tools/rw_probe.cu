// rw_probe.cu -- HBM probe for the run-set access pattern (n = 30, run set {0,1,2}+{16..24}):
// one read + one write of all 2^30 complex128 amplitudes with plain 16-byte loads/stores,
//   A  scattered read, scattered write (in place: the current run passes' pattern)
//   B  scattered read  -> contiguous write (other buffer: the tile lands as 64 KiB)
//   C  contiguous read -> scattered write (other buffer)
//   D  contiguous read, contiguous write (in place: the 12-bit set's pattern, the control)
//   R  scattered read only,  W  scattered write only
// "scattered" = the 4096 amplitudes of a tile are 512 rows of 128 B at a 1 MiB stride (bits
// 16..24); consecutive tiles are the neighbouring 128 B of each row (tile-id bits 3..15, 25..29).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/rw_probe tools/rw_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

typedef unsigned long long u64;
constexpr int N = 30;

__device__ __forceinline__ u64 scat(u64 tile, u64 e) {  // e: 12-bit element of the tile
    const u64 low = e & 7, run = e >> 3;                  // passengers, run bits
    const u64 t_lo = tile & ((1ull << 13) - 1), t_hi = tile >> 13;  // bits 3..15, 25..29
    return low | (t_lo << 3) | (run << 16) | (t_hi << 25);
}
__device__ __forceinline__ u64 cont(u64 tile, u64 e) { return (tile << 12) | e; }

template <int MODE>
__global__ void __launch_bounds__(256) probe(const double2 *__restrict__ in, double2 *__restrict__ out) {
    // each block handles whole tiles, cyclic over blocks; a thread moves 16 elements per tile
    const u64 ntiles = 1ull << (N - 12);
    for (u64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
        double2 v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const u64 e = (u64)threadIdx.x + 256ull * k;
            const u64 ai = (MODE == 0 || MODE == 1 || MODE == 4 || MODE == 5) ? scat(t, e) : cont(t, e);
            if (MODE != 5) v[k] = in[ai];
            else v[k] = make_double2((double)e, 0.0);
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const u64 e = (u64)threadIdx.x + 256ull * k;
            const u64 ao = (MODE == 0 || MODE == 2 || MODE == 5) ? scat(t, e) : cont(t, e);
            if (MODE == 4) {
                if (v[k].x == 12345.678) out[ao] = v[k];  // never true: keeps the load
            } else {
                out[ao] = make_double2(v[k].x * 1.0000001, v[k].y);
            }
        }
    }
}

// relabelling copy of the run slot R1 = {16..24}: tile id ut (bits = input positions 3..15, 25..29
// ascending); the tile goes to positions 0..11, the home bits 3..11 to 16..24.  ROT rotates the
// processing order so that tile-id bit ROT varies fastest (0: input position 3 first = adjacent
// 128 B read rows, output tiles 1 MiB apart; 9: position 12 first = output tiles consecutive)
template <int ROT>
__global__ void __launch_bounds__(256) relabel_copy(const double2 *__restrict__ in, double2 *__restrict__ out) {
    const u64 ntiles = 1ull << (N - 12);
    for (u64 k = blockIdx.x; k < ntiles; k += gridDim.x) {
        const u64 ut = ROT ? (((k << ROT) | (k >> (N - 12 - ROT))) & (ntiles - 1)) : k;
        const u64 home = ut & 511, b12 = (ut >> 9) & 15, b25 = ut >> 13;
        double2 v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const u64 e = (u64)threadIdx.x + 256ull * q;
            v[q] = in[(e & 7) | (home << 3) | (b12 << 12) | ((e >> 3) << 16) | (b25 << 25)];
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const u64 e = (u64)threadIdx.x + 256ull * q;
            out[e | (b12 << 12) | (home << 16) | (b25 << 25)] = make_double2(v[q].x * 1.0000001, v[q].y);
        }
    }
}
template <int ROT>
float run_rl(double2 *a, double2 *b, int grid, int reps) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    relabel_copy<ROT><<<grid, 256>>>(a, b);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) relabel_copy<ROT><<<grid, 256>>>(a, b);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / reps;
}

template <int MODE>
float run(double2 *a, double2 *b, int grid, int reps) {
    double2 *out = (MODE == 1 || MODE == 2) ? b : a;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    probe<MODE><<<grid, 256>>>(a, out);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) probe<MODE><<<grid, 256>>>(a, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / reps;
}

int main() {
    const size_t bytes = (size_t)16 << N;
    double2 *a, *b;
    if (cudaMalloc(&a, bytes) != cudaSuccess || cudaMalloc(&b, bytes) != cudaSuccess) return 1;
    cudaMemset(a, 0, bytes);
    cudaMemset(b, 0, bytes);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const char *names[6] = {"A scat R + scat W (in place)", "B scat R -> cont W", "C cont R -> scat W",
                            "D cont R + cont W (in place)", "R scat read only", "W scat write only"};
    for (int occ : {4, 8}) {
        const int grid = sms * occ;
        float t[6];
        t[0] = run<0>(a, b, grid, 5);
        t[1] = run<1>(a, b, grid, 5);
        t[2] = run<2>(a, b, grid, 5);
        t[3] = run<3>(a, b, grid, 5);
        t[4] = run<4>(a, b, grid, 5);
        t[5] = run<5>(a, b, grid, 5);
        for (int i = 0; i < 6; ++i) {
            const double by = (i >= 4 ? 1.0 : 2.0) * bytes;
            printf("grid %d x 256  %-30s %7.3f ms  %7.1f GB/s\n", grid, names[i], t[i], by / t[i] / 1e6);
        }
        const float r0 = run_rl<0>(a, b, grid, 5), r9 = run_rl<9>(a, b, grid, 5), r13 = run_rl<13>(a, b, grid, 5);
        printf("grid %d x 256  relabel copy, order home-first     %7.3f ms  %7.1f GB/s\n", grid, r0, 2.0 * bytes / r0 / 1e6);
        printf("grid %d x 256  relabel copy, order pos-12-first   %7.3f ms  %7.1f GB/s\n", grid, r9, 2.0 * bytes / r9 / 1e6);
        printf("grid %d x 256  relabel copy, order pos-25-first   %7.3f ms  %7.1f GB/s\n", grid, r13, 2.0 * bytes / r13 / 1e6);
    }
    cudaError_t e = cudaGetLastError();
    printf("%s\n", cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 1;
}
