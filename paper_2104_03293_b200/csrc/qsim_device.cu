// qsim_device.cu -- __global__ kernels of the hot path and their launchers.
#include "qsim_device.h"
#include "qsim_kernels.cuh"

namespace qk {

// dynamic shared memory layout of the pass / reduce kernels
struct SmemLayout {
    static constexpr size_t tile = SM_TILE_BYTES;                 // 64 KiB tile
    static constexpr size_t tables = sizeof(TileTables);
    static constexpr size_t hj = sizeof(double) * (NMAX + NMAX * NMAX);
    static constexpr size_t total = tile + ((tables + 15) / 16) * 16 + hj;
};

__device__ __forceinline__ void load_hj(double *sh, double *sJ, const double *hp, const double *Jp, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) sh[i] = hp[i];
    for (int i = threadIdx.x; i < n * n; i += blockDim.x) sJ[i] = Jp[i];
}

// ================================================================== tile pass kernel
// One HBM sweep of the shard: [init | load] -> mix1 (A,B,C) -> [phase -> mix2 (C,B,A)]
// -> [reduce] -> store.  Grid-stride over tiles; fixed tile->CTA assignment makes the
// reduction deterministic.
__global__ void __launch_bounds__(NTHR, 2) pass_kernel(const PassParams P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2 *sm = reinterpret_cast<double2 *>(smem_raw);
    TileTables &tt = *reinterpret_cast<TileTables *>(smem_raw + SmemLayout::tile);
    double *sh = reinterpret_cast<double *>(smem_raw + SmemLayout::tile +
                                            ((SmemLayout::tables + 15) / 16) * 16);
    double *sJ = sh + NMAX;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = P.n;
    const bool need_e = P.phase || P.reduce;

    load_hj(sh, sJ, P.hp, P.Jp, n);
    __syncthreads();

    // launch-constant energy pieces of frame C
    ThreadEnergy te;
    double2 uTT = make_double2(1.0, 0.0);
    double2 u[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) u[r] = make_double2(1.0, 0.0);
    if (need_e) {
        te = thread_energy<2>(sJ, n, P.L, lane, warp);
        if (P.phase) {
            uTT = expmi(P.gamma * te.eTT);
#pragma unroll
            for (int r = 0; r < 4; ++r) u[r] = expmi(P.gamma * te.w[r]);
        }
        if (tid < 16) {
            const double e = err_of<2>(sJ, n, P.L, tid);
            tt.eRR[tid] = e;
            tt.PRR[tid] = P.phase ? expmi(P.gamma * e) : make_double2(1.0, 0.0);
        }
    }

    const u64 offA = thread_offset<0>(P.L, lane, warp);
    const u64 offC = thread_offset<2>(P.L, lane, warp);
    const u64 sA0 = 1ull << P.L[8], sA1 = 1ull << P.L[9], sA2 = 1ull << P.L[10], sA3 = 1ull << P.L[11];
    const u64 sC0 = 1ull << P.L[4], sC1 = 1ull << P.L[5], sC2 = 1ull << P.L[6], sC3 = 1ull << P.L[7];

    double acc_e = 0.0, acc_n = 0.0;
    double2 v[NR];

    for (u64 ut = blockIdx.x; ut < P.ntiles; ut += gridDim.x) {
        __syncthreads();  // previous tile done with smem tile + tables
        const u64 tb = tile_base(P, ut);
        if (!P.init) {
            const double2 *src = P.psi + tb + offA;
#pragma unroll
            for (int j = 0; j < NR; ++j) {
                const u64 o = ((j & 1) ? sA0 : 0) + ((j & 2) ? sA1 : 0) + ((j & 4) ? sA2 : 0) +
                              ((j & 8) ? sA3 : 0);
                v[j] = __ldcs(src + o);
            }
        }
        if (need_e && warp == 0)
            tile_tables_warp<2>(tt, sh, sJ, n, P.L, P.lmask, tb | P.xglob, lane, P.phase, P.gamma,
                                P.scale);
        if (!P.init) {
            mix_frame<0>(v, P.mix1, P.c1);
            xch<0, 1>(v, sm, lane, warp);
            mix_frame<1>(v, P.mix1, P.c1);
            xch<1, 2>(v, sm, lane, warp);
            mix_frame<2>(v, P.mix1, P.c1);
        } else {
#pragma unroll
            for (int j = 0; j < NR; ++j) v[j] = make_double2(P.a0, 0.0);
            __syncthreads();  // tables visible
        }
        if (P.phase) {
            apply_phase<2>(v, tt, lane, warp, uTT, u);
            mix_frame<2>(v, P.mix2, P.c2);
            xch<2, 1>(v, sm, lane, warp);
            mix_frame<1>(v, P.mix2, P.c2);
            xch<1, 0>(v, sm, lane, warp);
            mix_frame<0>(v, P.mix2, P.c2);
            double2 *dst = P.psi + tb + offA;
#pragma unroll
            for (int j = 0; j < NR; ++j) {
                const u64 o = ((j & 1) ? sA0 : 0) + ((j & 2) ? sA1 : 0) + ((j & 4) ? sA2 : 0) +
                              ((j & 8) ? sA3 : 0);
                __stcs(dst + o, v[j]);
            }
        } else {
            if (P.scale.x != 1.0 || P.scale.y != 0.0) {
#pragma unroll
                for (int j = 0; j < NR; ++j) v[j] = cmul(v[j], P.scale);
            }
            if (P.reduce) accumulate<2>(v, tt, lane, warp, te, acc_e, acc_n);
            double2 *dst = P.psi + tb + offC;
#pragma unroll
            for (int j = 0; j < NR; ++j) {
                const u64 o = ((j & 1) ? sC0 : 0) + ((j & 2) ? sC1 : 0) + ((j & 4) ? sC2 : 0) +
                              ((j & 8) ? sC3 : 0);
                __stcs(dst + o, v[j]);
            }
        }
    }
    if (P.reduce) block_reduce2(tt, acc_e, acc_n, lane, warp, P.part + 2 * blockIdx.x);
}

// ============================================================ standalone reduction (frame A)
__global__ void __launch_bounds__(NTHR, 2) reduce_kernel(const PassParams P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TileTables &tt = *reinterpret_cast<TileTables *>(smem_raw + SmemLayout::tile);
    double *sh = reinterpret_cast<double *>(smem_raw + SmemLayout::tile +
                                            ((SmemLayout::tables + 15) / 16) * 16);
    double *sJ = sh + NMAX;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = P.n;
    load_hj(sh, sJ, P.hp, P.Jp, n);
    __syncthreads();
    const ThreadEnergy te = thread_energy<0>(sJ, n, P.L, lane, warp);
    if (tid < 16) tt.eRR[tid] = err_of<0>(sJ, n, P.L, tid);
    const u64 offA = thread_offset<0>(P.L, lane, warp);
    const u64 sA0 = 1ull << P.L[8], sA1 = 1ull << P.L[9], sA2 = 1ull << P.L[10], sA3 = 1ull << P.L[11];
    double acc_e = 0.0, acc_n = 0.0;
    double2 v[NR];
    for (u64 ut = blockIdx.x; ut < P.ntiles; ut += gridDim.x) {
        __syncthreads();
        const u64 tb = tile_base(P, ut);
        const double2 *src = P.psi + tb + offA;
#pragma unroll
        for (int j = 0; j < NR; ++j) {
            const u64 o = ((j & 1) ? sA0 : 0) + ((j & 2) ? sA1 : 0) + ((j & 4) ? sA2 : 0) +
                          ((j & 8) ? sA3 : 0);
            v[j] = __ldcs(src + o);
        }
        if (warp == 0)
            tile_tables_warp<0>(tt, sh, sJ, n, P.L, P.lmask, tb | P.xglob, lane, false, 0.0,
                                make_double2(1.0, 0.0));
        __syncthreads();
        accumulate<0>(v, tt, lane, warp, te, acc_e, acc_n);
    }
    block_reduce2(tt, acc_e, acc_n, lane, warp, P.part + 2 * blockIdx.x);
}

// sum the per-CTA partials in a fixed order
__global__ void sum_partials_kernel(const double *part, int nparts, double *res) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int i = 0; i < nparts; ++i) {
            a += part[2 * i];
            b += part[2 * i + 1];
        }
        res[0] = a;
        res[1] = b;
    }
}

// ====================================================== small states (m <= 12, one CTA)
// The whole state lives in shared memory; all p layers run in one launch (config n=12
// is launch-bound).  Phase: E(z) summed directly (exact for dyadic data),
// then sincos; mixer: one butterfly sweep per qubit (eq:twocomponentupdates).
__global__ void __launch_bounds__(512) small_kernel(const SmallParams P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2 *st = reinterpret_cast<double2 *>(smem_raw);
    __shared__ double sh[KT];
    __shared__ double sJ[KT * KT];
    __shared__ double red[2][16];
    const int n = P.n, dim = 1 << n, tid = threadIdx.x, nt = blockDim.x;
    for (int i = tid; i < n; i += nt) sh[i] = P.hp[i];
    for (int i = tid; i < n * n; i += nt) sJ[i] = P.Jp[i];
    for (int i = tid; i < dim; i += nt) st[i] = P.init ? make_double2(P.a0, 0.0) : P.psi[i];
    __syncthreads();
    for (int k = 0; k < P.p; ++k) {
        const double g = P.ang[k], b = P.ang[P.p + k];
        for (int z = tid; z < dim; z += nt) {
            double e = 0.0;
            for (int i = 0; i < n; ++i) {
                const double si = ((z >> i) & 1) ? 1.0 : -1.0;
                e += sh[i] * si;
                for (int j = i + 1; j < n; ++j) e += sJ[i * n + j] * si * (((z >> j) & 1) ? 1.0 : -1.0);
            }
            st[z] = cmul(st[z], expmi(g * e));
        }
        double sb, cb;
        sincos(b, &sb, &cb);
        for (int q = 0; q < n; ++q) {
            __syncthreads();
            for (int r = tid; r < dim / 2; r += nt) {
                const int z0 = ((r >> q) << (q + 1)) | (r & ((1 << q) - 1));
                const int z1 = z0 | (1 << q);
                const double2 a = st[z0], bb = st[z1];
                // a' = c a - i s b ; b' = -i s a + c b
                st[z0] = make_double2(fma(cb, a.x, sb * bb.y), fma(cb, a.y, -sb * bb.x));
                st[z1] = make_double2(fma(sb, a.y, cb * bb.x), fma(-sb, a.x, cb * bb.y));
            }
        }
        __syncthreads();
    }
    double acc_e = 0.0, acc_n = 0.0;
    for (int z = tid; z < dim; z += nt) {
        const double2 a = st[z];
        P.psi[z] = a;
        if (P.reduce) {
            double e = 0.0;
            for (int i = 0; i < n; ++i) {
                const double si = ((z >> i) & 1) ? 1.0 : -1.0;
                e += sh[i] * si;
                for (int j = i + 1; j < n; ++j) e += sJ[i * n + j] * si * (((z >> j) & 1) ? 1.0 : -1.0);
            }
            const double pz = fma(a.x, a.x, a.y * a.y);
            acc_e = fma(pz, e, acc_e);
            acc_n += pz;
        }
    }
    if (P.reduce) {
        const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            acc_e += __shfl_xor_sync(0xffffffffu, acc_e, o);
            acc_n += __shfl_xor_sync(0xffffffffu, acc_n, o);
        }
        if (lane == 0) {
            red[0][warp] = acc_e;
            red[1][warp] = acc_n;
        }
        __syncthreads();
        if (tid == 0) {
            double a = 0.0, b = 0.0;
            for (int w = 0; w < nt / 32; ++w) {
                a += red[0][w];
                b += red[1][w];
            }
            P.res[0] = a;
            P.res[1] = b;
        }
    }
}

// ======================================================================== utilities
__global__ void init_plus_kernel(double2 *psi, u64 count, double a0) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < count; i += (u64)gridDim.x * blockDim.x)
        psi[i] = make_double2(a0, 0.0);
}

// logical z -> physical full index via the permutation (pos[q] = physical bit of qubit q)
__device__ __forceinline__ u64 logical_to_physical(u64 z, const GatherParams &G) {
    u64 x = 0;
    for (int q = 0; q < G.n; ++q) x |= ((z >> q) & 1ull) << G.pos[q];
    return x;
}

__global__ void gather_kernel(const GatherParams G, const double2 *psi, double2 *out) {
    for (u64 k = blockIdx.x * (u64)blockDim.x + threadIdx.x; k < G.count; k += (u64)gridDim.x * blockDim.x) {
        const u64 z = G.list ? G.list[k] : G.first + k;
        const u64 x = logical_to_physical(z, G);
        out[k] = ((x >> G.m) == G.rank) ? psi[x & ((1ull << G.m) - 1ull)] : make_double2(0.0, 0.0);
    }
}

__global__ void energy_probe_kernel(const GatherParams G, const double *hp, const double *Jp,
                                    const ProbeSet S, double *out) {
    for (u64 k = blockIdx.x * (u64)blockDim.x + threadIdx.x; k < G.count; k += (u64)gridDim.x * blockDim.x) {
        const u64 x = logical_to_physical(G.first + k, G);
        out[k] = energy_point(hp, Jp, G.n, S.L, S.k, S.lmask, x);
    }
}

// ======================================================================== launchers
size_t pass_smem_bytes() { return SmemLayout::total; }

cudaError_t setup_kernels() {
    cudaError_t e = cudaFuncSetAttribute(pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)SmemLayout::total);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(reduce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)SmemLayout::total);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * TILE);
}

cudaError_t launch_pass(const PassParams &P, int grid, cudaStream_t s) {
    pass_kernel<<<grid, NTHR, SmemLayout::total, s>>>(P);
    return cudaGetLastError();
}

cudaError_t launch_reduce(const PassParams &P, int grid, cudaStream_t s) {
    reduce_kernel<<<grid, NTHR, SmemLayout::total, s>>>(P);
    return cudaGetLastError();
}

cudaError_t launch_sum_partials(const double *part, int nparts, double *res, cudaStream_t s) {
    sum_partials_kernel<<<1, 32, 0, s>>>(part, nparts, res);
    return cudaGetLastError();
}

cudaError_t launch_small(const SmallParams &P, cudaStream_t s) {
    small_kernel<<<1, 512, (size_t)16 << P.n, s>>>(P);
    return cudaGetLastError();
}

cudaError_t launch_init_plus(double2 *psi, u64 count, double a0, int grid, cudaStream_t s) {
    init_plus_kernel<<<grid, 256, 0, s>>>(psi, count, a0);
    return cudaGetLastError();
}

cudaError_t launch_gather(const GatherParams &G, const double2 *psi, double2 *out, int grid, cudaStream_t s) {
    gather_kernel<<<grid, 256, 0, s>>>(G, psi, out);
    return cudaGetLastError();
}

cudaError_t launch_energy_probe(const GatherParams &G, const double *hp, const double *Jp, const ProbeSet &S,
                                double *out, int grid, cudaStream_t s) {
    energy_probe_kernel<<<grid, 256, 0, s>>>(G, hp, Jp, S, out);
    return cudaGetLastError();
}

}  // namespace qk
