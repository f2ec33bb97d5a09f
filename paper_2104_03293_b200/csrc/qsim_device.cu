// qsim_device.cu -- __global__ kernels of the hot path and their launchers.
#include "qsim_device.h"
#include "qsim_kernels.cuh"

#include <algorithm>

namespace qk {

// dynamic shared memory of the standalone reduction: the launch constants only
struct SmemLayout {
    static constexpr size_t total = ((sizeof(CtaShared) + 15) / 16) * 16;
};
static_assert(sizeof(TileRec) == TILE_REC_BYTES, "TileRec size");

// ============================================================ per-tile fields (pre-pass)
// For every tile u of the pass's tile set: h'_i(z_H) (12 tile bits), E_H(z_H) and, for
// phase passes, their phase factors e^{-i gamma (.)}.  It removes all per-tile serial work
// from the streaming kernel.
//
// A warp takes 32 consecutive tiles: their labels differ only in the 5 lowest non-tile bits
// Hlo (tile_base places tile-id bit k at the k-th non-tile position), so the non-tile bits split
// into Hlo (per lane) and Hhi (common to the warp).  The warp computes once, lanes in parallel,
//   A_i = h_i + sum_{j in Hhi} J_ij s_j   (every position i),
//   E_hh = sum_{j in Hhi} s_j (h_j + sum_{k in Hhi, k > j} J_jk s_k),
// and each lane finishes its tile with the Hlo terms:
//   h'_i = A_i + sum_{j in Hlo} J_ij s_j,   E_H = E_hh + sum_{j in Hlo} s_j (A_j + sum_{k in Hlo, k > j} J_jk s_k).
// Every partial sum of dyadic data is exact, so the fields equal field_hprime / eh_term bit for
// bit (the per-thread form below serves shards with fewer than 5 tile-id bits).
constexpr int TF_WARPS = 4;
__global__ void __launch_bounds__(32 * TF_WARPS) tile_fields_kernel(const PassParams P, TileRec *rec) {
    __shared__ double sh[NMAX];
    __shared__ double sJ[NMAX * NMAX];
    __shared__ double sA[TF_WARPS][NMAX];
    const int n = P.n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) sh[i] = P.hp[i];
    for (int i = threadIdx.x; i < n * n; i += blockDim.x) sJ[i] = P.Jp[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // Hlo: the 5 lowest non-tile local positions
    int hlo[5];
    int nlo = 0;
    for (int b = 0; b < P.m && nlo < 5; ++b)
        if (!((P.lmask >> b) & 1ull)) hlo[nlo++] = b;
    if (nlo < 5) {  // fewer than 32 tiles: one thread per tile
        for (u64 u = blockIdx.x * (u64)blockDim.x + threadIdx.x; u < P.ntiles; u += (u64)gridDim.x * blockDim.x) {
            const u64 X = (tile_base(P, u) | P.xglob) ^ P.flip;
            TileRec r;
            double eh = 0.0;
            for (int j = 0; j < n; ++j)
                if (!((P.lmask >> j) & 1ull)) eh += eh_term(sh, sJ, n, j, X, P.lmask);
            r.e[KT] = eh;
#pragma unroll
            for (int i = 0; i < KT; ++i) r.e[i] = field_hprime(sh, sJ, n, P.L[i], X, P.lmask);
#pragma unroll
            for (int i = 0; i <= KT; ++i) r.f[i] = P.phase ? expmi(P.gamma * r.e[i]) : make_double2(1.0, 0.0);
            r.pad = 0.0;
            rec[u] = r;
        }
        return;
    }
    u64 lomask = 0;
#pragma unroll
    for (int k = 0; k < 5; ++k) lomask |= 1ull << hlo[k];
    const u64 himask = ~(P.lmask | lomask) & ((n >= 64) ? ~0ull : ((1ull << n) - 1ull));  // Hhi (incl. global bits)
    double *A = sA[warp];
    for (u64 wb = (blockIdx.x * (u64)TF_WARPS + warp) * 32; wb < P.ntiles; wb += (u64)gridDim.x * TF_WARPS * 32) {
        const u64 Xw = (tile_base(P, wb) | P.xglob) ^ P.flip;  // Hhi spins common to the warp
        double ehh = 0.0;
        for (int i = lane; i < n; i += 32) {
            const double *row = sJ + i * n;
            double a = sh[i], t = 0.0;
            for (int j = 0; j < n; ++j) {
                if (!((himask >> j) & 1ull)) continue;
                const double sj = spin(Xw, j);
                a += row[j] * sj;
                if (j > i) t += row[j] * sj;
            }
            A[i] = a;
            if ((himask >> i) & 1ull) ehh += spin(Xw, i) * (sh[i] + t);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) ehh += __shfl_xor_sync(0xffffffffu, ehh, o);
        __syncwarp();
        const u64 u = wb + lane;
        const u64 X = (tile_base(P, u) | P.xglob) ^ P.flip;
        double slo[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) slo[k] = spin(X, hlo[k]);
        TileRec r;
        double eh = ehh;
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            double t = A[hlo[k]];
#pragma unroll
            for (int k2 = k + 1; k2 < 5; ++k2) t += sJ[hlo[k] * n + hlo[k2]] * slo[k2];
            eh += slo[k] * t;
        }
        r.e[KT] = eh;
#pragma unroll
        for (int i = 0; i < KT; ++i) {
            double e = A[P.L[i]];
#pragma unroll
            for (int k = 0; k < 5; ++k) e += sJ[P.L[i] * n + hlo[k]] * slo[k];
            r.e[i] = e;
        }
#pragma unroll
        for (int i = 0; i <= KT; ++i) r.f[i] = P.phase ? expmi(P.gamma * r.e[i]) : make_double2(1.0, 0.0);
        r.pad = 0.0;
        if (u < P.ntiles) rec[u] = r;
        __syncwarp();
    }
}

// ================================================================== L2 prefetch
// L2 prefetch of tile `ut` (if it exists): its 512 lines of 128 B (tile bits t0..t2 are the
// low physical bits 0..2 in every set), 4 per thread, so HBM keeps streaming while the CTA
// computes on the current tile.
__device__ __forceinline__ void prefetch_next(const PassParams &P, u64 ut, int tid) {
    if (!P.prefetch || ut >= P.ntiles) return;
    const u64 tb = tile_base(P, ut);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int l = tid + q * NTHR;
        u64 off = tb;
#pragma unroll
        for (int b = 0; b < 9; ++b)
            if ((l >> b) & 1) off |= 1ull << P.L[3 + b];
        asm volatile("prefetch.global.L2 [%0];" ::"l"(P.psi + off));
    }
}

// ============================================================ standalone reduction (frame X)
template <typename V>
__global__ void __launch_bounds__(NTHR, 2) reduce_kernel(const PassParams P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    CtaShared &cs = *reinterpret_cast<CtaShared *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = P.n;
    const TileRec *recs = reinterpret_cast<const TileRec *>(P.rec);
    int ft = 0;
#pragma unroll
    for (int i = 0; i < KT; ++i) ft |= (int)((P.flip >> P.L[i]) & 1ull) << i;
    const int tX = Frame<FX>::tthr(lane, warp) ^ ft;
    const int fr = (ft >> Frame<FX>::RB) & 0x1F;
    const ThreadEnergy te = thread_energy<FX>(P.Jp, n, P.L, lane, warp, ft);
    if (tid < NR) cs.eRR[tid] = err_of<FX>(P.Jp, n, P.L, tid ^ fr);
    __syncthreads();
    const u64 offX = thread_offset<FX>(P.L, lane, warp);
    double acc_e = 0.0, acc_n = 0.0;
    V v[NR];
    const V *psi = reinterpret_cast<const V *>(P.psi);
    for (u64 ut = blockIdx.x; ut < P.ntiles; ut += gridDim.x) {
        const u64 tb = tile_base(P, ut);
        if (sizeof(V) == 16) prefetch_next(P, ut + gridDim.x, tid);
        load_tile<FX>(v, psi + tb + offX, P.L);
        accumulate<FX>(v, recs + ut, tX, fr, te, cs.eRR, acc_e, acc_n);
    }
    block_reduce2(cs, acc_e, acc_n, lane, warp, P.part + 2 * blockIdx.x);
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
template <typename V>
__global__ void __launch_bounds__(512) small_kernel(const SmallParams P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2 *st = reinterpret_cast<double2 *>(smem_raw);  // FP64 working copy (FP32 states round on store)
    double *et = reinterpret_cast<double *>(smem_raw + ((size_t)16 << P.n));  // E(z), once per launch
    V *psi = reinterpret_cast<V *>(P.psi);
    __shared__ double sh[KT];
    __shared__ double sJ[KT * KT];
    __shared__ double red[2][16];
    const int n = P.n, dim = 1 << n, tid = threadIdx.x, nt = blockDim.x;
    for (int i = tid; i < n; i += nt) sh[i] = P.hp[i];
    for (int i = tid; i < n * n; i += nt) sJ[i] = P.Jp[i];
    for (int i = tid; i < dim; i += nt) st[i] = P.init ? make_double2(P.a0, 0.0) : dcast(psi[i]);
    __syncthreads();
    for (int z = tid; z < dim; z += nt) et[z] = energy_direct(sh, sJ, n, (u64)z);  // same sum, cached
    for (int k = 0; k < P.p; ++k) {
        const double g = P.ang ? P.ang[k] : P.angv[k], b = P.ang ? P.ang[P.p + k] : P.angv[P.p + k];
        for (int z = tid; z < dim; z += nt) st[z] = cmul(st[z], expmi(g * et[z]));
        double sb, cb;
        sincos(b, &sb, &cb);
        for (int q = 0; q < n; ++q) {
            __syncthreads();
            if (P.gmat) {  // general per-qubit 2x2 (QSDS combined step)
                const double2 *M = P.gmat + ((size_t)k * n + q) * 4;
                const double2 m00 = M[0], m01 = M[1], m10 = M[2], m11 = M[3];
                for (int r = tid; r < dim / 2; r += nt) {
                    const int z0 = ((r >> q) << (q + 1)) | (r & ((1 << q) - 1));
                    const int z1 = z0 | (1 << q);
                    const double2 a = st[z0], bb = st[z1];
                    st[z0] = cmac(m00, a, cmac(m01, bb, make_double2(0.0, 0.0)));
                    st[z1] = cmac(m10, a, cmac(m11, bb, make_double2(0.0, 0.0)));
                }
                continue;
            }
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
        const V av = vcast<V>(st[z]);
        psi[z] = av;
        const double2 a = dcast(av);
        if (P.reduce) {
            const double e = et[z];
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

// ============================================ batched small states (grid scans, config n = 12)
// The QAOA p = 1 landscape of P:369 (and any batch of angle sets) on a state that fits one SM:
// CTA b evaluates point b -- |+>, p layers (phase with the launch's E table, one butterfly sweep per
// qubit), <H_C> -- with the state in shared memory, so 2-3 points run per SM concurrently and a
// 64 x 64 grid is one launch instead of 4096.
__global__ void energy_table_kernel(const double *hp, const double *Jp, int n, double *etab) {
    const int dim = 1 << n;
    for (int z = blockIdx.x * blockDim.x + threadIdx.x; z < dim; z += gridDim.x * blockDim.x)
        etab[z] = energy_direct(hp, Jp, n, (u64)z);
}

__global__ void __launch_bounds__(256) qaoa_batch_kernel(const BatchParams B) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int n = B.n, dim = 1 << n, tid = threadIdx.x, nt = blockDim.x;
    double2 *st = reinterpret_cast<double2 *>(smem_raw);
    double *et = reinterpret_cast<double *>(smem_raw + ((size_t)16 << n));
    __shared__ double red[8];
    for (int z = tid; z < dim; z += nt) {
        st[z] = make_double2(B.a0, 0.0);
        et[z] = B.etab[z];
    }
    __syncthreads();
    const double *gam = B.gamma + (size_t)blockIdx.x * B.p, *bet = B.beta + (size_t)blockIdx.x * B.p;
    for (int k = 0; k < B.p; ++k) {
        const double g = gam[k];
        for (int z = tid; z < dim; z += nt) st[z] = cmul(st[z], expmi(g * et[z]));
        double sb, cb;
        sincos(bet[k], &sb, &cb);
        for (int q = 0; q < n; ++q) {
            __syncthreads();
            for (int r = tid; r < dim / 2; r += nt) {
                const int z0 = ((r >> q) << (q + 1)) | (r & ((1 << q) - 1));
                const int z1 = z0 | (1 << q);
                const double2 a = st[z0], bb = st[z1];
                st[z0] = make_double2(fma(cb, a.x, sb * bb.y), fma(cb, a.y, -sb * bb.x));
                st[z1] = make_double2(fma(sb, a.y, cb * bb.x), fma(-sb, a.x, cb * bb.y));
            }
        }
        __syncthreads();
    }
    double acc = 0.0;
    for (int z = tid; z < dim; z += nt) acc = fma(fma(st[z].x, st[z].x, st[z].y * st[z].y), et[z], acc);
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((tid & 31) == 0) red[tid >> 5] = acc;
    __syncthreads();
    if (tid == 0) {
        double a = 0.0;
        for (int w = 0; w < nt / 32; ++w) a += red[w];
        B.out[blockIdx.x] = a;
    }
}

// ======================================================================== utilities
template <typename V>
__global__ void init_plus_kernel(V *psi, u64 count, double a0) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < count; i += (u64)gridDim.x * blockDim.x)
        psi[i] = vcast<V>(make_double2(a0, 0.0));
}

// logical z -> physical full index via the permutation (pos[q] = physical bit of qubit q)
__device__ __forceinline__ u64 logical_to_physical(u64 z, const GatherParams &G) {
    u64 x = 0;
    for (int q = 0; q < G.n; ++q) x |= ((z >> q) & 1ull) << G.pos[q];
    return x;
}

template <typename V>
__global__ void gather_kernel(const GatherParams G, const V *psi, double2 *out) {
    for (u64 k = blockIdx.x * (u64)blockDim.x + threadIdx.x; k < G.count; k += (u64)gridDim.x * blockDim.x) {
        const u64 z = G.list ? G.list[k] : G.first + k;
        const u64 x = logical_to_physical(z, G) ^ G.flip;
        QSIM_DCHECK((x >> G.n) == 0);
        out[k] = ((x >> G.m) == G.rank) ? dcast(psi[x & ((1ull << G.m) - 1ull)]) : make_double2(0.0, 0.0);
    }
}

// E(z) of the labels [first, first + count) with the hot path's own arithmetic (qsim_energies):
// m > 12: the record of the label's tile of set S (written by tile_fields_kernel, flip 0) and the
// thread / register decomposition of frame Z, summed exactly as accumulate<FZ> sums the reducing
// pass's energies (base, then the register-bit chain r = 0..4, then E_RR); m <= 12: the direct
// sum of small_kernel.  Multi-GPU: the rank owning the label's physical index writes E, the
// others 0 (the engine sums over ranks).
__global__ void energy_dump_kernel(const GatherParams G, const PassParams P, double *out) {
    const TileRec *recs = reinterpret_cast<const TileRec *>(P.rec);
    for (u64 k = blockIdx.x * (u64)blockDim.x + threadIdx.x; k < G.count; k += (u64)gridDim.x * blockDim.x) {
        const u64 x = logical_to_physical(G.first + k, G);
        if ((x >> G.m) != G.rank) {
            out[k] = 0.0;
            continue;
        }
        if (G.m <= KT) {
            out[k] = energy_direct(P.hp, P.Jp, G.n, x);
            continue;
        }
        const u64 xl = x & ((1ull << G.m) - 1ull);
        u64 u = 0;  // tile id: the non-tile bits in ascending order (inverse of tile_base)
        int src = 0;
        for (int sg = 0; sg < P.nseg; ++sg) {
            u |= ((xl >> P.seg_dst[sg]) & ((1ull << P.seg_len[sg]) - 1ull)) << src;
            src += P.seg_len[sg];
        }
        int t = 0;
#pragma unroll
        for (int i = 0; i < KT; ++i) t |= (int)((xl >> P.L[i]) & 1ull) << i;
        constexpr int RB = Frame<FZ>::RB;
        const int tthr = t & ~(0x1F << RB), j = (t >> RB) & 0x1F;
        const ThreadEnergy te = thread_energy<FZ>(P.Jp, G.n, P.L, tthr & 31, tthr >> 10, 0);
        QSIM_DCHECK(u < P.ntiles && t < TILE);
        const TileRec &R = recs[u];
        double e = R.e[KT] + te.eTT;
#pragma unroll
        for (int i = 0; i < KT; ++i) {
            if (i >= RB && i < RB + 5) continue;
            e += ((tthr >> i) & 1) ? R.e[i] : -R.e[i];
        }
#pragma unroll
        for (int r = 0; r < 5; ++r) {
            const double a = R.e[RB + r] + te.w[r];
            e = ((j >> r) & 1) ? e + a : e - a;
        }
        out[k] = e + err_of<FZ>(P.Jp, G.n, P.L, j);
    }
}

// ======================================================================== launchers

cudaError_t setup_kernels() {
    cudaError_t e;
    e = cudaFuncSetAttribute(reduce_kernel<double2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)SmemLayout::total);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(reduce_kernel<float2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)SmemLayout::total);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(qaoa_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 24 * TILE);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(small_kernel<float2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 24 * TILE);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(small_kernel<double2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 24 * TILE);
}

cudaError_t launch_tile_fields(const PassParams &P, void *rec, cudaStream_t s) {
    int grid = (int)std::min<u64>((P.ntiles + 32 * TF_WARPS - 1) / (32 * TF_WARPS), 8192);
    tile_fields_kernel<<<grid, 32 * TF_WARPS, 0, s>>>(P, reinterpret_cast<TileRec *>(rec));
    return cudaGetLastError();
}

cudaError_t launch_reduce(const PassParams &P, int grid, cudaStream_t s) {
    if (P.f32) reduce_kernel<float2><<<grid, NTHR, SmemLayout::total, s>>>(P);
    else reduce_kernel<double2><<<grid, NTHR, SmemLayout::total, s>>>(P);
    return cudaGetLastError();
}

cudaError_t launch_sum_partials(const double *part, int nparts, double *res, cudaStream_t s) {
    sum_partials_kernel<<<1, 32, 0, s>>>(part, nparts, res);
    return cudaGetLastError();
}

cudaError_t launch_small(const SmallParams &P, cudaStream_t s) {
    if (P.f32) small_kernel<float2><<<1, 512, (size_t)24 << P.n, s>>>(P);
    else small_kernel<double2><<<1, 512, (size_t)24 << P.n, s>>>(P);
    return cudaGetLastError();
}

cudaError_t launch_qaoa_batch(const BatchParams &B, double *etab, cudaStream_t s) {
    const int dim = 1 << B.n;
    energy_table_kernel<<<(dim + 255) / 256, 256, 0, s>>>(B.hp, B.Jp, B.n, etab);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    qaoa_batch_kernel<<<B.count, 256, (size_t)24 << B.n, s>>>(B);
    return cudaGetLastError();
}

cudaError_t launch_init_plus(double2 *psi, u64 count, double a0, int grid, cudaStream_t s, int f32) {
    if (f32) init_plus_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<float2 *>(psi), count, a0);
    else init_plus_kernel<<<grid, 256, 0, s>>>(psi, count, a0);
    return cudaGetLastError();
}

cudaError_t launch_gather(const GatherParams &G, const double2 *psi, double2 *out, int grid, cudaStream_t s, int f32) {
    if (f32) gather_kernel<<<grid, 256, 0, s>>>(G, reinterpret_cast<const float2 *>(psi), out);
    else gather_kernel<<<grid, 256, 0, s>>>(G, psi, out);
    return cudaGetLastError();
}

cudaError_t launch_energy_dump(const GatherParams &G, const PassParams &P, double *out, int grid, cudaStream_t s) {
    energy_dump_kernel<<<grid, 256, 0, s>>>(G, P, out);
    return cudaGetLastError();
}

}  // namespace qk
