// qsim_extra.cu -- SURVEY §8(f) NEXT rows built on the hot-path machinery:
//   NEXT-2  <sigma^z_i> of the current state (Fig. 5): one read-only sweep,
//           per-position sums of |psi|^2 s_i folded through the tile structure.
//   NEXT-3  full enumeration of E(z) over all 2^n labels (the paper's t_FE):
//           the tile factorisation of E turns every energy into a few adds
//           of a register tree instead of the O(n^2) sum; minimum and minimisers collected.
#include "qsim_device.h"
#include "qsim_kernels.cuh"

#include <algorithm>

namespace qk {

// ---------------------------------------------------------------------------------- NEXT-2
// per CTA: vec[x] = sum over its tiles of sum_z |psi_z|^2 s_x(z ^ F) for physical bit x
template <typename V>
__global__ void __launch_bounds__(NTHR, 1) spin_kernel(const PassParams P, double *part) {
    __shared__ double red[NTHR / 32][NMAX + KT];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = P.n;
    int ft = 0;
#pragma unroll
    for (int i = 0; i < KT; ++i) ft |= (int)((P.flip >> P.L[i]) & 1ull) << i;
    const int tX = Frame<FX>::tthr(lane, warp) ^ ft;  // flipped thread tile bits
    const int fr = (ft >> Frame<FX>::RB) & 0x1F;
    const u64 offX = thread_offset<FX>(P.L, lane, warp);
    double acc[NMAX];   // non-tile positions
    double acct[KT];    // tile bits
#pragma unroll
    for (int x = 0; x < NMAX; ++x) acc[x] = 0.0;
#pragma unroll
    for (int t = 0; t < KT; ++t) acct[t] = 0.0;
    V v[NR];
    const V *psi = reinterpret_cast<const V *>(P.psi);
    for (u64 ut = blockIdx.x; ut < P.ntiles; ut += gridDim.x) {
        const u64 tb = tile_base(P, ut);
        load_tile<FX>(v, psi + tb + offX, P.L);
        double Pt = 0.0, Sr[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int j = 0; j < NR; ++j) {
            const double2 a = dcast(v[j]);
            const double p = fma(a.x, a.x, a.y * a.y);
            Pt += p;
#pragma unroll
            for (int r = 0; r < 5; ++r) Sr[r] += ((j >> r) & 1) ? p : -p;
        }
        const u64 Xf = (tb | P.xglob) ^ P.flip;
#pragma unroll
        for (int x = 0; x < NMAX; ++x)
            if (x < n && !((P.lmask >> x) & 1ull)) acc[x] += ((Xf >> x) & 1ull) ? Pt : -Pt;
#pragma unroll
        for (int t = 0; t < KT; ++t) {
            if (t >= Frame<FX>::RB) {
                const int r = t - Frame<FX>::RB;
                acct[t] += ((fr >> r) & 1) ? -Sr[r] : Sr[r];
            } else {
                acct[t] += ((tX >> t) & 1) ? Pt : -Pt;
            }
        }
    }
    // block reduction in a fixed order
#pragma unroll
    for (int x = 0; x < NMAX + KT; ++x) {
        double a = x < NMAX ? acc[x] : acct[x - NMAX];
#pragma unroll
        for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) red[warp][x] = a;
    }
    __syncthreads();
    if (tid < n) {
        double s = 0.0;
        for (int w = 0; w < NTHR / 32; ++w) s += red[w][tid];
        for (int t = 0; t < KT; ++t)
            if (P.L[t] == tid)
                for (int w = 0; w < NTHR / 32; ++w) s += red[w][NMAX + t];
        part[(size_t)blockIdx.x * n + tid] = s;
    }
}

__global__ void sum_vec_kernel(const double *part, int nparts, int n, double *out) {
    const int x = threadIdx.x;
    if (x < n) {
        double s = 0.0;
        for (int i = 0; i < nparts; ++i) s += part[(size_t)i * n + x];
        out[x] = s;
    }
}

// ---------------------------------------------------------------------------------- NEXT-3
// Tiles of 4096 consecutive labels z (bits 0..11); frame X gives every thread 32 labels that
// differ in bits 7..11.  Per tile the CTA computes h'_i (i < 12) and E_H with the shared
// energy functions; per thread E_j = base + tree over 5 register bits + E_RR(j).
constexpr int EMAX = 48;  // qsim_enumerate accepts n <= 48 (the state-carrying handles n <= NMAX)
struct EnumCtx {
    double hL[KT];
    double ehp[EMAX];
};

__device__ __forceinline__ void enum_tile(const EnumParams &E, EnumCtx &c, u64 u, const ThreadEnergy &te,
                                          const double *eRR, int tX, double (&Q)[NR]) {
    const int tid = threadIdx.x;
    const u64 X = u << KT;
    const u64 lmask = (1ull << KT) - 1ull;
    if (tid < KT) c.hL[tid] = field_hprime(E.h, E.J, E.n, tid, X, lmask);
    if (tid >= KT && tid < E.n) c.ehp[tid] = eh_term(E.h, E.J, E.n, tid, X, lmask);
    __syncthreads();
    double eb = te.eTT;
    for (int j = KT; j < E.n; ++j) eb += c.ehp[j];
#pragma unroll
    for (int i = 0; i < Frame<FX>::RB; ++i) eb += ((tX >> i) & 1) ? c.hL[i] : -c.hL[i];
    Q[0] = eb;
#pragma unroll
    for (int r = 0; r < 5; ++r) {
        const double a = c.hL[Frame<FX>::RB + r] + te.w[r];
#pragma unroll
        for (int j = 0; j < (1 << r); ++j) {
            Q[j + (1 << r)] = Q[j] + a;
            Q[j] = Q[j] - a;
        }
    }
#pragma unroll
    for (int j = 0; j < NR; ++j) Q[j] += eRR[j];
    __syncthreads();  // hL / ehp reused by the next tile
}

// collect pass: every CTA writes the first max_out minimisers of its tiles in ascending label
// order to out[blockIdx.x * max_out ..] (its tiles ascend, and inside a tile the label order is
// (j, warp, lane) -- register bits 7..11 above the thread bits 0..6 -- which the ballot prefix
// below follows), and the number written to cta_cnt[blockIdx.x].  The host merges the per-CTA
// lists: the global first max_out minimisers are among them.  count += all minimisers.
__global__ void __launch_bounds__(NTHR) enum_kernel(const EnumParams E) {
    __shared__ EnumCtx c;
    __shared__ double eRR[NR];
    __shared__ double red[NTHR / 32];
    __shared__ int wc[NTHR / 32];
    __shared__ int stored;
    __shared__ unsigned long long tot_sh[NTHR / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int L[KT];
#pragma unroll
    for (int i = 0; i < KT; ++i) L[i] = i;
    const ThreadEnergy te = thread_energy<FX>(E.J, E.n, L, lane, warp, 0);
    if (tid < NR) eRR[tid] = err_of<FX>(E.J, E.n, L, tid);
    if (tid == 0) stored = 0;
    __syncthreads();
    const int tX = Frame<FX>::tthr(lane, warp);
    double emin = 1.0e300;
    unsigned long long tot = 0;
    double Q[NR];
    u64 *const out = E.collect ? E.out + (size_t)blockIdx.x * (size_t)E.max_out : nullptr;
    for (u64 u = E.u0 + blockIdx.x; u < E.u1; u += gridDim.x) {
        enum_tile(E, c, u, te, eRR, tX, Q);
        if (E.collect) {
            unsigned mm = 0;
#pragma unroll
            for (int j = 0; j < NR; ++j) mm |= (Q[j] == E.emin) ? (1u << j) : 0u;
            tot += __popc(mm);
            if (!__syncthreads_or(mm != 0u) || stored >= E.max_out) continue;  // block-uniform
            for (int j = 0; j < NR; ++j) {
                const bool f = (mm >> j) & 1u;
                if (!__syncthreads_or(f)) continue;
                const unsigned b = __ballot_sync(0xffffffffu, f);
                if (lane == 0) wc[warp] = __popc(b);
                __syncthreads();
                int before = stored + __popc(b & ((1u << lane) - 1u));
                for (int w = 0; w < warp; ++w) before += wc[w];
                if (f && before < E.max_out) out[before] = (u << KT) | (u64)(tX | (j << Frame<FX>::RB));
                __syncthreads();
                if (tid == 0) {
                    int s = stored;
                    for (int w = 0; w < NTHR / 32; ++w) s += wc[w];
                    stored = s;
                }
                __syncthreads();
                if (stored >= E.max_out) break;
            }
        } else {
#pragma unroll
            for (int j = 0; j < NR; ++j) emin = fmin(emin, Q[j]);
        }
    }
    if (E.collect) {
#pragma unroll
        for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        if (lane == 0) tot_sh[warp] = tot;
        __syncthreads();
        if (tid == 0) {
            unsigned long long t = 0;
            for (int w = 0; w < NTHR / 32; ++w) t += tot_sh[w];
            if (t) atomicAdd(E.count, t);
            E.cta_cnt[blockIdx.x] = (unsigned)min(stored, E.max_out);
        }
    } else {
#pragma unroll
        for (int o = 16; o; o >>= 1) emin = fmin(emin, __shfl_xor_sync(0xffffffffu, emin, o));
        if (lane == 0) red[warp] = emin;
        __syncthreads();
        if (tid == 0) {
            double m = red[0];
            for (int w = 1; w < NTHR / 32; ++w) m = fmin(m, red[w]);
            E.part[blockIdx.x] = m;
        }
    }
}

__global__ void min_partials_kernel(const double *part, int nparts, double *res) {
    if (threadIdx.x == 0) {
        double m = 1.0e300;
        for (int i = 0; i < nparts; ++i) m = fmin(m, part[i]);
        res[0] = m;
    }
}

cudaError_t launch_spin(const PassParams &P, double *part, int grid, cudaStream_t s) {
    if (P.f32) spin_kernel<float2><<<grid, NTHR, 0, s>>>(P, part);
    else spin_kernel<double2><<<grid, NTHR, 0, s>>>(P, part);
    return cudaGetLastError();
}
cudaError_t launch_sum_vec(const double *part, int nparts, int n, double *out, cudaStream_t s) {
    sum_vec_kernel<<<1, 64, 0, s>>>(part, nparts, n, out);
    return cudaGetLastError();
}
cudaError_t launch_enum(const EnumParams &E, int grid, cudaStream_t s) {
    enum_kernel<<<grid, NTHR, 0, s>>>(E);
    return cudaGetLastError();
}
cudaError_t launch_min_partials(const double *part, int nparts, double *res, cudaStream_t s) {
    min_partials_kernel<<<1, 32, 0, s>>>(part, nparts, res);
    return cudaGetLastError();
}

}  // namespace qk
