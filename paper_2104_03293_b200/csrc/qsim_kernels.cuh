// qsim_kernels.cuh -- sm_100a device code of the QAOA / AQA hot path
// (arXiv:2104.03293).
//
// One "tile pass" streams the local shard through HBM once: each CTA owns tiles of
// 2^12 amplitudes whose 12 "tile bits" sit at physical bit positions L[0..11]
// (ascending); for every tile it
//   (load)   reads the tile straight into registers (16 amplitudes per thread, frame A,
//            warp lanes on the lowest tile bits -> >= 128-byte coalesced runs),
//   (mix)    applies e^{-i beta sigma^x} to the tile bits in `mix1` as 2x2 butterflies
//            (eq:twocomponentupdates) on register bits, re-distributing the
//            tile between three register frames A -> B -> C through shared memory,
//   (phase)  optionally multiplies psi_z by e^{-i gamma E(z)} (eq:QAOA_state) with E(z)
//            evaluated on the fly by the tile factorisation of SURVEY §8a-a4
//            (no 2^n energy table), then mixes the bits in `mix2` (C -> B -> A),
//   (reduce) optionally accumulates sum |psi|^2 E(z) and sum |psi|^2,
//   (store)  writes the tile back in place (frame C or A, coalesced).
// An `init` pass synthesises |+>^n instead of loading (write-only pass).
//
// Scaled butterflies: e^{-i b X} = cos b (I - i tan b X)  (|cos b| >= |sin b|, form 0)
//                              = -i sin b (X - i(-cot b) ... ) (form 1, see mix_bfly),
// so each butterfly costs 2 FMA per output amplitude; the pass-wide scalar
// kappa^m is folded into the phase factor (or applied once per amplitude).
//
// No code here is shared with oracle/ (the CPU oracle is independent).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "qsim_device.h"

namespace qk {

// ------------------------------------------------------------------------------ helpers
__device__ __forceinline__ double spin(u64 x, int j) { return ((x >> j) & 1ull) ? 1.0 : -1.0; }

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -(a.y * b.y)), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 conjd(double2 a) { return make_double2(a.x, -a.y); }

// e^{-i theta}
__device__ __forceinline__ double2 expmi(double theta) {
    double s, c;
    sincos(theta, &s, &c);
    return make_double2(c, -s);
}

// shared-memory swizzle for 16-byte elements: conflict-free LDS/STS.128 in frames A, B, C
__device__ __forceinline__ int swz(int t) { return t ^ ((t >> 4) & 7); }

// ------------------------------------------------------------------ energy arithmetic
// Tile factorisation of E(z).  With the tile bits L and the other
// bits H (local non-tile + global):
//   E = E_H(z_H) + sum_{i in L} s_i h'_i(z_H) + E_LL(z_L),
//   h'_i(z_H) = h_i + sum_{j in H} J_ij s_j,  E_H = sum_{j in H} s_j (h_j + sum_{k in H, k>j} J_jk s_k).
// Every partial sum of dyadic data is exact, so E is bit-exact independent of order.
// These two functions are the single source of that arithmetic for the pass, reduce
// and probe kernels.
__device__ __forceinline__ double field_hprime(const double *hp, const double *Jp, int n, int pos,
                                               u64 X, u64 lmask) {
    const double *row = Jp + pos * n;
    double acc = hp[pos];
    for (int j = 0; j < n; ++j)
        if (!((lmask >> j) & 1ull)) acc += row[j] * spin(X, j);
    return acc;
}

__device__ __forceinline__ double eh_term(const double *hp, const double *Jp, int n, int j, u64 X,
                                          u64 lmask) {
    const double *row = Jp + j * n;
    double acc = hp[j];
    for (int k = j + 1; k < n; ++k)
        if (!((lmask >> k) & 1ull)) acc += row[k] * spin(X, k);
    return spin(X, j) * acc;
}

// E(X) for one full physical index X, composed from the same pieces (probe kernel).
__device__ double energy_point(const double *hp, const double *Jp, int n, const int *L, int k,
                               u64 lmask, u64 X) {
    double e = 0.0;
    for (int j = 0; j < n; ++j)
        if (!((lmask >> j) & 1ull)) e += eh_term(hp, Jp, n, j, X, lmask);
    for (int i = 0; i < k; ++i) e += spin(X, L[i]) * field_hprime(hp, Jp, n, L[i], X, lmask);
    for (int i = 0; i < k; ++i)
        for (int i2 = i + 1; i2 < k; ++i2)
            e += Jp[L[i] * n + L[i2]] * spin(X, L[i]) * spin(X, L[i2]);
    return e;
}

// ------------------------------------------------------------------------ register frames
// tile index t (12 bits) of register j held by (lane, warp):
//   A: lanes t0..t4, warps t5..t7, regs t8..t11     (load / turning-pass store)
//   B: regs  t0..t3, lanes t4..t8, warps t9..t11
//   C: lanes t0..t3,t8, regs t4..t7, warps t9..t11  (phase, reduce, plain-pass store)
template <int F> struct Frame;
template <> struct Frame<0> {
    static constexpr int RB = 8;
    __device__ static int tthr(int lane, int warp) { return lane | (warp << 5); }
    __host__ __device__ static constexpr int lbit(int b) { return b; }
    __host__ __device__ static constexpr int wbit(int b) { return 5 + b; }
};
template <> struct Frame<1> {
    static constexpr int RB = 0;
    __device__ static int tthr(int lane, int warp) { return (lane << 4) | (warp << 9); }
    __host__ __device__ static constexpr int lbit(int b) { return 4 + b; }
    __host__ __device__ static constexpr int wbit(int b) { return 9 + b; }
};
template <> struct Frame<2> {
    static constexpr int RB = 4;
    __device__ static int tthr(int lane, int warp) {
        return (lane & 15) | ((lane >> 4) << 8) | (warp << 9);
    }
    __host__ __device__ static constexpr int lbit(int b) { return b < 4 ? b : 8; }
    __host__ __device__ static constexpr int wbit(int b) { return 9 + b; }
};

// ------------------------------------------------------------------------- butterflies
// form 0: (a, b) <- (a - i t b, b - i t a)           [e^{-i b X} / cos b, t = tan b]
// form 1: (a, b) <- (b - i t a, a - i t b)           [e^{-i b X} / (-i sin b), t = -cot b]
template <int RBIT, bool FORM1>
__device__ __forceinline__ void bfly(double2 (&v)[NR], double t) {
#pragma unroll
    for (int j = 0; j < NR; ++j) {
        if (j & (1 << RBIT)) continue;
        const double2 a = v[j], b = v[j | (1 << RBIT)];
        const double2 x = make_double2(fma(t, b.y, a.x), fma(-t, b.x, a.y));
        const double2 y = make_double2(fma(t, a.y, b.x), fma(-t, a.x, b.y));
        if (FORM1) {
            v[j] = y;
            v[j | (1 << RBIT)] = x;
        } else {
            v[j] = x;
            v[j | (1 << RBIT)] = y;
        }
    }
}

template <int F>
__device__ __forceinline__ void mix_frame(double2 (&v)[NR], unsigned mask, Mix c) {
    const unsigned m4 = (mask >> Frame<F>::RB) & 0xFu;
    if (!m4) return;
    if (c.form) {
        if (m4 & 1) bfly<0, true>(v, c.t);
        if (m4 & 2) bfly<1, true>(v, c.t);
        if (m4 & 4) bfly<2, true>(v, c.t);
        if (m4 & 8) bfly<3, true>(v, c.t);
    } else {
        if (m4 & 1) bfly<0, false>(v, c.t);
        if (m4 & 2) bfly<1, false>(v, c.t);
        if (m4 & 4) bfly<2, false>(v, c.t);
        if (m4 & 8) bfly<3, false>(v, c.t);
    }
}

// frame change through shared memory (one barrier); every thread writes back exactly
// the elements it read in the previous exchange, so only the single barrier is needed.
template <int F1, int F2>
__device__ __forceinline__ void xch(double2 (&v)[NR], double2 *sm, int lane, int warp) {
    const int t1 = Frame<F1>::tthr(lane, warp);
#pragma unroll
    for (int j = 0; j < NR; ++j) sm[swz(t1 | (j << Frame<F1>::RB))] = v[j];
    __syncthreads();
    const int t2 = Frame<F2>::tthr(lane, warp);
#pragma unroll
    for (int j = 0; j < NR; ++j) v[j] = sm[swz(t2 | (j << Frame<F2>::RB))];
}

// physical element offset of the thread's tile-index bits (all bits except the register bits)
template <int F>
__device__ __forceinline__ u64 thread_offset(const int *L, int lane, int warp) {
    const int t = Frame<F>::tthr(lane, warp);
    u64 off = 0;
#pragma unroll
    for (int b = 0; b < KT; ++b)
        if ((t >> b) & 1) off |= 1ull << L[b];
    return off;
}

__device__ __forceinline__ u64 tile_base(const PassParams &P, u64 u) {
    u64 off = 0;
    int src = 0;
    for (int s = 0; s < P.nseg; ++s) {
        off |= ((u >> src) & ((1ull << P.seg_len[s]) - 1ull)) << P.seg_dst[s];
        src += P.seg_len[s];
    }
    return off;
}

// per-thread, tile-independent energy pieces of frame F (the thread's tile bits T and
// register bits R are fixed for the whole launch):
//   eTT = sum_{i<i' in T} J s_i s_i',  w_r = sum_{i in T} J_{R_r, i} s_i
struct ThreadEnergy {
    double eTT;
    double w[4];
};

template <int F>
__device__ ThreadEnergy thread_energy(const double *Jp, int n, const int *L, int lane, int warp) {
    const int t = Frame<F>::tthr(lane, warp);
    const unsigned rmask = 0xFu << Frame<F>::RB;
    ThreadEnergy te;
    te.eTT = 0.0;
    for (int i = 0; i < KT; ++i) {
        if ((rmask >> i) & 1) continue;
        const double si = ((t >> i) & 1) ? 1.0 : -1.0;
        for (int i2 = i + 1; i2 < KT; ++i2) {
            if ((rmask >> i2) & 1) continue;
            const double si2 = ((t >> i2) & 1) ? 1.0 : -1.0;
            te.eTT += Jp[L[i] * n + L[i2]] * si * si2;
        }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int ir = Frame<F>::RB + r;
        double w = 0.0;
        for (int i = 0; i < KT; ++i) {
            if ((rmask >> i) & 1) continue;
            w += Jp[L[ir] * n + L[i]] * (((t >> i) & 1) ? 1.0 : -1.0);
        }
        te.w[r] = w;
    }
    return te;
}

// E_RR(j) = sum_{r<r'} J_{R_r R_r'} s_r(j) s_r'(j) for the 16 register patterns
template <int F>
__device__ double err_of(const double *Jp, int n, const int *L, int j) {
    double e = 0.0;
    for (int r = 0; r < 4; ++r)
        for (int r2 = r + 1; r2 < 4; ++r2)
            e += Jp[L[Frame<F>::RB + r] * n + L[Frame<F>::RB + r2]] * (((j >> r) & 1) ? 1.0 : -1.0) *
                 (((j >> r2) & 1) ? 1.0 : -1.0);
    return e;
}

// shared per-CTA tables (per tile)
struct TileTables {
    double hL[KT];       // h'_i of the tile bits
    double EH;           // E_H(z_H)
    double2 f[KT + 1];   // e^{-i gamma h'_i}, f[KT] = e^{-i gamma E_H}
    double2 tabL[32];    // phase product over lane bits
    double2 tabW[8];     // phase product over warp bits * Phi_H * scale
    double2 fR[4];       // e^{-i gamma h'_{R_r}}
    double eL[32];       // energy sum over lane bits
    double eW[8];        // E_H + energy sum over warp bits
    double hR[4];        // h' of the register bits
    double2 PRR[16];     // e^{-i gamma E_RR(j)}   (launch constant)
    double eRR[16];      // E_RR(j)                (launch constant)
    double red[2][NTHR / 32];
};

// warp 0: fields of the tile with base X (bits at L are zero) and the frame-F tables
template <int F>
__device__ void tile_tables_warp(TileTables &tt, const double *hp, const double *Jp, int n,
                                 const int *L, u64 lmask, u64 X, int lane, bool do_phase,
                                 double gamma, double2 scale) {
    double t = 0.0;
    for (int j = lane; j < n; j += 32)
        if (!((lmask >> j) & 1ull)) t += eh_term(hp, Jp, n, j, X, lmask);
#pragma unroll
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    double hl = 0.0;
    if (lane < KT) {
        hl = field_hprime(hp, Jp, n, L[lane], X, lmask);
        tt.hL[lane] = hl;
    }
    if (lane == 0) tt.EH = t;
    if (do_phase) {
        if (lane < KT) tt.f[lane] = expmi(gamma * hl);
        if (lane == KT) tt.f[KT] = expmi(gamma * t);
    }
    __syncwarp();
    {   // lane-bit tables
        double e = 0.0;
        double2 ph = make_double2(1.0, 0.0);
#pragma unroll
        for (int b = 0; b < 5; ++b) {
            const int i = Frame<F>::lbit(b);
            const bool up = (lane >> b) & 1;
            e += up ? tt.hL[i] : -tt.hL[i];
            if (do_phase) ph = cmul(ph, up ? tt.f[i] : conjd(tt.f[i]));
        }
        tt.eL[lane] = e;
        if (do_phase) tt.tabL[lane] = ph;
    }
    if (lane < 8) {
        double e = tt.EH;
        double2 ph = do_phase ? cmul(tt.f[KT], scale) : make_double2(1.0, 0.0);
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            const int i = Frame<F>::wbit(b);
            const bool up = (lane >> b) & 1;
            e += up ? tt.hL[i] : -tt.hL[i];
            if (do_phase) ph = cmul(ph, up ? tt.f[i] : conjd(tt.f[i]));
        }
        tt.eW[lane] = e;
        if (do_phase) tt.tabW[lane] = ph;
    }
    if (lane < 4) {
        tt.hR[lane] = tt.hL[Frame<F>::RB + lane];
        if (do_phase) tt.fR[lane] = tt.f[Frame<F>::RB + lane];
    }
}

// multiply v[j] by e^{-i gamma E} for the thread's 16 amplitudes (frame F)
template <int F>
__device__ __forceinline__ void apply_phase(double2 (&v)[NR], const TileTables &tt, int lane,
                                            int warp, double2 uTT, const double2 (&u)[4]) {
    double2 P[NR];
    P[0] = cmul(cmul(tt.tabL[lane], tt.tabW[warp]), uTT);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const double2 g = cmul(tt.fR[r], u[r]);
        const double2 gc = conjd(g);
#pragma unroll
        for (int j = 0; j < (1 << r); ++j) {
            P[j + (1 << r)] = cmul(P[j], g);
            P[j] = cmul(P[j], gc);
        }
    }
#pragma unroll
    for (int j = 0; j < NR; ++j) v[j] = cmul(v[j], cmul(P[j], tt.PRR[j]));
}

// accumulate sum |psi|^2 E and sum |psi|^2 over the thread's 16 amplitudes (frame F)
template <int F>
__device__ __forceinline__ void accumulate(const double2 (&v)[NR], const TileTables &tt, int lane,
                                           int warp, const ThreadEnergy &te, double &acc_e,
                                           double &acc_n) {
    double Q[NR];
    Q[0] = tt.eL[lane] + tt.eW[warp] + te.eTT;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const double a = tt.hR[r] + te.w[r];
#pragma unroll
        for (int j = 0; j < (1 << r); ++j) {
            Q[j + (1 << r)] = Q[j] + a;
            Q[j] = Q[j] - a;
        }
    }
#pragma unroll
    for (int j = 0; j < NR; ++j) {
        const double p = fma(v[j].x, v[j].x, v[j].y * v[j].y);
        acc_e = fma(p, Q[j] + tt.eRR[j], acc_e);
        acc_n += p;
    }
}

__device__ __forceinline__ void block_reduce2(TileTables &tt, double a, double b, int lane, int warp,
                                              double *out) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    __syncthreads();
    if (lane == 0) {
        tt.red[0][warp] = a;
        tt.red[1][warp] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s0 = 0.0, s1 = 0.0;
        for (int w = 0; w < NTHR / 32; ++w) {
            s0 += tt.red[0][w];
            s1 += tt.red[1][w];
        }
        out[0] = s0;
        out[1] = s1;
    }
}

}  // namespace qk
