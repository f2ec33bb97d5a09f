// qsim_kernels.cuh -- sm_100a device code of the QAOA / AQA hot path
// (arXiv:2104.03293).
//
// One "tile pass" streams the local shard through HBM once.  A CTA of 128 threads owns
// one tile of 2^12 amplitudes at a time (32 per thread, held in registers); the tile's
// 12 "tile bits" t0..t11 sit at physical bit positions L[0..11] (ascending).  Per tile:
//   (load)   straight into registers, frame X (lanes on t0..t4 -> coalesced runs),
//   (mix)    e^{-i beta sigma^x} on the tile bits in `mix1` as 2x2 butterflies on
//            register bits (eq:twocomponentupdates); the tile moves between
//            register frames through a swizzled 64 KiB shared-memory buffer,
//   (phase)  optionally psi_z *= e^{-i gamma E(z)} (eq:QAOA_state), E(z) from the tile
//            factorisation of SURVEY §8a-a4 (per-tile fields precomputed by
//            tile_fields_kernel, no 2^n energy table), then mixes the bits in `mix2`,
//   (reduce) optionally accumulates sum |psi|^2 E(z), sum |psi|^2,
//   (store)  back in place from a coalesced frame.
//
// Scaled butterflies: e^{-i b X} = cos b (I - i tan b X) when |cos b| >= |sin b|, and
// (-i X) e^{-i (b - pi/2) X} otherwise (the X gates become an index flip mask, see bfly):
// 2 FMA per output amplitude; the pass-wide scalar kappa^m is folded into the phase (or
// applied once per amplitude).
//
// No code here is shared with oracle/ (the CPU oracle is independent).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

// Device-side bound checks of the debug build (libqsim_debug.so, -DQSIM_DEBUG): a failed check
// traps (cudaErrorAssert), so an out-of-range tile, address or handshake slot cannot go unseen.
#ifdef QSIM_DEBUG
#include <cassert>
#define QSIM_DCHECK(c) assert(c)
#else
#define QSIM_DCHECK(c) ((void)0)
#endif

#include "qsim_device.h"

namespace qk {

// ------------------------------------------------------------------------------ helpers
__device__ __forceinline__ double spin(u64 x, int j) { return ((x >> j) & 1ull) ? 1.0 : -1.0; }

// amplitude storage types: FP64 (double2, the north-star precision) or FP32 (float2, the
// NEXT-4 precision mode).  Energies, fields and phase tables are always FP64.
template <typename V> struct VT;
template <> struct VT<double2> {
    typedef double S;
    __device__ static double2 mk(double a, double b) { return make_double2(a, b); }
};
template <> struct VT<float2> {
    typedef float S;
    __device__ static float2 mk(float a, float b) { return make_float2(a, b); }
};
template <typename V> __device__ __forceinline__ V vcast(double2 a) {
    return VT<V>::mk((typename VT<V>::S)a.x, (typename VT<V>::S)a.y);
}
template <typename V> __device__ __forceinline__ double2 dcast(V a) { return make_double2((double)a.x, (double)a.y); }

template <typename V>
__device__ __forceinline__ V cmul(V a, V b) {
    return VT<V>::mk(fma(a.x, b.x, -(a.y * b.y)), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 conjd(double2 a) { return make_double2(a.x, -a.y); }

// e^{-i theta}
__device__ __forceinline__ double2 expmi(double theta) {
    double s, c;
    sincos(theta, &s, &c);
    return make_double2(c, -s);
}

// shared-memory swizzle for 16-byte elements: conflict-free LDS/STS.128 in all frames
// (every quarter-warp varies t0..t2 or t5..t7, and the XOR mixes exactly those).
__device__ __forceinline__ int swz(int t) { return t ^ ((t >> 5) & 7); }

// ------------------------------------------------------------------ energy arithmetic
// Tile factorisation of E(z).  With the tile bits L and the other bits
// H (local non-tile + global):
//   E = E_H(z_H) + sum_{i in L} s_i h'_i(z_H) + E_LL(z_L),
//   h'_i(z_H) = h_i + sum_{j in H} J_ij s_j,
//   E_H = sum_{j in H} s_j (h_j + sum_{k in H, k>j} J_jk s_k).
// Every partial sum of dyadic data is exact, so E is bit-exact in any order.  These
// two functions are the single source of that arithmetic for the tile-field, pass,
// reduce and probe kernels.
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

// E(X) summed directly (fields i ascending, each followed by its couplings j > i): the small-state
// kernel's energy (m <= 12), also read back by qsim_energies for such states.
__device__ __forceinline__ double energy_direct(const double *hp, const double *Jp, int n, u64 X) {
    double e = 0.0;
    for (int i = 0; i < n; ++i) {
        const double si = spin(X, i);
        e += hp[i] * si;
        for (int j = i + 1; j < n; ++j) e += Jp[i * n + j] * si * spin(X, j);
    }
    return e;
}

// ------------------------------------------------------------------------ register frames
// Tile index t (12 bits) of register j (5 bits) held by (lane, warp); the register bits
// are always the contiguous tile bits RB..RB+4:  t = tthr(lane, warp) | (j << RB).
//   X: lanes t0..t4,          warps t5,t6,   regs t7..t11   (load; turning-pass store)
//   Y: lanes t5..t9,          warps t10,t11, regs t0..t4
//   Z: lanes t0..t4,          warps t10,t11, regs t5..t9    (12-bit phase / store)
//   W: lanes t0,t1,t2,t8,t9,  warps t10,t11, regs t3..t7    (run phase / store)
//   V: lanes t0,t1,t7,t8,t9,  warps t10,t11, regs t2..t6    (run frame of the low-bit swap
//      schedule, multi-GPU: the passenger t2 is mixed with the run; lane-skewed)
//   A: lanes t2..t6,          warps t0,t1,   regs t7..t11   (per-warp turning run, 128B-swizzled
//   B: lanes t2,t8..t11,      warps t0,t1,   regs t3..t7     stage: tma_turn_pw_kernel; the warp
//      bits are passengers, so A <-> B exchanges stay inside a warp; B is lane-skewed on t3,t4)
//   B5: lanes t2,t3,t4,t10,t11, warps t0,t1, regs t5..t9  (frame B of a 5-passenger run: no skew)
enum { FX = 0, FY = 1, FZ = 2, FW = 3, FV = 4, FA = 5, FB = 6, FB5 = 7 };
template <int F> struct Frame;
template <> struct Frame<FX> {
    static constexpr int RB = 7;
    __device__ static int tthr(int lane, int warp) { return lane | (warp << 5); }
};
template <> struct Frame<FY> {
    static constexpr int RB = 0;
    __device__ static int tthr(int lane, int warp) { return (lane << 5) | (warp << 10); }
};
template <> struct Frame<FZ> {
    static constexpr int RB = 5;
    __device__ static int tthr(int lane, int warp) { return lane | (warp << 10); }
};
template <> struct Frame<FW> {
    static constexpr int RB = 3;
    __device__ static int tthr(int lane, int warp) {
        return (lane & 7) | ((lane >> 3) << 8) | (warp << 10);
    }
};

template <> struct Frame<FV> {
    static constexpr int RB = 2;
    __device__ static int tthr(int lane, int warp) { return (lane & 3) | ((lane >> 2) << 7) | (warp << 10); }
};
template <> struct Frame<FA> {
    static constexpr int RB = 7;
    __device__ static int tthr(int lane, int warp) { return warp | (lane << 2); }
};
template <> struct Frame<FB> {
    static constexpr int RB = 3;
    __device__ static int tthr(int lane, int warp) { return warp | ((lane & 1) << 2) | ((lane >> 1) << 8); }
};
template <> struct Frame<FB5> {
    static constexpr int RB = 5;
    __device__ static int tthr(int lane, int warp) { return warp | ((lane & 7) << 2) | ((lane >> 3) << 10); }
};

// Lane skew of a frame's register slots in linear shared memory (element t at t * sizeof(V)):
// slot j of a lane holds register pattern j ^ skew.  FP64 (16 B, 8 lanes per wavefront):
// frame Y (lanes on t5..t9) skews t0..t2.  FP32 (8 B, 16 lanes per wavefront): Y skews t0..t3;
// W (lanes t0,t1,t2,t8,t9) skews t3 by lane bit 3 (t8), so each half-warp covers 32 banks.
// Frame V (lanes t0,t1,t7,..): FP64 skews t2 by t7, FP32 skews t2,t3 by t7,t8.
template <int F, typename V>
__device__ __forceinline__ int frame_skew(int lane) {
    if (F == FB) return (lane >> 1) & 3;
    if (F == FA) return 0;
    if (F == FV) return sizeof(V) == 16 ? ((lane >> 2) & 1) : ((lane >> 2) & 3);
    if (sizeof(V) == 16) return F == FY ? (lane & 7) : 0;
    return F == FY ? (lane & 15) : (F == FW ? ((lane >> 3) & 1) : 0);
}

// ------------------------------------------------------------------------- butterflies
// (a, b) <- (a - i t b, b - i t a) = e^{-i beta X} / cos(beta) with t = tan(beta).
// For |tan beta| > 1 the host uses e^{-i beta X} = (-i X) e^{-i (beta - pi/2) X}
// (t = -cot beta, kappa = -i sin beta): the X gates commute with every mixer and are
// tracked as an index flip mask F (state holds psi_{x xor F} at physical index x), so
// there is one butterfly form and no data movement for them.
// (FP32: the packed FFMA2 form of these butterflies was measured slower on B200 -- FFMA2 runs at
// half the instruction rate of FFMA, so it saves no FP32 pipe time, and its register pairing
// added ~300 moves per turning pass; the scalar form is kept.)
template <int RBIT, typename V>
__device__ __forceinline__ void bfly(V (&v)[NR], double td) {
    typedef typename VT<V>::S S;
    const S t = (S)td;
#pragma unroll
    for (int j = 0; j < NR; ++j) {
        if (j & (1 << RBIT)) continue;
        const V a = v[j], b = v[j | (1 << RBIT)];
        v[j] = VT<V>::mk(fma(t, b.y, a.x), fma(-t, b.x, a.y));
        v[j | (1 << RBIT)] = VT<V>::mk(fma(t, a.y, b.x), fma(-t, a.x, b.y));
    }
}

// Butterfly stages on the register bits of a 5-bit mask m5.  The masks that occur (a contiguous
// block of register bits: all five, the part of a run in frame W or X, the arriving global
// qubits, frame Z of the 12-bit set) run as straight-line code: a run-time test per stage makes
// every stage a control-flow join, where the compiler must return the half of the outputs it
// renamed to their home registers (64 moves per 64 DFMA, measured in the SASS; straight-line
// stages have none).  `St` supplies the stage: St::template go<R>(v) mixes register bit R.
template <unsigned M, class St, typename V>
__device__ __forceinline__ void stages_c(V (&v)[NR], const St &st) {
    if (M & 1u) st.template go<0>(v);
    if (M & 2u) st.template go<1>(v);
    if (M & 4u) st.template go<2>(v);
    if (M & 8u) st.template go<3>(v);
    if (M & 16u) st.template go<4>(v);
}
// FS: the frame (its straight-line mask set); -1 = the union (the runtime-frame turning body)
template <int FS, class St, typename V>
__device__ __forceinline__ void stages(V (&v)[NR], unsigned m5, const St &st) {
    constexpr bool X = St::kFast && (FS == -1 || FS == FX), W = St::kFast && (FS == -1 || FS == FW);
    if (m5 == 0u) return;
    if (St::kFast && m5 == 0x1Fu && FS != FZ) stages_c<0x1Fu>(v, st);
    else if (W && m5 == 0x0Fu) stages_c<0x0Fu>(v, st);
    else if (W && m5 == 0x0Eu) stages_c<0x0Eu>(v, st);
    else if (W && m5 == 0x0Cu) stages_c<0x0Cu>(v, st);
    else if (W && m5 == 0x08u) stages_c<0x08u>(v, st);
    else if (X && m5 == 0x10u) stages_c<0x10u>(v, st);
    else if (X && m5 == 0x18u) stages_c<0x18u>(v, st);
    else if (X && m5 == 0x1Cu) stages_c<0x1Cu>(v, st);
    else if (St::kFast && FS == FZ && m5 == 0x03u) stages_c<0x03u>(v, st);
    else {
        if (m5 & 1) st.template go<0>(v);
        if (m5 & 2) st.template go<1>(v);
        if (m5 & 4) st.template go<2>(v);
        if (m5 & 8) st.template go<3>(v);
        if (m5 & 16) st.template go<4>(v);
    }
}
struct RxStage {  // scaled R_x butterfly
    static constexpr bool kFast = true;
    double t;
    template <int R, typename V> __device__ __forceinline__ void go(V (&v)[NR]) const { bfly<R>(v, t); }
};
template <typename V>
__device__ __forceinline__ void mix5(V (&v)[NR], unsigned m5, double t) {
    stages<-1>(v, m5, RxStage{t});
}

// mix the tile bits of `mask` that are register bits of frame F
template <int F, typename V>
__device__ __forceinline__ void mix_frame(V (&v)[NR], unsigned mask, double t) {
    stages<F>(v, (mask >> Frame<F>::RB) & 0x1Fu, RxStage{t});
}

// general 2x2 butterfly: (a, b) <- (m00 a + m01 b, m10 a + m11 b)
template <typename V>
__device__ __forceinline__ V cmac(V m, V x, V acc) {
    return VT<V>::mk(fma(m.x, x.x, fma(-m.y, x.y, acc.x)), fma(m.x, x.y, fma(m.y, x.x, acc.y)));
}
template <int RBIT, typename V>
__device__ __forceinline__ void gbfly(V (&v)[NR], const double2 (&M)[4]) {
    const V m00 = vcast<V>(M[0]), m01 = vcast<V>(M[1]), m10 = vcast<V>(M[2]), m11 = vcast<V>(M[3]);
    const V zero = VT<V>::mk(0, 0);
#pragma unroll
    for (int j = 0; j < NR; ++j) {
        if (j & (1 << RBIT)) continue;
        const V a = v[j], b = v[j | (1 << RBIT)];
        v[j] = cmac(m00, a, cmac(m01, b, zero));
        v[j | (1 << RBIT)] = cmac(m10, a, cmac(m11, b, zero));
    }
}
// Hadamard butterfly without its 1/sqrt2 (applied once per pass): (a, b) <- (a + b, a - b)
template <int RBIT, typename V>
__device__ __forceinline__ void hbfly(V (&v)[NR]) {
#pragma unroll
    for (int j = 0; j < NR; ++j) {
        if (j & (1 << RBIT)) continue;
        const V a = v[j], b = v[j | (1 << RBIT)];
        v[j] = VT<V>::mk(a.x + b.x, a.y + b.y);
        v[j | (1 << RBIT)] = VT<V>::mk(a.x - b.x, a.y - b.y);
    }
}
// In a lane-skewed or flipped slot (register slot 0 holds the |1> amplitude) the lane applies
// X H X: (slot0, slot1) <- (slot1 - slot0, slot1 + slot0)
// Branch-free for both: with sg = -1 in such a slot (+1 otherwise), (a, b) <- (sg a + b, a - sg b).
template <int RBIT, typename V>
__device__ __forceinline__ void hbfly_sk(V (&v)[NR], int skew) {
    typedef typename VT<V>::S S;
    const S sg = ((skew >> RBIT) & 1) ? (S)-1 : (S)1;
#pragma unroll
    for (int j = 0; j < NR; ++j) {
        if (j & (1 << RBIT)) continue;
        const V a = v[j], b = v[j | (1 << RBIT)];
        v[j] = VT<V>::mk(fma(sg, a.x, b.x), fma(sg, a.y, b.y));
        v[j | (1 << RBIT)] = VT<V>::mk(fma(-sg, b.x, a.x), fma(-sg, b.y, a.y));
    }
}
struct HStage {
    static constexpr bool kFast = true;
    int skew;
    template <int R, typename V> __device__ __forceinline__ void go(V (&v)[NR]) const { hbfly_sk<R>(v, skew); }
};
template <int F, typename V>
__device__ __forceinline__ void hmix_frame(V (&v)[NR], unsigned mask, int skew = 0) {
    stages<F>(v, (mask >> Frame<F>::RB) & 0x1Fu, HStage{skew});
}

// `skew`: register bits whose tile bit is inverted in this lane (the lane-skewed frame Y of the
// TMA kernel); there register slot 0 holds the |1> amplitude, so the lane applies X M X
template <int RBIT, typename V>
__device__ __forceinline__ void gbfly_sk(V (&v)[NR], const double2 (&M)[4], int skew) {
    const bool sw = (skew >> RBIT) & 1;
    const double2 G[4] = {sw ? M[3] : M[0], sw ? M[2] : M[1], sw ? M[1] : M[2], sw ? M[0] : M[3]};
    gbfly<RBIT>(v, G);
}
// skews reach register bits 0..2 (FP64 frame Y) or 0..3 (FP32 frames Y, W)
template <int RB>
struct GStage {
    // general 2x2 stages are 4x the FMAs: straight-line copies of them would overflow the
    // instruction cache, so they keep the per-stage tests (moves are 1/4 of their work)
    static constexpr bool kFast = false;
    const double2 (*G)[4];  // G[tile bit]
    int skew;
    template <int R, typename V> __device__ __forceinline__ void go(V (&v)[NR]) const {
        if (R < 3 || (R == 3 && sizeof(V) == 8)) gbfly_sk<R>(v, G[RB + R], skew);
        else gbfly<R>(v, G[RB + R]);
    }
};
template <int F, typename V>
__device__ __forceinline__ void gmix_frame(V (&v)[NR], unsigned mask, const double2 (&G)[KT][4],
                                           int skew = 0) {
    stages<F>(v, (mask >> Frame<F>::RB) & 0x1Fu, GStage<Frame<F>::RB>{G, skew});
}

// runtime-frame variants (one copy of code for every frame): element t = tthr | ((j ^ sk) << rb)
template <typename V>
__device__ __forceinline__ void lds_rt(V (&v)[NR], const V *sm, int tthr, int rb, int sk = 0) {
#pragma unroll
    for (int j = 0; j < NR; ++j) v[j] = sm[tthr | ((j ^ sk) << rb)];
}
template <typename V>
__device__ __forceinline__ void sts_rt(const V (&v)[NR], V *sm, int tthr, int rb, int sk = 0) {
#pragma unroll
    for (int j = 0; j < NR; ++j) sm[tthr | ((j ^ sk) << rb)] = v[j];
}

// frame change through shared memory (one barrier); every thread writes back exactly
// the elements it read in the previous exchange, so one barrier per exchange suffices.
template <int F1, int F2, typename V>
__device__ __forceinline__ void xch(V (&v)[NR], V *sm, int lane, int warp) {
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

template <int F, typename V>
__device__ __forceinline__ void load_tile(V (&v)[NR], const V *base, const int *L) {
    const u64 s0 = 1ull << L[Frame<F>::RB], s1 = 1ull << L[Frame<F>::RB + 1], s2 = 1ull << L[Frame<F>::RB + 2],
              s3 = 1ull << L[Frame<F>::RB + 3], s4 = 1ull << L[Frame<F>::RB + 4];
#pragma unroll
    for (int j = 0; j < NR; ++j) {
        const u64 o = ((j & 1) ? s0 : 0) + ((j & 2) ? s1 : 0) + ((j & 4) ? s2 : 0) + ((j & 8) ? s3 : 0) +
                      ((j & 16) ? s4 : 0);
        v[j] = __ldcs(base + o);
    }
}

// `sk`: the frame's lane skew (slot j holds register pattern j ^ sk, see frame_skew)
template <int F, typename V>
__device__ __forceinline__ void store_tile(const V (&v)[NR], V *base, const int *L, int sk = 0) {
    const u64 s0 = 1ull << L[Frame<F>::RB], s1 = 1ull << L[Frame<F>::RB + 1], s2 = 1ull << L[Frame<F>::RB + 2],
              s3 = 1ull << L[Frame<F>::RB + 3], s4 = 1ull << L[Frame<F>::RB + 4];
#pragma unroll
    for (int j = 0; j < NR; ++j) {
        const int k = j ^ sk;
        const u64 o = ((k & 1) ? s0 : 0) + ((k & 2) ? s1 : 0) + ((k & 4) ? s2 : 0) + ((k & 8) ? s3 : 0) +
                      ((k & 16) ? s4 : 0);
        __stcs(base + o, v[j]);
    }
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
    double w[5];
};

template <int F>
__device__ inline ThreadEnergy thread_energy(const double *Jp, int n, const int *L, int lane, int warp, int ft) {
    const int t = Frame<F>::tthr(lane, warp) ^ ft;  // spins of the flipped index
    const unsigned rmask = 0x1Fu << Frame<F>::RB;
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
    for (int r = 0; r < 5; ++r) {
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

// E_RR(j) = sum_{r<r'} J_{R_r R_r'} s_r(j) s_r'(j) for the 32 register patterns
// (j already xor-ed with the register-bit flips by the caller)
template <int F>
__device__ inline double err_of(const double *Jp, int n, const int *L, int j) {
    double e = 0.0;
    for (int r = 0; r < 5; ++r)
        for (int r2 = r + 1; r2 < 5; ++r2)
            e += Jp[L[Frame<F>::RB + r] * n + L[Frame<F>::RB + r2]] * (((j >> r) & 1) ? 1.0 : -1.0) *
                 (((j >> r2) & 1) ? 1.0 : -1.0);
    return e;
}

// per-CTA launch constants and reduction scratch in shared memory
struct CtaShared {
    double2 PRR[NR];     // e^{-i gamma E_RR(j)}
    float2 PRRf[NR];     // the same in FP32 (FP32 precision mode)
    double eRR[NR];      // E_RR(j)
    double red[2][NTHR / 32];
};

// per-tile record written by tile_fields_kernel:
//   e[i] = h'_i(z_H) for the 12 tile bits, e[12] = E_H(z_H);  f[i] = e^{-i gamma e[i]}
struct __align__(16) TileRec {
    double2 f[13];
    double e[13];
    double pad;
};

// psi_z *= e^{-i gamma E} for the thread's 32 amplitudes (frame F):
//   E = E_H + sum_{i in T} s_i h'_i + E_TT + sum_r s_r (h'_{R_r} + w_r) + E_RR(j)
// pconst = kappa-scale * e^{-i gamma E_TT};  u[r] = e^{-i gamma w_r}.
// The register-bit factor is lo[j & 3] * hi[j >> 2] (conjugate symmetry halves the work).
// tthr is the thread's tile index xor the tile-bit flips; fr = register-bit flips; sk = the
// frame's lane skew (register slot j holds register pattern j ^ sk; PRR is indexed by pattern).
// FP32 states take the factor products in FP32 from FP64 tables (PRRf = PRR in FP32).
template <int F>
__device__ __forceinline__ void apply_phase(double2 (&v)[NR], const TileRec *R, int tthr, int fr, double2 pconst,
                                            const double2 (&u)[5], const double2 *PRR, const float2 * = nullptr,
                                            int sk = 0) {
    fr ^= sk;  // slot j holds pattern j ^ sk: its spins are those of (j ^ sk ^ flips)
    // base = f_H * pconst * prod over the 7 thread tile bits of f_i^{s_i}, as a product tree
    // (depth 3 instead of a chain of 8 dependent complex multiplies)
    double2 fac[8];
    fac[0] = cmul(R->f[12], pconst);
    {
        int k = 1;
#pragma unroll
        for (int i = 0; i < KT; ++i) {
            if (i >= Frame<F>::RB && i < Frame<F>::RB + 5) continue;
            const double2 fi = R->f[i];
            const double sg = ((tthr >> i) & 1) ? 1.0 : -1.0;
            fac[k++] = make_double2(fi.x, sg * fi.y);
        }
    }
#pragma unroll
    for (int w = 1; w < 8; w <<= 1)
#pragma unroll
        for (int a = 0; a < 8; a += 2 * w) fac[a] = cmul(fac[a], fac[a + w]);
    const double2 base = fac[0];
    double2 g[5];
#pragma unroll
    for (int r = 0; r < 5; ++r) {
        const double2 gr = cmul(R->f[Frame<F>::RB + r], u[r]);
        g[r] = ((fr >> r) & 1) ? conjd(gr) : gr;  // flipped register bit: s_r -> -s_r
    }
    // lo over register bits 0,1 (times base): {c(A), B, c(B), A} with A = g0 g1, B = g0 c(g1)
    const double2 A = cmul(g[0], g[1]), B = cmul(g[0], conjd(g[1]));
    double2 lo[4];
    lo[0] = cmul(base, conjd(A));
    lo[1] = cmul(base, B);
    lo[2] = cmul(base, conjd(B));
    lo[3] = cmul(base, A);
    // hi over register bits 2,3,4: hi[k|4] = h4[k] g4, hi[k] = conj(hi[(3-k)|4])
    const double2 C = cmul(g[2], g[3]), D = cmul(g[2], conjd(g[3]));
    double2 hi[8];
    hi[4] = cmul(conjd(C), g[4]);
    hi[5] = cmul(D, g[4]);
    hi[6] = cmul(conjd(D), g[4]);
    hi[7] = cmul(C, g[4]);
    hi[0] = conjd(hi[7]);
    hi[1] = conjd(hi[6]);
    hi[2] = conjd(hi[5]);
    hi[3] = conjd(hi[4]);
#pragma unroll
    for (int j = 0; j < NR; ++j) v[j] = cmul(v[j], cmul(cmul(lo[j & 3], hi[j >> 2]), PRR[j ^ sk]));
}
template <int F>
__device__ __forceinline__ void apply_phase(float2 (&v)[NR], const TileRec *R, int tthr, int fr, double2 pconst,
                                            const double2 (&u)[5], const double2 *, const float2 *PRRf,
                                            int sk = 0) {
    fr ^= sk;  // slot j holds pattern j ^ sk: its spins are those of (j ^ sk ^ flips)
    double2 base = cmul(R->f[12], pconst);
#pragma unroll
    for (int i = 0; i < KT; ++i) {
        if (i >= Frame<F>::RB && i < Frame<F>::RB + 5) continue;
        const double2 fi = R->f[i];
        const double sg = ((tthr >> i) & 1) ? 1.0 : -1.0;
        base = cmul(base, make_double2(fi.x, sg * fi.y));
    }
    double2 g[5];
#pragma unroll
    for (int r = 0; r < 5; ++r) {
        const double2 gr = cmul(R->f[Frame<F>::RB + r], u[r]);
        g[r] = ((fr >> r) & 1) ? conjd(gr) : gr;
    }
    const double2 A = cmul(g[0], g[1]), B = cmul(g[0], conjd(g[1]));
    float2 lo[4];
    lo[0] = vcast<float2>(cmul(base, conjd(A)));
    lo[1] = vcast<float2>(cmul(base, B));
    lo[2] = vcast<float2>(cmul(base, conjd(B)));
    lo[3] = vcast<float2>(cmul(base, A));
    const double2 C = cmul(g[2], g[3]), D = cmul(g[2], conjd(g[3]));
    float2 hi[8];
    hi[4] = vcast<float2>(cmul(conjd(C), g[4]));
    hi[5] = vcast<float2>(cmul(D, g[4]));
    hi[6] = vcast<float2>(cmul(conjd(D), g[4]));
    hi[7] = vcast<float2>(cmul(C, g[4]));
    hi[0] = make_float2(hi[7].x, -hi[7].y);
    hi[1] = make_float2(hi[6].x, -hi[6].y);
    hi[2] = make_float2(hi[5].x, -hi[5].y);
    hi[3] = make_float2(hi[4].x, -hi[4].y);
#pragma unroll
    for (int j = 0; j < NR; ++j) v[j] = cmul(v[j], cmul(cmul(lo[j & 3], hi[j >> 2]), PRRf[j ^ sk]));
}

// accumulate sum |psi|^2 E and sum |psi|^2 over the thread's 32 amplitudes (frame F)
template <int F, typename V>
__device__ __forceinline__ void accumulate(const V (&v)[NR], const TileRec *R, int tthr, int fr,
                                           const ThreadEnergy &te, const double *eRR, double &acc_e,
                                           double &acc_n, int sk = 0) {
    fr ^= sk;
    double Q[NR];
    double eb = R->e[12] + te.eTT;
#pragma unroll
    for (int i = 0; i < KT; ++i) {
        if (i >= Frame<F>::RB && i < Frame<F>::RB + 5) continue;
        const double ei = R->e[i];
        eb += ((tthr >> i) & 1) ? ei : -ei;
    }
    Q[0] = eb;
#pragma unroll
    for (int r = 0; r < 5; ++r) {
        const double a0 = R->e[Frame<F>::RB + r] + te.w[r];
        const double a = ((fr >> r) & 1) ? -a0 : a0;
#pragma unroll
        for (int j = 0; j < (1 << r); ++j) {
            Q[j + (1 << r)] = Q[j] + a;
            Q[j] = Q[j] - a;
        }
    }
#pragma unroll
    for (int j = 0; j < NR; ++j) {
        const double2 a = dcast(v[j]);
        const double p = fma(a.x, a.x, a.y * a.y);
        acc_e = fma(p, Q[j] + eRR[j ^ sk], acc_e);
        acc_n += p;
    }
}

__device__ __forceinline__ void block_reduce2(CtaShared &tt, double a, double b, int lane, int warp,
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
