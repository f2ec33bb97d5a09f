// qsim_tma_impl.cuh -- TMA-pipelined tile pass (sm_100a), the streaming hot loop of SURVEY §8a
// rows a3-a7.  Kernel templates and their launch / setup templates; the instances are compiled in
// separate translation units (qsim_tma_f64.cu, qsim_tma_f64mv.cu, qsim_tma_f32.cu, qsim_tma_pw.cu)
// so the build runs them in parallel, and qsim_tma.cu dispatches to them.
//
// One persistent CTA per SM: NG consumer groups of 128 threads (4 warps, 32 amplitudes per
// thread) and a ring of 3 shared-memory stages of one 2^12-amplitude tile (64 KiB) each.
// Tile i of the CTA lives in stage i % 3 and is processed by group i % NG.  A tile and its
// per-tile energy record arrive together by TMA (cp.async.bulk.tensor 5-D box + a 320 B bulk
// copy) on the stage's mbarrier.  The group then runs the pass program of qsim_kernels.cuh:
// each round reads the tile from the stage in one register frame, applies butterflies (and
// the phase), and writes it back; the frame of the last round is read, the stage is released
// at once (the group's elected thread issues the TMA of tile i+3 into it) and the tile is
// finished in registers and stored to HBM with coalesced 16-byte stores.  Shared memory is
// linear (element t at 16 t); frame Y is lane-skewed instead, so every frame is
// bank-conflict free.
#pragma once
#include <cuda.h>

#include "qsim_device.h"
#include "qsim_kernels.cuh"

namespace qk {

constexpr int NSTAGE = 3;
constexpr int TMA_NG = 2;  // consumer groups per CTA

struct TmaSmem {
    static constexpr size_t stage = SM_TILE_BYTES;
    static constexpr size_t rec_off = NSTAGE * stage;
    static constexpr size_t bar_off = rec_off + NSTAGE * TILE_REC_BYTES;
    static constexpr size_t iss_off = bar_off + 32;  // int issued[NSTAGE]
    static constexpr size_t cs_off = bar_off + 64;
    static constexpr size_t red_off = cs_off + ((sizeof(CtaShared) + 15) / 16) * 16;
    // per-thread phase constants of the turning-run body (u[0..4], pconst), [slot][thread]:
    // kept out of the register file, which holds the tile (they caused ~200 B of spills)
    static constexpr size_t uc_off = red_off + 2 * 8 * TMA_NG * 4;
    static constexpr size_t total = uc_off + 6 * TMA_NG * 128 * sizeof(double2);
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_5d(void *dst, const CUtensorMap *tm, const int (&c)[5], uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]),
        "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_5d(const CUtensorMap *tm, const int (&c)[5], const void *src) {
    asm volatile(
        "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(
            reinterpret_cast<uint64_t>(tm)),
        "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(smem_u32(src))
        : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void tile_coords(const PassParams &P, u64 ut, int (&c)[5]) {
#pragma unroll
    for (int d = 0; d < 5; ++d)
        c[d] = P.tm_clen[d] ? (int)((ut >> P.tm_cshift[d]) & ((1ull << P.tm_clen[d]) - 1ull)) : 0;
}
__device__ __forceinline__ void group_bar(int g) {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(128) : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// linear-layout frame I/O; skewed frames (frame_skew) permute a lane's register slots so
// that every wavefront hits distinct banks
template <int F, typename V>
__device__ __forceinline__ void lds_frame(V (&v)[NR], const V *sm, int lane, int warp) {
    const int t = Frame<F>::tthr(lane, warp);
    const int sk = frame_skew<F, V>(lane);
#pragma unroll
    for (int j = 0; j < NR; ++j) v[j] = sm[t | ((j ^ sk) << Frame<F>::RB)];
}
template <int F, typename V>
__device__ __forceinline__ void sts_frame(const V (&v)[NR], V *sm, int lane, int warp) {
    const int t = Frame<F>::tthr(lane, warp);
    const int sk = frame_skew<F, V>(lane);
#pragma unroll
    for (int j = 0; j < NR; ++j) sm[t | ((j ^ sk) << Frame<F>::RB)] = v[j];
}

struct TmaIssue {
    const CUtensorMap *tm;
    const CUtensorMap *tms;  // output tensor map (TMA stores)
    const TileRec *grec;
    unsigned char *stages;  // stage s at stages + s * SM_TILE_BYTES (FP32 tiles use half of it)
    uint32_t tile_bytes;    // TILE * sizeof(amplitude)
    TileRec *srec;
    uint64_t *full;
    volatile int *issued;  // tiles issued into each stage so far
};

// tile id of the CTA's k-th tile (PassParams::ord_rot, ::xor_cp; multi-GPU moving passes only)
template <int MV>
__device__ __forceinline__ u64 tile_of(const PassParams &P, u64 k) {
    if (!MV) return k;
    u64 u = k;
    if (P.ord_rot) {
        const u64 mask = (1ull << P.ord_bits) - 1ull;
        u = ((k << P.ord_rot) | (k >> (P.ord_bits - P.ord_rot))) & mask;
    }
    if (P.ip && P.mv == 1) u ^= (u64)P.rank << P.xor_cp;
    return u;
}

// ---- in-place fused swap handshake (PassParams::ip)
// relaxed, not release: the flag only reports that this tile's TMA load has landed (observed
// through the mbarrier before this store); a release would first wait for every earlier store
// of the thread, including its NVLink stores of the previous tiles (measured: the in-place
// boundary pass 16.9 ms with release vs ...)
__device__ __forceinline__ void ip_signal(const PassParams &P, int dest, u64 slot) {
    QSIM_DCHECK(dest >= 0 && dest < (1 << P.gbits) && dest != P.rank && slot < P.fl_stride);
    unsigned *f = P.fl_peer[dest] + (u64)P.rank * P.fl_stride + slot;
    asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(f), "r"(P.epoch) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void ip_wait(const PassParams &P, int src, u64 slot) {
    QSIM_DCHECK(src >= 0 && src < (1 << P.gbits) && src != P.rank && slot < P.fl_stride);
    const unsigned *f = P.fl_own + (u64)src * P.fl_stride + slot;
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
    if ((int)(v - P.epoch) >= 0) return;
    const uint64_t t0 = globaltimer_ns();
    for (unsigned k = 0;; ++k) {
        __nanosleep(128);
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if ((int)(v - P.epoch) >= 0) return;
        if ((k & 1023u) == 1023u && globaltimer_ns() - t0 > 20000000000ull) {
            atomicExch_system(P.err, 1);
            return;
        }
    }
}
// the tile of slot s was loaded: tell the ranks that will store into it
__device__ __forceinline__ void ip_signal_tile(const PassParams &P, u64 tb, u64 slot) {
    if (P.mv == 2) {
        for (int c = 0; c < (1 << P.gbits); ++c)
            if (c != P.rank) ip_signal(P, c, slot);
    } else if (P.mv == 1) {
        const int sh = P.m - P.gbits;
        const unsigned vr = (unsigned)((tb >> sh) & ((1ull << P.gbits) - 1ull));
        const unsigned pr = (unsigned)((tb >> P.mv_pshift) & ((1ull << P.mv_pbits) - 1ull));
        if (vr != (unsigned)P.rank && pr >= P.mv_lo && pr < P.mv_hi) ip_signal(P, (int)vr, slot);
    }
}
// before storing into the peers' slot-s tiles: wait for their loads (one thread, then the group)
__device__ __forceinline__ void ip_wait_peers(const PassParams &P, int gt, int g, u64 slot, int only = -1) {
    if (gt == 0) {
        if (only >= 0) ip_wait(P, only, slot);
        else
            for (int c = 0; c < (1 << P.gbits); ++c)
                if (c != P.rank) ip_wait(P, c, slot);
    }
    asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(128) : "memory");
}

// global sequence index of the CTA's i-th tile (cyclic over CTAs)
__device__ __forceinline__ u64 seq_of(const PassParams &, u64 i) { return blockIdx.x + i * (u64)gridDim.x; }

// ---- spatial split (PassParams::sp): combos (group, destination) of the moving stream are
// grp in [mv_lo, mv_hi) x dest != rank; the local stream has the same groups with dest == rank,
// then every other group with any dest.  Within a combo the remaining tile-id bits run fastest.
__device__ __forceinline__ u64 sp_rest_bits(const PassParams &P) { return (u64)(P.m - KT - P.mv_pbits - P.gbits); }
__device__ __forceinline__ u64 sp_count(const PassParams &P, bool moving) {
    const u64 G = 1ull << P.gbits, ng = 1ull << P.mv_pbits, nm = (u64)(P.mv_hi - P.mv_lo) * (G - 1);
    return (moving ? nm : ng * G - nm) << sp_rest_bits(P);
}
__device__ __forceinline__ u64 sp_tile(const PassParams &P, bool moving, u64 j) {
    const u64 G = 1ull << P.gbits, span = (u64)(P.mv_hi - P.mv_lo);
    const u64 c = j >> sp_rest_bits(P);
    u64 r = j & ((1ull << sp_rest_bits(P)) - 1ull);
    u64 grp, d;
    if (moving) {  // dest = rank ^ (c' + 1): a tile and its partner on the peer share j
        grp = P.mv_lo + c / (G - 1);
        d = (u64)P.rank ^ (c % (G - 1) + 1);
    } else if (c < span) {
        grp = P.mv_lo + c;
        d = (u64)P.rank;
    } else {
        const u64 c2 = c - span, gi = c2 / G;
        d = c2 % G;
        grp = gi < P.mv_lo ? gi : gi + span;
    }
    const int gp = P.sp_gpos, ge = P.sp_gpos + P.mv_pbits, dp = P.sp_dpos;
    const u64 lo = r & ((1ull << gp) - 1ull);
    r >>= gp;
    const u64 mid = r & ((1ull << (dp - ge)) - 1ull);
    r >>= (dp - ge);
    return lo | (grp << gp) | (mid << ge) | (d << dp) | (r << (dp + P.gbits));
}
// the CTA's tile count and its i-th tile id
template <int MV>
__device__ __forceinline__ u64 cta_ntiles(const PassParams &P) {
    if (MV && P.sp) {
        const bool mvs = (int)blockIdx.x < P.sp_ctas;
        const u64 k = mvs ? (u64)blockIdx.x : (u64)(blockIdx.x - P.sp_ctas);
        const u64 w = mvs ? (u64)P.sp_ctas : (u64)(gridDim.x - P.sp_ctas), cnt = sp_count(P, mvs);
        return cnt > k ? (cnt - k + w - 1) / w : 0;
    }
    return (P.ntiles > blockIdx.x) ? (P.ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
}
// the handshake slot of the CTA's i-th tile (in-place swap): its visiting index, which a moving
// tile shares with its partner on the destination rank
template <int MV>
__device__ __forceinline__ u64 cta_slot(const PassParams &P, u64 i) {
    if (MV && P.sp) {
        const bool mvs = (int)blockIdx.x < P.sp_ctas;
        const u64 k = mvs ? (u64)blockIdx.x : (u64)(blockIdx.x - P.sp_ctas);
        const u64 w = mvs ? (u64)P.sp_ctas : (u64)(gridDim.x - P.sp_ctas);
        return (mvs ? 0 : sp_count(P, true)) + k + i * w;
    }
    return seq_of(P, i);
}
template <int MV>
__device__ __forceinline__ u64 cta_tile(const PassParams &P, u64 i) {
    if (MV && P.sp) {
        const bool mvs = (int)blockIdx.x < P.sp_ctas;
        const u64 k = mvs ? (u64)blockIdx.x : (u64)(blockIdx.x - P.sp_ctas);
        const u64 w = mvs ? (u64)P.sp_ctas : (u64)(gridDim.x - P.sp_ctas);
        return sp_tile(P, mvs, k + i * w);
    }
    return tile_of<MV>(P, seq_of(P, i));
}

template <int MV>
__device__ __forceinline__ void issue_tile(const PassParams &P, const TmaIssue &I, u64 i, int s, bool load_state,
                                           bool load_rec) {
    const u64 ut = cta_tile<MV>(P, i);
    const uint32_t bytes = (load_state ? I.tile_bytes : 0u) + (load_rec ? (uint32_t)TILE_REC_BYTES : 0u);
    if (!bytes) {
        I.issued[s] = I.issued[s] + 1;
        return;
    }
    mbar_expect_tx(&I.full[s], bytes);
    if (load_state) {
        int c[5];
#pragma unroll
        for (int d = 0; d < 5; ++d)
            c[d] = P.tm_clen[d] ? (int)((ut >> P.tm_cshift[d]) & ((1ull << P.tm_clen[d]) - 1ull)) : 0;
        tma_load_5d(I.stages + (size_t)s * SM_TILE_BYTES, I.tm, c, &I.full[s]);
    }
    if (load_rec) bulk_load(I.srec + s, I.grec + ut, (uint32_t)TILE_REC_BYTES, &I.full[s]);
    __threadfence_block();
    I.issued[s] = I.issued[s] + 1;
}

// Stage s is consumed alternately by the two groups, so a group may reach its wait for tile i
// while the stage still holds tile i-3 (not yet consumed by the other group).  The parity wait
// would then test the *preceding* phase and pass at once; waiting first until tile i has been
// issued into the stage (which happens only after tile i-3 was consumed) makes it exact.
__device__ __forceinline__ void wait_tile(const TmaIssue &I, u64 i) {
    const int s = (int)(i % NSTAGE);
    const int need = (int)(i / NSTAGE) + 1;
    while (I.issued[s] < need) __nanosleep(32);
    QSIM_DCHECK(I.issued[s] == need);  // the stage cannot be refilled before this tile is consumed
    mbar_wait(&I.full[s], (uint32_t)((i / NSTAGE) & 1));
}

constexpr unsigned TMX = 0xF80u, TMY = 0x01Fu, TMZ = 0x060u, TMW = 0x078u;

// store with the fused global-qubit swap: local index x = (c | y) with c the top
// g local bits goes to rank c's other buffer at (rank | y); 1/G of the stores stay local, the
// rest cross NVLink as 16-byte stores coalesced into >= 128-byte rows.  With the split swap
// only the amplitudes whose group (PassParams::mv_*) this pass owns move; the others are
// written unswapped into the local other buffer (a later pass of the layer moves them).
template <int F, typename V>
__device__ __forceinline__ void store_tile_swapped(const V (&v)[NR], const PassParams &P, u64 xb) {
    const int sh = P.m - P.gbits;
    const u64 ymask = (1ull << sh) - 1ull;
    const u64 rofs = (u64)P.rank << sh;
    const u64 pmask = (1ull << P.mv_pbits) - 1ull;
    V *const own = reinterpret_cast<V *>(P.dst[P.rank]);
    const u64 s0 = 1ull << P.L[Frame<F>::RB], s1 = 1ull << P.L[Frame<F>::RB + 1], s2 = 1ull << P.L[Frame<F>::RB + 2],
              s3 = 1ull << P.L[Frame<F>::RB + 3], s4 = 1ull << P.L[Frame<F>::RB + 4];
#pragma unroll
    for (int j = 0; j < NR; ++j) {
        const u64 x = xb + ((j & 1) ? s0 : 0) + ((j & 2) ? s1 : 0) + ((j & 4) ? s2 : 0) + ((j & 8) ? s3 : 0) +
                      ((j & 16) ? s4 : 0);
        QSIM_DCHECK((x >> P.m) == 0 && (x >> sh) < (1ull << P.gbits));
        const unsigned pr = (unsigned)((x >> P.mv_pshift) & pmask);
        V *a = (pr >= P.mv_lo && pr < P.mv_hi) ? reinterpret_cast<V *>(P.dst[x >> sh]) + (rofs | (x & ymask)) : own + x;
        __stcs(a, v[j]);
    }
}

// store with the low-bit swap (PassParams::wsh): the swap bits are lane bits of frame F, so all
// 32 amplitudes of a thread go to the same rank c (its base pointer is per thread)
template <int F, typename V>
__device__ __forceinline__ void store_lowswap(const V (&v)[NR], const PassParams &P, u64 xb, int sk) {
    const u64 wm = ((1ull << P.gbits) - 1ull) << P.wsh;
    const unsigned c = (unsigned)((xb >> P.wsh) & ((1ull << P.gbits) - 1ull));
    V *const base = reinterpret_cast<V *>(P.dst[c]) + ((xb & ~wm) | ((u64)P.rank << P.wsh));
    store_tile<F>(v, base, P.L, sk);
}
__device__ __forceinline__ bool lowswap_moves(const PassParams &P, u64 tb) {
    const unsigned grp = (unsigned)((tb >> P.mv_pshift) & ((1ull << P.mv_pbits) - 1ull));
    return grp >= P.mv_lo && grp < P.mv_hi;
}

// the mixer of a frame: scaled R_x butterflies, or the general per-bit 2x2 (GMIX)
// mixer modes: GMIX 0 = scaled R_x, 1 = general per-bit 2x2, 2 = Hadamard
#define MIXF(FR, MASK, WHICH)                                                             \
    do {                                                                                  \
        if (GMIX == 1) gmix_frame<FR>(v, (MASK), (WHICH) == 1 ? P.gm1 : P.gm2, frame_skew<FR, V>(lane)); \
        else if (GMIX == 2) hmix_frame<FR>(v, (MASK), frame_skew<FR, V>(lane) ^ ((ft >> Frame<FR>::RB) & 31)); \
        else mix_frame<FR>(v, (MASK), (WHICH) == 1 ? P.c1.t : P.c2.t);                     \
    } while (0)

// MV: multi-GPU variant (fused / split global-qubit swap stores, tile order rotation); the
// single-GPU instances compile without that code (it costs ~3 % in the hot loop)
template <int KIND, int GMIX, typename V, int MV>
__global__ void __launch_bounds__(TMA_NG * 128, 1)
    tma_pass_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap smap,
                    const PassParams P) {
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char *stages = smem;
    TileRec *srec = reinterpret_cast<TileRec *>(smem + TmaSmem::rec_off);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + TmaSmem::bar_off);
    CtaShared &cs = *reinterpret_cast<CtaShared *>(smem + TmaSmem::cs_off);
    double *red = reinterpret_cast<double *>(smem + TmaSmem::red_off);
    constexpr bool RUN = (KIND == K_PLAIN_RUN || KIND == K_TURN_RUN);
    constexpr bool TURN = (KIND == K_TURN12 || KIND == K_TURN_RUN);
    // run frame: W, or V in the low-bit swap schedule (MV == 2, the passenger t2 mixes)
    constexpr int FRN = (MV == 2) ? FV : FW;
    constexpr unsigned TMR = (MV == 2) ? 0x07Cu : TMW;
    constexpr int FE = RUN ? FRN : FZ;

    const int tid = threadIdx.x, g = tid >> 7, gt = tid & 127, lane = gt & 31, warp = gt >> 5;
    const int n = P.n;
    const bool need_e = TURN || P.reduce;
    const bool load_state = !(TURN && P.init) && !(P.dbg & 2);
    const u64 ntl = cta_ntiles<MV>(P);
    volatile int *issued = reinterpret_cast<volatile int *>(smem + TmaSmem::iss_off);
    const TmaIssue I{&tmap, MV ? &smap : &tmap, reinterpret_cast<const TileRec *>(P.rec), stages, (uint32_t)(TILE * sizeof(V)),
                     srec, full, issued};
// STG output base (out of place when moving), re-read from the parameter bank at each use
#define OUTB (reinterpret_cast<V *>(MV && P.mv ? P.dst[P.rank] : P.psi))

    if (tid == 0) {
        for (int s = 0; s < NSTAGE; ++s) {
            mbar_init(&full[s], 1);
            issued[s] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0)
        for (int i = 0; i < NSTAGE && (u64)i < ntl; ++i)
            issue_tile<MV>(P, I, (u64)i, i, load_state, need_e);

    int ft = 0;  // tile-bit flips (X gates of the |tan beta| > 1 mixer form)
#pragma unroll
    for (int i = 0; i < KT; ++i) ft |= (int)((P.flip >> P.L[i]) & 1ull) << i;
    const int tE = Frame<FE>::tthr(lane, warp) ^ ft;
    const int fr = (ft >> Frame<FE>::RB) & 0x1F;

    ThreadEnergy te;
    double2 pconst = P.scale;
    double2 u[5];
    te.eTT = 0.0;
#pragma unroll
    for (int r = 0; r < 5; ++r) {
        te.w[r] = 0.0;
        u[r] = make_double2(1.0, 0.0);
    }
    if (need_e) {
        te = thread_energy<FE>(P.Jp, n, P.L, lane, warp, ft);
        if (TURN) {
            pconst = cmul(P.scale, expmi(P.gamma * te.eTT));
#pragma unroll
            for (int r = 0; r < 5; ++r) u[r] = expmi(P.gamma * te.w[r]);
        }
        if (tid < NR) {
            const double e = err_of<FE>(P.Jp, n, P.L, tid ^ fr);
            cs.eRR[tid] = e;
            cs.PRR[tid] = TURN ? expmi(P.gamma * e) : make_double2(1.0, 0.0);
            cs.PRRf[tid] = vcast<float2>(cs.PRR[tid]);
        }
    }
    if constexpr (KIND == K_TURN_RUN && GMIX == 0) {
        double2 *uc = reinterpret_cast<double2 *>(smem + TmaSmem::uc_off) + tid;
#pragma unroll
        for (int r = 0; r < 5; ++r) uc[r * TMA_NG * 128] = u[r];
        uc[5 * TMA_NG * 128] = pconst;
    }
    const u64 offX = thread_offset<FX>(P.L, lane, warp);
    const u64 offS = thread_offset<RUN ? FRN : FZ>(P.L, lane, warp);
    __syncthreads();

    const int skE = frame_skew<FE, V>(lane);  // skew of the phase / reduction frame
    double acc_e = 0.0, acc_n = 0.0;
    V v[NR];
    long long pend = -1;  // tile whose TMA store still reads its stage (deferred refill)
    int pend_s = 0;
    // deferred refill: the TMA store of the group's previous tile is left running and its stage
    // is refilled once this group's next tile is in, so the elected thread does not stall its warp
    // (and the group's next barrier) on the store
    auto refill_pending = [&]() {
        if (gt == 0 && pend >= 0) {
            bulk_wait_read0();
            if ((u64)pend + NSTAGE < ntl) issue_tile<MV>(P, I, (u64)pend + NSTAGE, pend_s, load_state, need_e);
            pend = -1;
        }
    };
    for (u64 i = g; i < ntl; i += TMA_NG) {
        const int s = (int)(i % NSTAGE);
        const u64 ut = cta_tile<MV>(P, i);
        const u64 tb = tile_base(P, ut);
        QSIM_DCHECK(ut < P.ntiles && (tb >> P.m) == 0 && (tb & P.lmask) == 0);
        V *sm = reinterpret_cast<V *>(stages + (size_t)s * SM_TILE_BYTES);
        const TileRec *R = srec + s;
        if (load_state || need_e) wait_tile(I, i);
        // the deferred refill as soon as this tile is in, before its first frame load (after it:
        // 12-bit pass 5.45 -> 5.40 ms, plain run 6.80 -> 6.66 in the bench step)
        refill_pending();
        if (MV && P.ip && gt == 0) ip_signal_tile(P, tb, cta_slot<MV>(P, i));
        // ------------------------------------------------ compact turning-run body
        // (instruction-cache footprint: one copy of the butterflies, the smem sweeps and the
        // phase, driven by four mix steps X(mix1) W(mix1) [phase] W(mix2) X(mix2))
        if constexpr (KIND == K_TURN_RUN && GMIX == 0) {
            const int skW = frame_skew<FRN, V>(lane);
            constexpr int RBW = Frame<FRN>::RB;
            const unsigned mx1 = (P.mix1 & TMX) >> 7, mw1 = (P.mix1 & TMR) >> RBW;
            const unsigned mw2 = (P.mix2 & TMR) >> RBW, mx2 = (P.mix2 & TMX) >> 7;
            if (!load_state) {
#pragma unroll
                for (int j = 0; j < NR; ++j) v[j] = VT<V>::mk((typename VT<V>::S)P.a0, 0);
            }
            if (!load_state) refill_pending();
            int prev = -1;  // frame of the registers: 0 = X, 1 = W
            // frame I/O as compile-time frames (immediate smem offsets; a run-time frame
            // index cost ~4 integer instructions per element, a quarter of the pass's issue)
#pragma unroll 1
            for (int stp = load_state ? 0 : 2; stp < 4; ++stp) {
                const int fr_now = (stp == 1 || stp == 2) ? 1 : 0;
                if (load_state && fr_now != prev) {
                    if (prev >= 0) {
                        if (prev) sts_frame<FRN>(v, sm, lane, warp);
                        else sts_frame<FX>(v, sm, lane, warp);
                        group_bar(g);
                    }
                    if (fr_now) lds_frame<FRN>(v, sm, lane, warp);
                    else lds_frame<FX>(v, sm, lane, warp);
                    if (prev < 0) refill_pending();
                } else if (!load_state && stp == 3) {
                    sts_frame<FRN>(v, sm, lane, warp);
                    group_bar(g);
                    lds_frame<FX>(v, sm, lane, warp);
                }
                prev = fr_now;
                if (stp == 2) {
                    const double2 *uc = reinterpret_cast<const double2 *>(smem + TmaSmem::uc_off) + tid;
                    double2 uu[5];
#pragma unroll
                    for (int r = 0; r < 5; ++r) uu[r] = uc[r * TMA_NG * 128];
                    // FP64 frame W has no lane skew: the pattern factors come from the constant bank
                    apply_phase<FRN>(v, R, tE, fr, uc[5 * TMA_NG * 128], uu,
                                     (sizeof(V) == 16 && MV != 2) ? P.PRR : cs.PRR, cs.PRRf, skW);
                }
                if (stp == 3) {  // last smem read done: release the stage unless TMA-storing
                    if (!(P.tma_store && !(MV && P.swap_store))) {
                        fence_async_smem();
                        group_bar(g);
                        if (gt == 0 && i + NSTAGE < ntl)
                            issue_tile<MV>(P, I, i + NSTAGE, s, load_state, need_e);
                    }
                }
                mix5(v, stp == 0 ? mx1 : stp == 1 ? mw1 : stp == 2 ? mw2 : mx2, stp < 2 ? P.c1.t : P.c2.t);
            }
            if (MV == 2 && P.mv == 3 && lowswap_moves(P, tb)) {  // low-bit swap: per-thread destination
                if (P.tma_store) {  // the stage is still held (TMA-store mode): release it now
                    fence_async_smem();
                    group_bar(g);
                    if (gt == 0 && i + NSTAGE < ntl) issue_tile<MV>(P, I, i + NSTAGE, s, load_state, need_e);
                }
                store_lowswap<FX>(v, P, tb + offX, 0);
            } else if (MV && P.swap_store) {
                if (P.ip) ip_wait_peers(P, gt, g, cta_slot<MV>(P, i));
                store_tile_swapped<FX>(v, P, tb + offX);
            } else if (P.tma_store) {
                sts_frame<FX>(v, sm, lane, warp);
                fence_async_smem();
                group_bar(g);
                if (gt == 0) {
                    int c[5];
                    tile_coords(P, ut, c);
                    tma_store_5d(I.tms, c, sm);
                    pend = (long long)i;
                    pend_s = s;
                }
            } else
                store_tile<FX>(v, OUTB + tb + offX, P.L);
        } else {
        // ------------------------------------------------ rounds up to the last smem read
        if (load_state) {
            lds_frame<FX>(v, sm, lane, warp);
            refill_pending();
            MIXF(FX, P.mix1 & TMX, 1);
            sts_frame<FX>(v, sm, lane, warp);
            group_bar(g);
            if (RUN) {
                lds_frame<FRN>(v, sm, lane, warp);
                if (TURN) MIXF(FRN, P.mix1 & TMR, 1);
            } else {
                lds_frame<FY>(v, sm, lane, warp);
                MIXF(FY, P.mix1 & TMY, 1);
                sts_frame<FY>(v, sm, lane, warp);
                group_bar(g);
                lds_frame<FZ>(v, sm, lane, warp);
                if (TURN) MIXF(FZ, P.mix1 & TMZ, 1);
            }
        } else {
            refill_pending();
#pragma unroll
            for (int j = 0; j < NR; ++j) v[j] = VT<V>::mk((typename VT<V>::S)P.a0, 0);
        }
        if (TURN) {
            if (GMIX == 2) {  // no phase; the pass-wide 2^{-m/2} of the Hadamards
                const typename VT<V>::S sc = (typename VT<V>::S)P.scale.x;
#pragma unroll
                for (int j = 0; j < NR; ++j) v[j] = VT<V>::mk(v[j].x * sc, v[j].y * sc);
            } else if (!(GMIX == 1 && P.gamma == 0.0 && P.scale.x == 1.0 && P.scale.y == 0.0))  // identity phase
                apply_phase<FE>(v, R, tE, fr, pconst, u, cs.PRR, cs.PRRf, skE);
            if (RUN) {
                MIXF(FRN, P.mix2 & TMR, 2);
                sts_frame<FRN>(v, sm, lane, warp);
                group_bar(g);
            } else {
                MIXF(FZ, P.mix2 & TMZ, 2);
                sts_frame<FZ>(v, sm, lane, warp);
                group_bar(g);
                lds_frame<FY>(v, sm, lane, warp);
                MIXF(FY, P.mix2 & TMY, 2);
                sts_frame<FY>(v, sm, lane, warp);
                group_bar(g);
            }
            lds_frame<FX>(v, sm, lane, warp);
        }
        // ------------------------------------------------ release the stage, refill it
        // (a reducing pass reads the stage's tile record, so it finishes before the refill)
        // TMA-store mode keeps the stage until the store has read it back
        const bool tstore = P.tma_store && !(MV && P.swap_store) && !(P.dbg & 1);
        const bool late_release = (!TURN && P.reduce) || tstore;
        if (!late_release) {
            fence_async_smem();
            group_bar(g);
            if (gt == 0 && i + NSTAGE < ntl)
                issue_tile<MV>(P, I, i + NSTAGE, s, load_state, need_e);
        }
        // ------------------------------------------------ finish in registers, store
        if (TURN) {
            MIXF(FX, P.mix2 & TMX, 2);
            if (MV && P.swap_store) {
                if (P.ip) ip_wait_peers(P, gt, g, cta_slot<MV>(P, i));
                store_tile_swapped<FX>(v, P, tb + offX);
            } else if (tstore) {
                sts_frame<FX>(v, sm, lane, warp);
                fence_async_smem();
                group_bar(g);
                if (gt == 0) {
                    int c[5];
                    tile_coords(P, ut, c);
                    tma_store_5d(I.tms, c, sm);
                    bulk_wait_read0();
                    if (i + NSTAGE < ntl) issue_tile<MV>(P, I, i + NSTAGE, s, load_state, need_e);
                }
            } else
                store_tile<FX>(v, OUTB + tb + offX, P.L);
        } else {
            if (RUN) MIXF(FRN, P.mix1 & TMR, 1);
            else MIXF(FZ, P.mix1 & TMZ, 1);
            if (P.dbg & 1) {  // diagnostics: read-only pass (keep the values alive)
                double s = 0.0;
#pragma unroll
                for (int j = 0; j < NR; ++j) s += v[j].x;
                if (s == 12345.678) OUTB[0] = v[0];
                continue;
            }
            if (P.scale.x != 1.0 || P.scale.y != 0.0) {
                const V sc = vcast<V>(P.scale);
#pragma unroll
                for (int j = 0; j < NR; ++j) v[j] = cmul(v[j], sc);
            }
            if (P.reduce) accumulate<FE>(v, R, tE, fr, te, cs.eRR, acc_e, acc_n, skE);
            if (MV == 2 && P.mv == 3 && lowswap_moves(P, tb)) {  // low-bit swap: per-thread destination
                if (late_release) {
                    fence_async_smem();
                    group_bar(g);
                    if (gt == 0 && i + NSTAGE < ntl)
                        issue_tile<MV>(P, I, i + NSTAGE, s, load_state, need_e);
                }
                store_lowswap<RUN ? FRN : FZ>(v, P, tb + offS, skE);
                continue;
            }
            if (MV && P.mv == 1) {  // split swap: this tile may belong to a peer (whole tile moves)
                const int sh = P.m - P.gbits;
                const unsigned vr = (unsigned)((tb >> sh) & ((1ull << P.gbits) - 1ull));
                const unsigned pr = (unsigned)((tb >> P.mv_pshift) & ((1ull << P.mv_pbits) - 1ull));
                if (vr != (unsigned)P.rank && pr >= P.mv_lo && pr < P.mv_hi) {
                    if (P.dmaps && tstore) {  // TMA tensor store of the whole tile into rank vr's buffer
                        sts_frame<RUN ? FRN : FZ>(v, sm, lane, warp);
                        fence_async_smem();
                        group_bar(g);
                        if (gt == 0) {
                            if (P.ip) {
                                ip_wait(P, (int)vr, cta_slot<MV>(P, i));
                                asm volatile("fence.proxy.async.global;" ::: "memory");
                            }
                            const u64 cm = ((1ull << P.gbits) - 1ull) << P.chunk_cp;
                            int c[5];
                            QSIM_DCHECK((((ut & ~cm) | ((u64)P.rank << P.chunk_cp)) < P.ntiles) &&
                                        ((ut & cm) >> P.chunk_cp) == vr);
                            tile_coords(P, (ut & ~cm) | ((u64)P.rank << P.chunk_cp), c);
                            tma_store_5d(reinterpret_cast<const CUtensorMap *>(P.dmaps) + vr, c, sm);
                            pend = (long long)i;
                            pend_s = s;
                        }
                        continue;
                    }
                    if (late_release) {
                        fence_async_smem();
                        group_bar(g);
                        if (gt == 0 && i + NSTAGE < ntl)
                            issue_tile<MV>(P, I, i + NSTAGE, s, load_state, need_e);
                    }
                    if (P.ip) ip_wait_peers(P, gt, g, cta_slot<MV>(P, i), (int)vr);
                    const u64 wm = ((1ull << P.gbits) - 1ull) << sh;
                    QSIM_DCHECK(((((tb & ~wm) | ((u64)P.rank << sh)) + offS) >> P.m) == 0);
                    store_tile<RUN ? FRN : FZ>(v, reinterpret_cast<V *>(P.dst[vr]) + ((tb & ~wm) | ((u64)P.rank << sh)) + offS,
                                              P.L, skE);
                    continue;
                }
            }
            if (tstore) {
                sts_frame<RUN ? FRN : FZ>(v, sm, lane, warp);
                fence_async_smem();
                group_bar(g);
                if (gt == 0) {
                    int c[5];
                    tile_coords(P, ut, c);
                    tma_store_5d(I.tms, c, sm);
                    pend = (long long)i;
                    pend_s = s;
                }
                continue;
            }
            if (late_release) {
                fence_async_smem();
                group_bar(g);
                if (gt == 0 && i + NSTAGE < ntl)
                    issue_tile<MV>(P, I, i + NSTAGE, s, load_state, need_e);
            }
            store_tile<RUN ? FRN : FZ>(v, OUTB + tb + offS, P.L, skE);
        }
        }  // generic body
    }
    if (pend >= 0) bulk_wait_read0();  // the stage must stay valid until the last store read it
    if (MV && (P.swap_store || P.mv)) __threadfence_system();  // NVLink stores visible before the pass completes
    if (P.reduce) {
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            acc_e += __shfl_xor_sync(0xffffffffu, acc_e, o);
            acc_n += __shfl_xor_sync(0xffffffffu, acc_n, o);
        }
        const int w = tid >> 5;
        if (lane == 0) {
            red[2 * w] = acc_e;
            red[2 * w + 1] = acc_n;
        }
        __syncthreads();
        if (tid == 0) {
            double a = 0.0, b = 0.0;
            for (int k = 0; k < TMA_NG * 4; ++k) {
                a += red[2 * k];
                b += red[2 * k + 1];
            }
            P.part[2 * blockIdx.x] = a;
            P.part[2 * blockIdx.x + 1] = b;
        }
    }
}

// ------------------------------------------------------------------ per-warp turning-run pass
// The single-GPU FP64 turning pass on a run set with 3 passengers (t0..t2) and a 9-bit run
// (t3..t11): mix1 on the run, the cost phase, mix2 on the run.  The tile arrives through a
// SWIZZLE_128B tensor map: 16-byte granule g of 128-byte row r sits at granule g ^ (r & 7), i.e.
// element t at smem index t ^ ((t >> 3) & 7).  Warp wi (0..3) of a consumer group owns the 1024
// amplitudes with passenger bits (t0, t1) = wi in both of its frames (Frame<FA>, Frame<FB>), so
// its frame changes are warp-private (__syncwarp) and conflict-free (the swizzle spreads the
// fixed t0,t1 over all banks; frame B is lane-skewed on t3,t4); the four warps meet once per tile,
// before the TMA store.  Per tile and warp: B read, mix1 (t3..t6), B -> A, mix1 (t7..t11), phase
// (frame A: its register patterns are lane-independent, so the 32 pattern factors come from the
// constant bank), mix2 (t7..t11), A -> B, mix2 (t3..t6), B write.
__device__ __forceinline__ int swz128(int t) { return t ^ ((t >> 3) & 7); }

// frame B element index of slot j: t = tthr_B | ((j ^ sk) << 3), swizzled; baseB folds the lane
// parts (tthr_B ^ sk ^ (sk << 3)), the rest is a compile-time constant per j
__device__ __forceinline__ void lds_pwB(double2 (&v)[NR], const double2 *sm, int baseB) {
#pragma unroll
    for (int j = 0; j < NR; ++j) v[j] = sm[baseB ^ ((j & 7) ^ (j << 3))];
}
__device__ __forceinline__ void sts_pwB(const double2 (&v)[NR], double2 *sm, int baseB) {
#pragma unroll
    for (int j = 0; j < NR; ++j) sm[baseB ^ ((j & 7) ^ (j << 3))] = v[j];
}
// frame B5 (5 passengers): t = tthr_B5 | (j << 5); the swizzle XORs t3, t4 (lane bits, folded into
// baseB5) and t5 = j bit 0 (compile-time per j)
__device__ __forceinline__ void lds_pwB5(double2 (&v)[NR], const double2 *sm, int baseB5) {
#pragma unroll
    for (int j = 0; j < NR; ++j) v[j] = sm[baseB5 ^ ((j << 5) | ((j & 1) << 2))];
}
__device__ __forceinline__ void sts_pwB5(const double2 (&v)[NR], double2 *sm, int baseB5) {
#pragma unroll
    for (int j = 0; j < NR; ++j) sm[baseB5 ^ ((j << 5) | ((j & 1) << 2))] = v[j];
}
__device__ __forceinline__ void lds_pwA(double2 (&v)[NR], const double2 *sm, int baseA) {
#pragma unroll
    for (int j = 0; j < NR; ++j) v[j] = sm[baseA | (j << 7)];
}
__device__ __forceinline__ void sts_pwA(const double2 (&v)[NR], double2 *sm, int baseA) {
#pragma unroll
    for (int j = 0; j < NR; ++j) sm[baseA | (j << 7)] = v[j];
}

struct PwSmem {
    static constexpr size_t align = 1024;  // SWIZZLE_128B stages must be 1024-byte aligned
    static constexpr size_t total = TmaSmem::total + align;
};

// NP: passengers, run = tile bits NP..11.  Frame A (registers t7..t11) holds the top of every
// run; the run bits below t7 are mixed in frame B (registers t3..t7: mask of t_NP..t6) or, for
// NP = 5, in frame B5 (registers t5..t9).  NP >= 7: the whole run is in frame A's registers (no
// frame change at all).  M1: mix1 = the whole run (0; nothing on the write-only init pass) or only
// the top M1 run bits (the arriving global qubits of a multi-GPU boundary pass: frame A alone, one
// frame change fewer; NP = 5)
template <int NP>
struct PwMasks {
    static constexpr bool AONLY = NP >= 7;
    static constexpr unsigned B = NP == 5 ? 0x03u : ((0x0Fu << (NP - 3)) & 0x0Fu);  // frame B(5) slots
    static constexpr unsigned A = AONLY ? ((0x1Fu << (NP - 7)) & 0x1Fu) : 0x1Fu;    // frame A slots
};
template <int NP, int M1>
__device__ __forceinline__ void pw_ldsB(double2 (&v)[NR], const double2 *sm, int baseB) {
    if (NP == 5) lds_pwB5(v, sm, baseB);
    else lds_pwB(v, sm, baseB);
}
template <int NP, int M1>
__device__ __forceinline__ void pw_stsB(const double2 (&v)[NR], double2 *sm, int baseB) {
    if (NP == 5) sts_pwB5(v, sm, baseB);
    else sts_pwB(v, sm, baseB);
}
template <int NP>
__device__ __forceinline__ void pw_mixB(double2 (&v)[NR], double t) {
    stages_c<PwMasks<NP>::B>(v, RxStage{t});  // NP = 3: t3..t6, 4: t4..t6, 6: t6, 5 (B5): t5, t6
}

template <int NP, int M1>
__global__ void __launch_bounds__(TMA_NG * 128, 1)
    tma_turn_pw_kernel(const __grid_constant__ CUtensorMap tmap, const PassParams P) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // align by an offset from smem_raw (keeps the shared address space visible: LDS/STS, not
    // generic LD/ST)
    unsigned char *smem = smem_raw + ((PwSmem::align - (smem_u32(smem_raw) & (PwSmem::align - 1))) & (PwSmem::align - 1));
    unsigned char *stg = smem;
    TileRec *srec = reinterpret_cast<TileRec *>(smem + TmaSmem::rec_off);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + TmaSmem::bar_off);
    volatile int *issued = reinterpret_cast<volatile int *>(smem + TmaSmem::iss_off);
    double2 *uc = reinterpret_cast<double2 *>(smem + TmaSmem::uc_off);

    const int tid = threadIdx.x, g = tid >> 7, gt = tid & 127, lane = gt & 31, wi = gt >> 5;
    const bool load_state = !P.init;
    const u64 ntl = (P.ntiles > blockIdx.x) ? (P.ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    const TmaIssue I{&tmap, &tmap, reinterpret_cast<const TileRec *>(P.rec), stg, (uint32_t)(TILE * 16), srec,
                     full, issued};
    if (tid == 0) {
        for (int s = 0; s < NSTAGE; ++s) {
            mbar_init(&full[s], 1);
            issued[s] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0)
        for (int i = 0; i < NSTAGE && (u64)i < ntl; ++i) issue_tile<0>(P, I, (u64)i, i, load_state, true);

    int ft = 0;
#pragma unroll
    for (int i = 0; i < KT; ++i) ft |= (int)((P.flip >> P.L[i]) & 1ull) << i;
    const int tE = Frame<FA>::tthr(lane, wi) ^ ft;
    const int fr = (ft >> Frame<FA>::RB) & 0x1F;
    {
        const ThreadEnergy te = thread_energy<FA>(P.Jp, P.n, P.L, lane, wi, ft);
        uc[5 * TMA_NG * 128 + tid] = cmul(P.scale, expmi(P.gamma * te.eTT));
#pragma unroll
        for (int r = 0; r < 5; ++r) uc[r * TMA_NG * 128 + tid] = expmi(P.gamma * te.w[r]);
    }
    const int skB = frame_skew<FB, double2>(lane);
    const int baseA = swz128(Frame<FA>::tthr(lane, wi));
    const int baseB = NP != 5 ? (Frame<FB>::tthr(lane, wi) ^ skB ^ (skB << 3))
                              : (Frame<FB5>::tthr(lane, wi) ^ ((lane >> 1) & 3));
    __syncthreads();

    double2 v[NR];
    long long pend = -1;  // tile whose TMA store still reads its stage (deferred refill)
    int pend_s = 0;
    for (u64 i = g; i < ntl; i += TMA_NG) {
        const int s = (int)(i % NSTAGE);
        QSIM_DCHECK(tile_of<0>(P, seq_of(P, i)) < P.ntiles);
        double2 *sm = reinterpret_cast<double2 *>(stg + (size_t)s * SM_TILE_BYTES);
        const TileRec *R = srec + s;
        // (refilling the previous stage before this wait when the tile is not in yet was measured
        // slower: 6.54 -> 7.3 ms; the store's smem read completes late, so its wait stalls warp 0)
        wait_tile(I, i);
        // deferred refill of the group's previous stage, as soon as this tile is in and before its
        // first frame load (after the load: 7.05-7.08 ms per turning pass in the bench step, here
        // 6.91; a TMA L2 prefetch of the tile 1-3 refills ahead was measured slower: 6.5 -> 7.4-8.3)
        if (gt == 0 && pend >= 0) {
            bulk_wait_read0();
            if ((u64)pend + NSTAGE < ntl) issue_tile<0>(P, I, (u64)pend + NSTAGE, pend_s, load_state, true);
            pend = -1;
        }
        if (load_state) {
            if (M1 == 0 && !PwMasks<NP>::AONLY) pw_ldsB<NP, M1>(v, sm, baseB);
            else lds_pwA(v, sm, baseA);
        } else {
#pragma unroll
            for (int j = 0; j < NR; ++j) v[j] = make_double2(P.a0, 0.0);
        }
        if (load_state) {  // mix1 as the engine checked: the whole run, or the M1 arriving bits
            if (M1 == 0 && PwMasks<NP>::AONLY) {
                stages_c<PwMasks<NP>::A>(v, RxStage{P.c1.t});
            } else if (M1 == 0) {
                pw_mixB<NP>(v, P.c1.t);
                pw_stsB<NP, M1>(v, sm, baseB);
                __syncwarp();
                lds_pwA(v, sm, baseA);
                stages_c<0x1Fu>(v, RxStage{P.c1.t});
            } else {
                stages_c<(((1u << M1) - 1u) << (5 - M1)) & 0x1Fu>(v, RxStage{P.c1.t});
            }
        }
        {
            double2 uu[5];
#pragma unroll
            for (int r = 0; r < 5; ++r) uu[r] = uc[r * TMA_NG * 128 + tid];
            apply_phase<FA>(v, R, tE, fr, uc[5 * TMA_NG * 128 + tid], uu, P.PRR, nullptr, 0);
        }
        stages_c<PwMasks<NP>::A>(v, RxStage{P.c2.t});
        if constexpr (PwMasks<NP>::AONLY) {
            sts_pwA(v, sm, baseA);
        } else {
            sts_pwA(v, sm, baseA);
            __syncwarp();
            pw_ldsB<NP, M1>(v, sm, baseB);
            pw_mixB<NP>(v, P.c2.t);
            pw_stsB<NP, M1>(v, sm, baseB);
        }
        // (re-reading the tile in frame X, releasing the stage at once and storing from registers
        // was measured slower: 6.5 -> 7.0-7.2 ms)
        fence_async_smem();
        group_bar(g);
        if (gt == 0) {
            int c[5];
            tile_coords(P, tile_of<0>(P, seq_of(P, i)), c);
            tma_store_5d(&tmap, c, sm);
            pend = (long long)i;
            pend_s = s;
        }
    }
    if (pend >= 0) bulk_wait_read0();
}

template <int GMIX, typename V, int MV>
cudaError_t setup_tma_kernels_g() {
    const int sh = (int)TmaSmem::total;
    cudaError_t e;
    e = cudaFuncSetAttribute(tma_pass_kernel<K_PLAIN12, GMIX, V, MV>, cudaFuncAttributeMaxDynamicSharedMemorySize, sh);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(tma_pass_kernel<K_PLAIN_RUN, GMIX, V, MV>, cudaFuncAttributeMaxDynamicSharedMemorySize, sh);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(tma_pass_kernel<K_TURN12, GMIX, V, MV>, cudaFuncAttributeMaxDynamicSharedMemorySize, sh);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(tma_pass_kernel<K_TURN_RUN, GMIX, V, MV>, cudaFuncAttributeMaxDynamicSharedMemorySize, sh);
}

template <typename V, int MV>
cudaError_t setup_tma_kernels_v() {
    cudaError_t e = setup_tma_kernels_g<0, V, MV>();
    if constexpr (MV != 2) {  // the low-bit swap schedule runs R_x mixers only
        if (e == cudaSuccess) e = setup_tma_kernels_g<1, V, MV>();
        if (e == cudaSuccess) e = setup_tma_kernels_g<2, V, MV>();
    }
    return e;
}

template <int GMIX, typename V, int MV>
cudaError_t launch_tma_pass_g(const CUtensorMap &tm, const CUtensorMap &sm, const PassParams &P, int grid,
                              cudaStream_t s) {
    const size_t sh = TmaSmem::total;
    switch (P.kind) {
        case K_PLAIN12: tma_pass_kernel<K_PLAIN12, GMIX, V, MV><<<grid, TMA_NG * 128, sh, s>>>(tm, sm, P); break;
        case K_PLAIN_RUN: tma_pass_kernel<K_PLAIN_RUN, GMIX, V, MV><<<grid, TMA_NG * 128, sh, s>>>(tm, sm, P); break;
        case K_TURN12: tma_pass_kernel<K_TURN12, GMIX, V, MV><<<grid, TMA_NG * 128, sh, s>>>(tm, sm, P); break;
        case K_TURN_RUN: tma_pass_kernel<K_TURN_RUN, GMIX, V, MV><<<grid, TMA_NG * 128, sh, s>>>(tm, sm, P); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

template <typename V, int MV>
cudaError_t launch_tma_pass_v(const CUtensorMap &tm, const CUtensorMap &sm, const PassParams &P, int grid,
                              cudaStream_t s) {
    if constexpr (MV == 2) {  // the low-bit swap schedule runs R_x mixers only
        return P.gmix == 0 ? launch_tma_pass_g<0, V, 2>(tm, sm, P, grid, s) : cudaErrorInvalidValue;
    } else {
        switch (P.gmix) {
            case 0: return launch_tma_pass_g<0, V, MV>(tm, sm, P, grid, s);
            case 1: return launch_tma_pass_g<1, V, MV>(tm, sm, P, grid, s);
            case 2: return launch_tma_pass_g<2, V, MV>(tm, sm, P, grid, s);
            default: return cudaErrorInvalidValue;
        }
    }
}


}  // namespace qk
