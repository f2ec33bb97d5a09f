// qsim_device.h -- parameter blocks and launchers shared by the engine (qsim_engine.cu)
// and the kernels (qsim_device.cu).  Plain structs; no device code.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

struct CUtensorMap_st;  // <cuda.h>

namespace qk {

typedef unsigned long long u64;
constexpr int KT = 12;          // tile bits per pass
constexpr int TILE = 1 << KT;   // amplitudes per tile
constexpr int NTHR = 128;       // threads per CTA (one tile in flight per CTA)
constexpr int NR = 32;          // amplitudes per thread (5 register bits)
constexpr int NMAX = 40;        // max qubits
constexpr int SM_TILE_BYTES = TILE * 16;

struct Mix {
    double t;   // tan(beta), or -cot(beta) when |tan beta| > 1 (then the X gates go to the flip mask)
    int form;   // 1 in the latter case (host bookkeeping only)
};

// pass programs: which register frames a tile visits
enum PassKind {
    K_PLAIN12 = 0,   // 12-bit set (bits 0..11), mix1 only:        X -> Y -> Z, store Z
    K_PLAIN_RUN = 1, // run set (passengers + <= 9 mixed), mix1:    X -> W, store W
    K_TURN12 = 2,    // 12-bit set, mix1 -> phase -> mix2:          X -> Y -> Z(phase) -> Y -> X
    K_TURN_RUN = 3   // run set, mix1 -> phase -> mix2:             X -> W(phase) -> X
};

struct PassParams {
    int kind;            // PassKind
    int f32;             // amplitude storage: 0 = FP64 (double2), 1 = FP32 (float2, NEXT-4 mode)
    int multi;           // multi-GPU pass (swap stores / moving passes possible): MV kernel instances
    double2 *psi;        // local shard, 2^m amplitudes (float2 * when f32; all state pointers alike)
    const double *hp;    // physical-frame fields, n
    const double *Jp;    // physical-frame couplings, n*n symmetric, zero diagonal
    int n, m;
    u64 xglob;           // global (rank) bits placed at positions m..n-1
    u64 flip;            // index flip mask F for the energies of this pass (psi_{x^F} stored at x)
    u64 lmask;           // mask of the tile-bit positions
    int L[KT];           // tile-bit positions (ascending)
    int nseg;            // complement segments: tile id bits -> physical positions
    int seg_len[8];
    int seg_dst[8];
    u64 ntiles;
    unsigned mix1, mix2; // tile-bit masks mixed before / after the phase
    Mix c1, c2;
    double2 scale;       // kappa1^|mix1| * kappa2^|mix2|
    int init, phase, reduce;
    double a0;           // 2^(-n/2)
    double gamma;
    double *part;        // reduce partials, 2 per CTA
    const void *rec;     // per-tile records (TileRec), written by tile_fields_kernel
    int prefetch;        // L2-prefetch the CTA's next tile
    int tm_clen[5];      // TMA path: tile id bits feeding each tensor-map coordinate (0: tile dim)
    int tm_cshift[5];
    // fused global-qubit swap: amplitude at local x = (c | y), c = top g bits, is stored at
    // dst[c][(rank << (m-g)) | y] (dst[c] = rank c's other state buffer, mapped over NVLink)
    int swap_store, gbits, rank;
    double2 *dst[8];
    // split swap: the swap's data movement is shared by the passes of a layer.
    // Group of an amplitude = bits [mv_pshift, mv_pshift + mv_pbits) of its local index (top-run
    // bits below the swapped ones, never tile bits of the non-boundary sets).  A pass moves the
    // amplitudes whose group lies in [mv_lo, mv_hi): mv == 2 (boundary pass, per element in
    // store_tile_swapped), mv == 1 (other passes, whole tiles: tile at local (v | u), v != rank,
    // is stored into rank v's other buffer at (rank | u)); everything else stays local, written
    // out of place to dst[rank].
    int mv, mv_pshift, mv_pbits;
    // low-bit swap schedule (mv == 3, MV == 2 kernels): the g global bits are exchanged with the
    // passenger positions [wsh, wsh + g) (wsh = 3 - g); a moving tile's amplitude at local x goes
    // to rank c = x's bits there, at x with those bits set to this rank (tiles of group
    // [mv_lo, mv_hi) move, the others are written out of place locally)
    int wsh;
    unsigned mv_lo, mv_hi;
    // in-place fused swap (multi-GPU without a second shard buffer, the n = 36 path): a moving
    // pass stores its peer-bound amplitudes into the peers' CURRENT buffers, in place.  The
    // partner of a moving tile (the tile its data replaces) sits at the same visiting slot s on
    // the peer: the boundary pass (mv 2) visits the same tile ids on every rank; mv-1 passes visit
    // tile id (slot tile) ^ (rank << xor_cp) (xor_cp = tile-id position of the swapped bits).
    // Handshake per slot: after its tile's TMA load has landed, rank c writes epoch into
    // fl_peer[d][c * fl_stride + s] of every destination d; a rank stores into rank c's slot-s
    // tile only after seeing fl_own[c * fl_stride + s] >= epoch (release / acquire, system scope).
    // A wait longer than ~20 s sets *err (mapped host word) and gives up (no GPU hang).
    // whole-tile moves (mv 1) with TMA tensor stores: dmaps[c] = tensor map of the set's view of
    // rank c's destination buffer (device memory, 128 B each); chunk_cp = tile-id position of the
    // swapped bits (a moving tile u lands at tile id u with those bits = rank); nullptr = STG
    const ::CUtensorMap_st *dmaps;
    int chunk_cp;
    int ip;
    unsigned epoch;
    int xor_cp;
    u64 fl_stride;
    unsigned *fl_own;
    unsigned *fl_peer[8];
    int *err;
    // tile visiting order: the CTA's k-th tile is rotl(k, ord_rot) over ord_bits tile-id bits,
    // so that the tiles in flight at one time span all groups (moving passes interleave NVLink
    // and HBM traffic instead of alternating phases of each); 0 = natural order
    int ord_rot, ord_bits;
    // spatial split of a whole-tile moving pass (mv 1, out of place): CTAs [0, sp_ctas) visit the
    // moving tiles, the others the local ones, each stream in natural tile order (no group-bits-
    // first rotation, which breaks the run sets' DRAM locality).  Tile id = low bits | group
    // (sp_gpos, mv_pbits bits) | middle bits | destination rank (sp_dpos, gbits bits) | top bits.
    int sp, sp_ctas, sp_gpos, sp_dpos;
    // e^{-i gamma E_RR(j ^ fr)} of the turning-run phase frame's 32 register patterns, computed on
    // the host (FP64 R_x turning-run passes of the single-GPU and top-bit schedules): read from
    // the constant bank instead of shared memory
    double2 PRR[NR];
    int pw;              // per-warp turning-run kernel (tma_turn_pw_kernel; 128B-swizzled stage)
    int dbg;             // diagnostics (qsim_bench_pass): bit 0 skip stores, bit 1 skip state loads
    int tma_store;       // store tiles with TMA from the stage instead of STG from registers
    // general mixer (QSDS combined step, NEXT-1): per tile bit a 2x2 complex matrix
    // {m00, m01, m10, m11} acting on (|0>, |1>) instead of the scaled R_x butterfly
    int gmix;
    double2 gm1[KT][4], gm2[KT][4];
};

constexpr size_t TILE_REC_BYTES = 320;  // sizeof(TileRec)

struct SmallParams {
    int f32;             // FP32 state (float2 *) instead of FP64
    double2 *psi;
    const double *hp, *Jp;
    const double *ang;   // gamma[p], beta[p] in device memory, or nullptr: in angv (p <= SMALL_PMAX)
    const double2 *gmat; // optional general mixers: [p][n][4] (then beta is unused)
    int n, p, init, reduce;
    double a0;
    double *res;         // 2 doubles
    double angv[2 * 64]; // the angles by value (no host copy, no sync: the n = 12 grid scans)
};
constexpr int SMALL_PMAX = 64;

// batched small-state QAOA (qsim_qaoa_batch): one CTA per parameter point, the whole 2^n state
// (n <= 12) in shared memory; E(z) precomputed once per launch (etab, 2^n doubles)
struct BatchParams {
    const double *hp, *Jp;
    const double *gamma, *beta;  // [count][p]
    const double *etab;          // E(z), written by the energy-table kernel of the same launch
    double *out;                 // [count] <H_C>
    int n, p, count;
    double a0;
};

struct GatherParams {
    int n, m;
    u64 rank;
    u64 flip;            // physical index flip mask
    u64 first, count;
    const u64 *list;     // optional explicit logical labels (device)
    unsigned char pos[NMAX];
};

struct EnumParams {
    const double *h, *J;     // logical frame
    int n;
    u64 u0, u1;              // tile range (tile u = labels u*4096 .. u*4096+4095)
    int collect;             // 0: per-CTA minimum into part; 1: collect labels with E == emin
    double emin;
    u64 *out;                // collect: per CTA max_out slots (out + blockIdx.x * max_out), ascending
    unsigned *cta_cnt;       // collect: labels written per CTA
    unsigned long long *count;  // collect: += number of minimisers
    int max_out;
    double *part;
};


cudaError_t launch_spin(const PassParams &P, double *part, int grid, cudaStream_t s);
cudaError_t launch_sum_vec(const double *part, int nparts, int n, double *out, cudaStream_t s);
cudaError_t launch_enum(const EnumParams &E, int grid, cudaStream_t s);
cudaError_t launch_min_partials(const double *part, int nparts, double *res, cudaStream_t s);
size_t tma_smem_bytes();
cudaError_t setup_tma_kernels();
// TMA-pipelined pass (qsim_tma.cu); `tensor_map` points to a CUtensorMap (128 B)
// `store_map` is the tensor map of the output buffer (the same as `tensor_map` in place)
cudaError_t launch_tma_pass(const ::CUtensorMap_st &tensor_map, const ::CUtensorMap_st &store_map,
                            const PassParams &P, int grid, cudaStream_t s);
cudaError_t setup_kernels();
cudaError_t launch_tile_fields(const PassParams &P, void *rec, cudaStream_t s);
cudaError_t launch_reduce(const PassParams &P, int grid, cudaStream_t s);
cudaError_t launch_sum_partials(const double *part, int nparts, double *res, cudaStream_t s);
cudaError_t launch_small(const SmallParams &P, cudaStream_t s);
cudaError_t launch_qaoa_batch(const BatchParams &B, double *etab, cudaStream_t s);
cudaError_t launch_init_plus(double2 *psi, u64 count, double a0, int grid, cudaStream_t s, int f32 = 0);
cudaError_t launch_gather(const GatherParams &G, const double2 *psi, double2 *out, int grid, cudaStream_t s,
                          int f32 = 0);
cudaError_t launch_energy_dump(const GatherParams &G, const PassParams &P, double *out, int grid, cudaStream_t s);

}  // namespace qk
