// qsim_engine.cu -- host engine and C-ABI (include/qsim.h) of the B200-native QAOA/AQA
// state-vector engine (arXiv:2104.03293).
//
//  * pass planner: tile sets over the local bits, boustrophedon layer order on one GPU
//    ((P-1) p + 1 HBM passes for p layers), fixed global-qubit swap
//    schedule on G > 1 GPUs (P p + 1 passes, one swap per layer),
//  * angle generation for AQA (eq:beta_k / eq:gamma_k),
//  * permutation bookkeeping (the paper's "local permutation array"),
//  * NCCL all-to-all qubit swap and all-reduce of the reduction scalars.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/qsim.h"
#include "qsim_comm.h"
#include "qsim_device.h"

using qk::u64;

namespace {

std::string g_create_error;

struct TileSet {
    int L[qk::KT];
    u64 lmask;
    unsigned own;  // tile-bit mask of the bits this set mixes
    bool full12;   // the 12-bit set of bits 0..11 (all mixed) vs a "run" set with passengers
    // TMA view of the shard for this set (units: doubles): up to 5 dims, innermost first
    int tm_rank;
    cuuint64_t tm_dim[5], tm_stride[5];  // stride in bytes of dims 1..rank-1
    cuuint32_t tm_box[5];
    int tm_clen[5], tm_cshift[5];        // tile id bits feeding non-tile coordinates
    bool tm_ok;
    int nseg;
    int seg_len[8], seg_dst[8];
    u64 ntiles;
};

struct PassOp {
    int set;
    bool init, phase, reduce;
    unsigned mix1, mix2;
    double b1, b2, gamma;
    bool swap_after;  // multi-GPU: global-qubit swap (NCCL, in place) after this pass
    bool swap_fused;  // multi-GPU: this pass stores its output swapped into the peers' buffers
    int l1 = 0, l2 = 0;  // layer indices of mix1 / mix2 (general-mixer mode)
    // split swap: share of the swap's data this pass moves (PassParams::mv, groups [lo, hi));
    // swap_done marks the layer's last moving pass (the relabelling takes effect after it)
    int mv = 0;
    unsigned lo = 0, hi = 0;
    bool swap_done = false;
    // low-bit swap schedule: this pass also mixes the swap positions (turning passes and the
    // final pass on a turning set)
    bool wmix = false;
    int gshift = 0;  // low-bit swap: lowest group bit (PassParams::mv_pshift) of a moving pass
};

// es = bytes per amplitude (16 FP64, 8 FP32)
TileSet make_set(int m, const std::vector<int> &Lpos, unsigned own, int es = 16) {
    TileSet S{};
    u64 lm = 0;
    for (int i = 0; i < qk::KT; ++i) {
        S.L[i] = Lpos[i];
        lm |= 1ull << Lpos[i];
    }
    S.lmask = lm;
    S.own = own;
    int ns = 0, p = 0;
    while (p < m) {
        if ((lm >> p) & 1ull) { ++p; continue; }
        int a = p;
        while (p < m && !((lm >> p) & 1ull)) ++p;
        S.seg_dst[ns] = a;
        S.seg_len[ns] = p - a;
        ++ns;
    }
    S.nseg = ns;
    S.ntiles = 1ull << (m - qk::KT);
    // ---- TMA tensor view: walk the bits [0, m) as maximal tile / non-tile segments.  Tile
    // segments become box dims (<= 8 bits, box <= 256; the innermost carries re/im, so <= 7
    // bits), non-tile segments become single-coordinate dims fed by tile-id bits in ascending
    // order (matching tile_base).
    S.tm_rank = 0;
    S.tm_ok = true;
    int ubit = 0;
    int b = 0;
    while (b < m && S.tm_ok) {
        const bool tile = (lm >> b) & 1ull;
        int e = b;
        while (e < m && (((lm >> e) & 1ull) != 0) == tile) ++e;
        int len = e - b;
        int pos = b;
        while (len > 0) {
            if (S.tm_rank == 5) { S.tm_ok = false; break; }
            const int d = S.tm_rank;
            int take;
            // a run set's passengers go in an innermost box of 3 bits (8 amplitudes = 128 bytes: the
            // SWIZZLE_128B span of the per-warp turning kernel; the linear smem order is the same);
            // the 12-bit set keeps 7 (1 KiB rows)
            if (tile) take = std::min(len, d == 0 ? (own == (1u << qk::KT) - 1u ? 7 : 3) : 8);
            else take = len;
            const cuuint64_t sz = 1ull << take;
            S.tm_dim[d] = (d == 0) ? 2 * sz : sz;
            S.tm_stride[d] = (cuuint64_t)es << pos;
            S.tm_box[d] = tile ? (cuuint32_t)S.tm_dim[d] : 1u;
            S.tm_clen[d] = tile ? 0 : take;
            S.tm_cshift[d] = tile ? 0 : ubit;
            if (!tile) ubit += take;
            if (d == 0 && !tile) S.tm_ok = false;  // bit 0 is always a tile bit
            pos += take;
            len -= take;
            ++S.tm_rank;
        }
        b = e;
    }
    // pad to 5 dims (the kernel always issues the .5d form of cp.async.bulk.tensor)
    for (int d = S.tm_rank; d < 5; ++d) {
        S.tm_dim[d] = 1;
        S.tm_stride[d] = (cuuint64_t)es << m;  // past the end of the shard; dim size 1
        S.tm_box[d] = 1;
        S.tm_clen[d] = 0;
        S.tm_cshift[d] = 0;
    }
    return S;
}

// Tile sets over m >= 13 local bits: S_0 = bits 0..11 (all mixed); then runs of <= 12 - minpass
// mixed bits taken top-down from bit m-1, each completed to 12 tile bits with the
// lowest bits as unmixed "passengers" (>= minpass of them: 3 -> >= 128-byte coalesced rows in
// FP64, 64-byte rows in FP32 unless minpass = 4).
// The runs are balanced (lengths differ by at most one): the pass count is fixed by the longest
// allowed run, and shorter runs leave more passengers, i.e. longer contiguous rows.
std::vector<TileSet> build_sets(int m, int es = 16, int minpass = 3, bool balanced = true) {
    std::vector<std::pair<int, int>> runs;  // [a, a+len)
    const int maxrun = qk::KT - minpass;
    const int K = m > qk::KT ? (m - qk::KT + maxrun - 1) / maxrun : 0;
    int end = m;
    for (int k = 0; k < K; ++k) {
        const int rem = end - qk::KT, left = K - k;
        // the top runs take the ceiling (unbalanced: maximal runs top-down, for experiments)
        const int len = balanced ? (rem + left - 1) / left : std::min(maxrun, rem);
        runs.push_back({end - len, len});
        end -= len;
    }
    std::reverse(runs.begin(), runs.end());
    std::vector<TileSet> sets;
    std::vector<int> L0(qk::KT);
    for (int i = 0; i < qk::KT; ++i) L0[i] = i;
    sets.push_back(make_set(m, L0, (1u << qk::KT) - 1, es));
    sets.back().full12 = true;
    for (auto &r : runs) {
        std::vector<int> L;
        int npass = qk::KT - r.second;
        for (int i = 0; i < npass; ++i) L.push_back(i);
        for (int i = 0; i < r.second; ++i) L.push_back(r.first + i);
        sets.push_back(make_set(m, L, ((1u << r.second) - 1) << npass, es));
        sets.back().full12 = false;
    }
    return sets;
}

// pass schedule for p layers; `first_init` fuses |+>^n into pass 0.
// One GPU: boustrophedon over the set order [R_1, S_12, R_2, ..., R_{P-1}] (the 12-bit
// set sits in the middle, so every phase-carrying "turning" pass is a run set); the
// pass on the last set of layer k also does phase_{k+1} and the first mix of layer k+1:
// (P-1) p + 1 passes.  G > 1: fixed schedule, top run first (boundary pass: arrivals
// with beta_{k-1}, phase_k, set with beta_k), the other sets, then the swap of the top
// g local bits with the global bits: P p + 1 passes, p swaps.
// `split` (fused swap only): the share of the swap's amplitude groups each pass of the layer
// moves (weights per pass, boundary pass first; empty = the boundary pass moves everything).
struct SwapSplit {
    int ngroups = 1;             // 2^mv_pbits
    std::vector<double> weights; // per pass of the layer, boundary pass first
};

// `lowswap` (G > 1, P >= 3): the single-GPU boustrophedon, with the g global bits exchanged
// once per layer with passenger positions by the 12-bit set's pass (low-bit swap)
// `ls_groups` / `ls_first` (low-bit swap): the swap's amplitudes are split into ls_groups groups
// (tile-id bits of the next turning set's run, `ls_gshift[set]`); the turning pass before the
// 12-bit set's pass moves groups [0, ls_first), the 12-bit set's pass the rest.
std::vector<PassOp> build_schedule(int nsets, int g, int p, const double *gam, const double *bet,
                                   bool first_init, bool fused = false, const SwapSplit *split = nullptr,
                                   bool lowswap = false, unsigned ls_groups = 1, unsigned ls_first = 0,
                                   const int *ls_gshift = nullptr) {
    std::vector<PassOp> ops;
    const int P = nsets;
    if (g == 0 || lowswap) {
        std::vector<int> order;
        order.push_back(P > 1 ? 1 : 0);
        if (P > 1) order.push_back(0);
        for (int i = 2; i < P; ++i) order.push_back(i);
        auto seq = [&](int k, int idx) { return order[(k % 2 == 0) ? idx : P - 1 - idx]; };
        ops.push_back({seq(0, 0), first_init, true, false, 0u, ~0u, 0.0, bet[0], gam[0], false, false, 0, 0});
        ops.back().wmix = lowswap;
        for (int k = 0; k < p; ++k) {
            for (int idx = 1; idx < P; ++idx) {
                int s = seq(k, idx);
                if (idx == P - 1 && k < p - 1)
                    ops.push_back({s, false, true, false, ~0u, ~0u, bet[k], bet[k + 1], gam[k + 1], false, false, k, k + 1});
                else
                    ops.push_back({s, false, false, false, ~0u, 0u, bet[k], 0.0, 0.0, false, false, k, 0});
                if (!lowswap) continue;
                PassOp &o = ops.back();
                o.wmix = (idx == P - 1);
                if (s == 0) {  // the 12-bit set's pass completes the layer's swap
                    const int gs = ls_gshift ? ls_gshift[seq(k, P - 1)] : 0;
                    o.mv = 3;
                    o.lo = ls_first;
                    o.hi = ls_groups;
                    o.gshift = gs;
                    o.swap_done = true;
                    o.swap_fused = true;
                    if (ls_first > 0) {  // the preceding turning pass moves groups [0, ls_first)
                        PassOp &t = ops[ops.size() - 1 - (size_t)idx];
                        t.mv = 3;
                        t.lo = 0;
                        t.hi = ls_first;
                        t.gshift = gs;
                    }
                }
            }
        }
    } else {
        // G > 1: per layer the boundary pass on the top run (arrivals of the last swap get
        // beta_{k-1}, phase_k, the set gets beta_k), then the other sets with beta_k.  The swap
        // of the top g local bits with the global bits either rides on the boundary pass's
        // stores (fused: output written straight into the peers' second buffers over NVLink;
        // with `split` the data movement is shared by all passes of the layer, each moving whole
        // groups of amplitudes) or follows the layer's last pass (NCCL, in place).  The trailing
        // pass gives the last arrivals beta_{p-1}.
        const int top = P - 1;
        const unsigned arrivals = ((1u << g) - 1) << (qk::KT - g);  // top g tile bits of the top set
        // group ranges [b_i, b_{i+1}) per pass of the layer
        std::vector<unsigned> bnd(P + 1, 0u);
        const int ng = (fused && split && (int)split->weights.size() == P) ? split->ngroups : 1;
        if (ng > 1) {
            double tot = 0.0;
            for (double w : split->weights) tot += w;
            double acc = 0.0;
            for (int i = 0; i < P; ++i) {
                acc += split->weights[i];
                bnd[i + 1] = (unsigned)std::lround(acc / tot * ng);
            }
            bnd[P] = (unsigned)ng;
        } else {
            for (int i = 1; i <= P; ++i) bnd[i] = 1u;
        }
        for (int k = 0; k < p; ++k) {
            const size_t first = ops.size();
            if (k == 0)
                ops.push_back({top, first_init, true, false, 0u, ~0u, 0.0, bet[0], gam[0], false, fused, 0, 0});
            else
                ops.push_back({top, false, true, false, arrivals, ~0u, bet[k - 1], bet[k], gam[k], false, fused, k - 1, k});
            for (int s = P - 2; s >= 0; --s)
                ops.push_back({s, false, false, false, ~0u, 0u, bet[k], 0.0, 0.0, false, false, k, 0});
            if (!fused) {
                ops.back().swap_after = true;
                continue;
            }
            // a pass with a non-empty group range moves (out of place): the boundary pass per
            // element (mv 2), the others whole tiles (mv 1); the rest run in place
            size_t last = first;
            for (int i = 0; i < P; ++i) {
                PassOp &o = ops[first + i];
                o.lo = bnd[i];
                o.hi = bnd[i + 1];
                o.mv = (o.hi > o.lo) ? (i == 0 ? 2 : 1) : 0;
                if (o.mv) last = first + i;
            }
            ops[last].swap_done = true;
        }
        ops.push_back({top, false, false, false, arrivals, 0u, bet[p - 1], 0.0, 0.0, false, false, p - 1, 0});
    }
    ops.back().reduce = true;
    return ops;
}

// e^{-i b X} = kappa * (scaled butterfly):  form 0 kappa = cos b, t = tan b; form 1
// kappa = -i sin b, t = -cot b (|tan b| > 1).  Exact 2x2 unitary either way.
qk::Mix mix_coef(double b, std::complex<double> &kappa) {
    double s = std::sin(b), c = std::cos(b);
    qk::Mix mx;
    if (std::fabs(c) >= std::fabs(s)) {
        mx.form = 0;
        mx.t = s / c;
        kappa = {c, 0.0};
    } else {
        mx.form = 1;
        mx.t = -c / s;
        kappa = {0.0, -s};
    }
    return mx;
}

std::complex<double> cpow_int(std::complex<double> z, int e) {
    std::complex<double> r(1.0, 0.0);
    for (int i = 0; i < e; ++i) r *= z;
    return r;
}

double pwl(const double *ks, const double *kv, int m, double s) {
    if (s <= ks[0]) return kv[0];
    for (int j = 0; j + 1 < m; ++j)
        if (s <= ks[j + 1]) return kv[j] + (kv[j + 1] - kv[j]) * (s - ks[j]) / (ks[j + 1] - ks[j]);
    return kv[m - 1];
}

int ilog2(int w) {
    int g = 0;
    while ((1 << g) < w) ++g;
    return (1 << g) == w ? g : -1;
}

}  // namespace

struct qsim {
    int n = 0, m = 0, g = 0, rank = 0, world = 1;
    int f32 = 0;        // QSIM_FP32: float2 amplitudes (NEXT-4 precision mode)
    size_t es = 16;     // bytes per amplitude
    int dev = 0, num_sms = 148;
    double2 *psi = nullptr;
    bool own_psi = false;
    double2 *tmp = nullptr;  // swap buffer (multi-GPU, when memory allows)
    void *user_buf = nullptr; // caller-owned state storage (never freed here)
    // fused swap: both state buffers of every rank mapped through CUDA IPC
    bool fused_swap = false;
    // split swap (QSIM_SPLIT_SWAP, default on): the passes of a layer share the swap's NVLink
    // traffic; groups = local bits [mv_pshift, mv_pshift + mv_pbits) (the top run below the
    // swapped bits); per-pass weights QSIM_SPLIT_W ("boundary,next,...")
    bool split = false;
    // low-bit swap schedule (G = 2 with the fused swap, opt-in QSIM_LOWSWAP=1): 2 passes per
    // layer like one GPU; the global bit is exchanged with passenger position 2 by the 12-bit
    // set's pass (PassParams::wsh)
    bool lowswap = false;
    bool ls_now = false;  // the current apply_layers call runs the low-bit swap schedule (R_x mixers)
    double ls_share = 0.5;  // share of the swap moved by the turning pass
    int mv_pshift = 0, mv_pbits = 0;
    std::vector<double> split_w;
    int cur = 0;                       // which of bufs[] currently holds the state
    double2 *bufs[2] = {nullptr, nullptr};
    double2 *peer[2][8] = {};          // peer[b][c] = rank c's buffer b (own buffer for c == rank)
    // in-place fused swap (no second buffer; PassParams::ip): peer[0][c] = rank c's state, the
    // per-slot handshake flags (world x tiles u32 per rank) and a mapped host error word
    bool ipfused = false;
    unsigned epoch = 0;
    unsigned *d_flags = nullptr;
    unsigned *fl_peer[8] = {};
    int *h_err = nullptr, *d_err = nullptr;
    int grid_cap = 0;                  // moving passes' grid (loopback ranks sharing one device)
    void *d_maps = nullptr;            // per-destination tensor maps of the whole-tile moving passes
    int tma_moves = 1;                 // QSIM_TMA_MOVES=0: whole-tile moves as STG from registers
    cudaStream_t st = nullptr;
    bool own_stream = false;
    qc::Comm *comm = nullptr;          // cross-rank transport (NCCL + CUDA IPC, or the loopback)
    bool has_ising = false;
    std::vector<double> h, J;  // logical, J symmetric with zero diagonal
    int pos[qk::NMAX];         // logical qubit -> physical bit position (the paper's permutation array)
    int qat[qk::NMAX];         // physical bit position -> logical qubit
    u64 flip = 0;              // index flip mask F: physical x holds the amplitude of x ^ F
    static constexpr int NFR = 4;
    double *d_fr[NFR] = {};    // ring of physical-frame (h, J) copies: hp[n] then Jp[n*n]
    int fr_slot = 0;
    bool fr_valid = false;     // d_fr[fr_slot] matches pos[]
    const double *cur_hp = nullptr, *cur_Jp = nullptr;
    double *d_hlog = nullptr;  // logical-frame (h, J) for the enumeration kernel
    // general-mixer mode (QSDS combined step): per layer, per logical qubit a 2x2 matrix; the
    // phase uses the J-only frame (frame_noh)
    const std::vector<double2> *gmats = nullptr;  // [layer][qubit][4]
    bool hmode = false;        // Hadamard layers (gmats holds H): dedicated butterfly
    bool frame_noh = false;
    bool fr_noh_built = false;
    double *d_part = nullptr, *d_res = nullptr, *d_ang = nullptr;
    size_t ang_cap = 0;
    void *d_scratch = nullptr;
    size_t scratch_cap = 0;
    void *d_rec = nullptr;     // per-tile records of the current pass (tile_fields_kernel)
    std::vector<TileSet> sets;
    bool pending_plus = true;
    bool res_valid = false;
    uint64_t launches = 0;
    int tma_store = 1;         // TMA stores from the stage (QSIM_TMA_STORE=0: STG from registers)
    // spatial split of the whole-tile moving run passes (PassParams::sp): share of the CTAs on
    // the moving tiles; >= 1 = the fraction of tiles that move, 0 = group-bits-first order
    // instead (QSIM_SP)
    double sp_frac = 1.0;
    // L2 promotion of the run sets' tensor maps when tiles are visited in natural order: 256 B,
    // i.e. a 128-byte row also pulls the neighbouring tile's row, which the next CTA is loading
    // at the same time (single GPU: turning pass 6.95 -> 6.81 ms; 2 GPUs, spatial split: plain run
    // 6.45 -> 5.6 ms).  The 12-bit set (contiguous), the in-place swap path and group-bits-first
    // orders keep 128 B (in place: 7.2 -> 7.9 ms with 256 B).  QSIM_L2PROMO=128 / 64 / 0 for A/B
    CUtensorMapL2promotion l2promo_run = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    std::string err;
    // optional per-pass timing (CUDA events on the handle's stream around each pass launch)
    bool prof = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    std::vector<double> prof_bytes;  // algorithmic bytes of each recorded pass
    std::vector<int> prof_kind;      // its pass program (qsim_profile_passes)
};

namespace {

int fail(qsim *q, int code, const std::string &msg) {
    if (q) q->err = msg;
    else g_create_error = msg;
    return code;
}

#define CK(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(q, QSIM_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));   \
    } while (0)

#define CM(call)                                                                              \
    do {                                                                                      \
        if (!(call)) return fail(q, QSIM_ENCCL, std::string(#call) + ": " + q->comm->error()); \
    } while (0)

// stream sync that also reports a timed-out in-place swap handshake (PassParams::err)
#define SYNC(q)                                                                                      \
    do {                                                                                             \
        CK(cudaStreamSynchronize((q)->st));                                                          \
        if ((q)->h_err && *(q)->h_err)                                                               \
            return fail(q, QSIM_ECUDA, "in-place swap handshake timed out (a rank stopped?)");       \
    } while (0)

int grid_for(const qsim *q, u64 ntiles) {
    u64 g = (u64)q->num_sms * 2;
    return (int)std::min<u64>(g, ntiles);
}

// physical position of logical qubit qb in permutation state `par`
// low-bit swap schedule: positions [3-g, 3) <-> [m, n).  Opt-in (QSIM_LOWSWAP=1): measured on
// 2 B200s at n = 31 it saves the third pass per layer but its swap moves 64-byte chunks (the
// passenger granularity), which cross NVLink at ~400 GB/s in the pass kernels instead of ~705 for
// the top-bit schedule's rows: 21.9-22.3 vs 22.4-22.5 ms per layer
bool lowswap_layout(int m, int g) {
    const char *e = std::getenv("QSIM_LOWSWAP");
    return e && std::atoi(e) == 1 && g == 1 && m >= qk::KT + 10 && m <= 32;
}
int phys_pos_low(int n, int m, int g, int par, int qb) {
    (void)n;
    if (!par || g == 0) return qb;
    const int w = 3 - g;
    if (qb >= w && qb < 3) return m + (qb - w);
    if (qb >= m) return w + (qb - m);
    return qb;
}
int phys_pos(int n, int m, int g, int par, int qb) {
    if (!par || g == 0) return qb;
    if (qb >= m - g && qb < m) return qb + g;  // top local <-> global
    if (qb >= m) return qb - g;
    return qb;
}

void reset_perm(qsim *q) {
    for (int i = 0; i < q->n; ++i) q->pos[i] = q->qat[i] = i;
    q->flip = 0;
    q->fr_valid = false;
}

// relabel the qubits: the qubit at physical position x moves to position newp[x] (data moved
// by the pass that realises it); the flip mask's bits travel with the qubits
void relabel(qsim *q, const int *newp) {
    for (int a = 0; a < q->n; ++a) q->pos[a] = newp[q->pos[a]];
    for (int a = 0; a < q->n; ++a) q->qat[q->pos[a]] = a;
    u64 f = 0;
    for (int x = 0; x < q->n; ++x)
        if ((q->flip >> x) & 1ull) f |= 1ull << newp[x];
    q->flip = f;
    q->fr_valid = false;
}

// make cur_hp / cur_Jp the physical-frame copy of (h, J) for the current permutation
// (stream-ordered upload into the next ring slot; older slots stay valid for queued kernels)
int ensure_frame(qsim *q) {
    if (q->fr_valid && q->fr_noh_built == q->frame_noh) return QSIM_OK;
    const int n = q->n;
    std::vector<double> fr((size_t)n + (size_t)n * n, 0.0);
    for (int a = 0; a < n; ++a) {
        const int pa = q->pos[a];
        fr[pa] = q->frame_noh ? 0.0 : q->h[a];
        for (int b = 0; b < n; ++b) fr[n + (size_t)pa * n + q->pos[b]] = q->J[(size_t)a * n + b];
    }
    const int slot = (q->fr_slot + 1) % qsim::NFR;
    CK(cudaMemcpyAsync(q->d_fr[slot], fr.data(), sizeof(double) * fr.size(), cudaMemcpyHostToDevice, q->st));
    q->fr_slot = slot;
    q->cur_hp = q->d_fr[slot];
    q->cur_Jp = q->d_fr[slot] + n;
    q->fr_valid = true;
    q->fr_noh_built = q->frame_noh;
    return QSIM_OK;
}

int scratch(qsim *q, size_t bytes) {
    if (q->scratch_cap >= bytes) return QSIM_OK;
    if (q->d_scratch) cudaFree(q->d_scratch);
    q->d_scratch = nullptr;
    q->scratch_cap = 0;
    CK(cudaMalloc(&q->d_scratch, bytes));
    q->scratch_cap = bytes;
    return QSIM_OK;
}

int materialize_plus(qsim *q) {
    if (!q->pending_plus) return QSIM_OK;
    double a0 = std::pow(2.0, -0.5 * q->n);
    CK(qk::launch_init_plus(q->psi, 1ull << q->m, a0, q->num_sms * 8, q->st, q->f32));
    q->launches++;
    q->pending_plus = false;
    reset_perm(q);  // |+>^n is invariant under qubit relabelling
    q->res_valid = false;
    return QSIM_OK;
}

qk::PassParams base_params(qsim *q, const TileSet &S) {
    qk::PassParams P{};
    P.f32 = q->f32;
    P.multi = q->ls_now ? 2 : (q->fused_swap ? 1 : 0);
    P.psi = q->psi;
    P.hp = q->cur_hp;
    P.Jp = q->cur_Jp;
    P.n = q->n;
    P.m = q->m;
    P.xglob = (u64)q->rank << q->m;
    P.lmask = S.lmask;
    for (int i = 0; i < qk::KT; ++i) P.L[i] = S.L[i];
    P.nseg = S.nseg;
    for (int i = 0; i < 8; ++i) {
        P.seg_len[i] = S.seg_len[i];
        P.seg_dst[i] = S.seg_dst[i];
    }
    P.ntiles = S.ntiles;
    P.a0 = std::pow(2.0, -0.5 * q->n);
    P.part = q->d_part;
    P.scale = make_double2(1.0, 0.0);
    // L2 prefetch (standalone reduction) pays only for the contiguous 64 KiB tiles of the 12-bit
    // set; for run sets every tile touches up to 512 distinct 2 MiB pages (measured slower)
    P.prefetch = S.full12;
    P.tma_store = q->tma_store;
    return P;
}

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult qr;
        void *ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &qr) == cudaSuccess &&
            qr == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    return fn;
}

// launch one pass: TMA-pipelined kernel (one CTA per SM)
// `out`: output buffer of an out-of-place pass (TMA stores go there), nullptr = in place
int launch_pass(qsim *q, const TileSet &S, qk::PassParams &P, int *grid_out, double2 *out = nullptr,
                int grid_max = 0) {
    if (P.kind == qk::K_TURN_RUN && P.gmix == 0 && !P.f32 && P.multi != 2) {
        // pattern factors of the phase frame (W: register bits = tile bits 3..7; A of the per-warp
        // kernel: tile bits 7..11), the same sums as err_of<F> over the current physical frame of J
        const int n = q->n, RB = P.pw ? 7 : 3;
        int fr = 0;
        for (int r = 0; r < 5; ++r) fr |= (int)((P.flip >> S.L[RB + r]) & 1ull) << r;
        for (int j = 0; j < qk::NR; ++j) {
            const int jj = j ^ fr;
            double e = 0.0;
            for (int r = 0; r < 5; ++r)
                for (int r2 = r + 1; r2 < 5; ++r2)
                    e += q->J[(size_t)q->qat[S.L[RB + r]] * n + q->qat[S.L[RB + r2]]] * (((jj >> r) & 1) ? 1.0 : -1.0) *
                         (((jj >> r2) & 1) ? 1.0 : -1.0);
            const double th = P.gamma * e;
            P.PRR[j] = make_double2(std::cos(th), -std::sin(th));
        }
    }
    {
        auto enc = tmap_encoder();
        if (!enc) return fail(q, QSIM_ECUDA, "cuTensorMapEncodeTiled unavailable");
        CUtensorMap tm[2];
        cuuint32_t es[5] = {1, 1, 1, 1, 1};
        const CUtensorMapDataType dt = q->f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
        for (int k = 0; k < (out ? 2 : 1); ++k) {
            CUresult r = enc(&tm[k], dt, 5u, (void *)(k ? out : q->psi), S.tm_dim,
                             S.tm_stride + 1, S.tm_box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             P.pw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                             (S.full12 || q->ipfused || P.ord_rot) ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                                   : q->l2promo_run,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS)
                return fail(q, QSIM_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
        }
        for (int d = 0; d < 5; ++d) {
            P.tm_clen[d] = S.tm_clen[d];
            P.tm_cshift[d] = S.tm_cshift[d];
        }
        int grid = (int)std::min<u64>((u64)(grid_max > 0 ? grid_max : q->num_sms), S.ntiles);
        CK(qk::launch_tma_pass(tm[0], out ? tm[1] : tm[0], P, grid, q->st));
        *grid_out = grid;
    }
    q->launches++;
    return QSIM_OK;
}

// the per-warp turning-run kernel (tma_turn_pw_kernel): FP64, R_x mixers, a run set of 3..11
// passengers (the innermost box is 128 bytes: the SWIZZLE_128B span), mix2 = the
// whole run, mix1 = the whole run, nothing (init) or the top g run bits (a multi-GPU boundary
// pass's arrivals), no fused reduction, no swap stores (any world: non-moving passes only).
// Returns P.pw (0 = not eligible).  QSIM_TURN_PW=0 selects the group-synchronous kernel instead.
int pw_eligible(const qsim *q, const TileSet &S, const qk::PassParams &P) {
    const bool off = std::getenv("QSIM_TURN_PW") && std::atoi(std::getenv("QSIM_TURN_PW")) == 0;
    if (off || q->f32 || P.gmix || P.kind != qk::K_TURN_RUN || P.reduce || P.mv || P.multi == 2) return 0;
    int np = 0;
    while (np < qk::KT && S.L[np] == np && !((S.own >> np) & 1u)) ++np;
    if (np < 3 || np > 11 || S.full12 || S.own != (((1u << (qk::KT - np)) - 1u) << np) || S.tm_box[0] != 16)
        return 0;
    if (P.mix2 != S.own) return 0;
    int m1 = -1;
    if (P.mix1 == S.own || (P.mix1 == 0u && P.init)) m1 = 0;
    for (int g = 1; g <= 3 && m1 < 0; ++g)
        if (P.mix1 == (((1u << g) - 1u) << (qk::KT - g))) m1 = g;
    if (m1 < 0 || (m1 > 0 && np != 5)) return 0;  // arrivals-only mix1 occurs on 7-bit runs (>= 4 sets)
    return 1 | (m1 << 2) | (np << 4);
}

// tensor maps of set S over every rank's destination buffer of a whole-tile moving pass
// (P.dst[c]), copied stream-ordered into q->d_maps (the previous pass's kernel has finished with
// them by then); the kernel stores a moving tile with the map of its destination rank
int encode_dest_maps(qsim *q, const TileSet &S, qk::PassParams &P) {
    auto enc = tmap_encoder();
    if (!enc) return fail(q, QSIM_ECUDA, "cuTensorMapEncodeTiled unavailable");
    if (!q->d_maps) CK(cudaMalloc(&q->d_maps, sizeof(CUtensorMap) * 8));
    CUtensorMap maps[8];
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    const CUtensorMapDataType dt = q->f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
    for (int c = 0; c < q->world; ++c) {
        CUresult r = enc(&maps[c], dt, 5u, (void *)P.dst[c], S.tm_dim, S.tm_stride + 1, S.tm_box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(q, QSIM_ECUDA, "cuTensorMapEncodeTiled (peer) failed: " + std::to_string((int)r));
    }
    CK(cudaMemcpyAsync(q->d_maps, maps, sizeof(CUtensorMap) * q->world, cudaMemcpyHostToDevice, q->st));
    P.dmaps = reinterpret_cast<const CUtensorMap_st *>(q->d_maps);
    const int cb = q->m - q->g;
    P.chunk_cp = cb - __builtin_popcountll(S.lmask & ((1ull << cb) - 1ull));
    return QSIM_OK;
}

int finish_reduce(qsim *q, int nparts) {
    CK(qk::launch_sum_partials(q->d_part, nparts, q->d_res, q->st));
    q->launches++;
    if (q->world > 1) CM(q->comm->allreduce(q->d_res, 2, qc::Op::Sum, q->st));
    q->res_valid = true;
    return QSIM_OK;
}

// bookkeeping of a swap of positions [m-g, m) <-> [m, n): permutation and flip mask
void swap_bookkeeping(qsim *q) {
    int newp[qk::NMAX];
    for (int x = 0; x < q->n; ++x)
        newp[x] = q->ls_now ? phys_pos_low(q->n, q->m, q->g, 1, x) : phys_pos(q->n, q->m, q->g, 1, x);
    relabel(q, newp);
}

// after a moving pass of the fused swap: wait until every rank's pass (and its NVLink stores)
// is done, then the other buffer holds the state; after the layer's last moving pass the
// relabelling takes effect
int finish_fused_swap(qsim *q, bool done) {
    CM(q->comm->barrier(q->st));
    if (!q->ipfused) {  // out of place: the other buffer now holds the state
        q->cur ^= 1;
        q->psi = q->bufs[q->cur];
        q->tmp = q->bufs[q->cur ^ 1];
    }
    if (done) swap_bookkeeping(q);
    return QSIM_OK;
}

// global-qubit swap: positions [m-g, m) <-> [m, n); rank r's chunk c <-> rank c's chunk r
int do_swap(qsim *q) {
    const int G = q->world;
    swap_bookkeeping(q);
    const u64 chunk = 1ull << (q->m - q->g);  // amplitudes per chunk
    const size_t cbytes = chunk * q->es;
    auto at = [&](double2 *b, u64 amp) { return (double2 *)((char *)b + amp * q->es); };
    if (q->tmp) {
        std::vector<qc::XPair> xs;
        for (int c = 0; c < G; ++c)
            if (c != q->rank) xs.push_back({c, at(q->psi, c * chunk), at(q->tmp, c * chunk), cbytes});
        CM(q->comm->exchange(xs, q->st));
        CK(cudaMemcpyAsync(at(q->tmp, q->rank * chunk), at(q->psi, q->rank * chunk), cbytes,
                           cudaMemcpyDeviceToDevice, q->st));
        std::swap(q->psi, q->tmp);
        if (q->fused_swap) q->cur ^= 1;
    } else {
        // in place through a bounded staging ring: piece by piece, copy the outgoing
        // piece of every peer chunk to staging, then send it and receive in place
        u64 piece = std::min<u64>(chunk, 1ull << 26);  // 1 GiB per peer
        int rc = scratch(q, (size_t)(G - 1) * piece * q->es);
        if (rc) return rc;
        double2 *stg = (double2 *)q->d_scratch;
        for (u64 off = 0; off < chunk; off += piece) {
            std::vector<qc::XPair> xs;
            int slot = 0;
            for (int c = 0; c < G; ++c) {
                if (c == q->rank) continue;
                CK(cudaMemcpyAsync(at(stg, (u64)slot * piece), at(q->psi, c * chunk + off), piece * q->es,
                                   cudaMemcpyDeviceToDevice, q->st));
                xs.push_back({c, at(stg, (u64)slot * piece), at(q->psi, c * chunk + off), piece * q->es});
                ++slot;
            }
            CM(q->comm->exchange(xs, q->st));
        }
    }
    return QSIM_OK;
}

int prof_events(qsim *q, cudaEvent_t *a, cudaEvent_t *b) {
    while (q->ev_pool.size() < q->ev_used + 2) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        q->ev_pool.push_back(e);
    }
    *a = q->ev_pool[q->ev_used];
    *b = q->ev_pool[q->ev_used + 1];
    q->ev_used += 2;
    return QSIM_OK;
}

// general-mixer mode: per tile bit the 2x2 matrix of the qubit sitting there, for the layers
// of mix1 / mix2; no scaled-butterfly scalar and no X-gate flips
void set_gmix(const qsim *q, qk::PassParams &P, const int *L, const PassOp &op) {
    if (!q->gmats) return;
    const std::vector<double2> &G = *q->gmats;
    if (q->hmode) {  // (a + b, a - b) butterflies, 2^{-|mixed|/2} once per pass; flips commute
        P.gmix = 2;
        P.c1.form = P.c2.form = 0;
        const int nm = __builtin_popcount(P.mix1) + __builtin_popcount(P.mix2);
        P.scale = make_double2(std::pow(0.5, 0.5 * nm), 0.0);
        return;
    }
    P.gmix = 1;
    P.c1.form = P.c2.form = 0;
    P.c1.t = P.c2.t = 0.0;
    P.scale = make_double2(1.0, 0.0);
    for (int t = 0; t < qk::KT; ++t) {
        const int a = q->qat[L[t]];
        // a flipped position stores the logical |1> amplitude in its 0 slot: use X M X
        const bool fl = (q->flip >> L[t]) & 1ull;
        for (int e = 0; e < 4; ++e) {
            const int es = fl ? 3 - e : e;
            P.gm1[t][e] = G[((size_t)op.l1 * q->n + a) * 4 + es];
            P.gm2[t][e] = G[((size_t)op.l2 * q->n + a) * 4 + es];
        }
    }
}

int apply_layers(qsim *q, const double *gam, const double *bet, int p) {
    if (q->pending_plus) reset_perm(q);  // the first pass writes |+>^n: any labelling is valid
    {
        int rc = ensure_frame(q);
        if (rc) return rc;
    }
    if (q->m <= qk::KT) {  // whole state in one CTA (single GPU only)
        qk::SmallParams S{};
        std::vector<double> ang(2 * p);
        std::copy(gam, gam + p, ang.begin());
        std::copy(bet, bet + p, ang.begin() + p);
        bool sync = q->gmats != nullptr;  // host buffers that the async copies read
        if (p <= qk::SMALL_PMAX) {  // angles by value: no copy, no sync
            std::copy(ang.begin(), ang.end(), S.angv);
            S.ang = nullptr;
        } else {
            if ((size_t)2 * p > q->ang_cap) {
                if (q->d_ang) cudaFree(q->d_ang);
                q->d_ang = nullptr;
                CK(cudaMalloc(&q->d_ang, sizeof(double) * 2 * p));
                q->ang_cap = 2 * p;
            }
            CK(cudaMemcpyAsync(q->d_ang, ang.data(), sizeof(double) * 2 * p, cudaMemcpyHostToDevice, q->st));
            S.ang = q->d_ang;
            sync = true;
        }
        S.f32 = q->f32;
        S.psi = q->psi;
        S.hp = q->cur_hp;
        S.Jp = q->cur_Jp;
        S.n = q->n;
        S.p = p;
        S.init = q->pending_plus ? 1 : 0;
        S.reduce = q->gmats ? 0 : 1;
        S.gmat = nullptr;
        if (q->gmats) {
            const std::vector<double2> &G = *q->gmats;
            int rc = scratch(q, sizeof(double2) * G.size());
            if (rc) return rc;
            CK(cudaMemcpyAsync(q->d_scratch, G.data(), sizeof(double2) * G.size(), cudaMemcpyHostToDevice, q->st));
            S.gmat = (const double2 *)q->d_scratch;
        }
        S.a0 = std::pow(2.0, -0.5 * q->n);
        S.res = q->d_res;
        CK(qk::launch_small(S, q->st));
        q->launches++;
        if (sync) CK(cudaStreamSynchronize(q->st));  // the host copies must outlive the async copies
        q->pending_plus = false;
        q->res_valid = !q->gmats;
        return QSIM_OK;
    }
    SwapSplit sp;
    if (q->split) {
        sp.ngroups = 1 << q->mv_pbits;
        sp.weights = q->split_w;
    }
    q->ls_now = q->lowswap && !q->gmats;  // general / Hadamard mixers keep the top-bit schedule
    std::vector<int> gsh(q->sets.size(), 0);
    unsigned ls_groups = 1, ls_first = 0;
    if (q->ls_now) {
        // groups: up to 4 bits of the lowest run bits of each run set (tile-id bits of the 12-bit
        // set and of the other turning set)
        int gb = 4;
        for (size_t k = 1; k < q->sets.size(); ++k) {
            const TileSet &T = q->sets[k];
            int lo = q->m, len = 0;
            for (int i = 0; i < qk::KT; ++i)
                if ((T.own >> i) & 1u) {
                    lo = std::min(lo, T.L[i]);
                    ++len;
                }
            gsh[k] = lo;
            gb = std::min(gb, len);
        }
        ls_groups = 1u << gb;
        ls_first = (unsigned)std::lround(q->ls_share * ls_groups);
        ls_first = std::min(ls_first, ls_groups);
    }
    std::vector<PassOp> ops = build_schedule((int)q->sets.size(), q->g, p, gam, bet, q->pending_plus, q->fused_swap,
                                             q->split ? &sp : nullptr, q->ls_now, ls_groups, ls_first, gsh.data());
    const int ls_gbits = ilog2((int)ls_groups);
    const unsigned wtile = q->ls_now ? ((1u << q->g) - 1u) << (3 - q->g) : 0u;  // swap positions (tile bits)
    int last_grid = 0;
    // the scaled butterflies' pass-wide scalars kappa^m are global factors: the plain passes'
    // ones ride on the next phase (turning) or reducing pass, which multiplies anyway, so the
    // plain passes do no per-amplitude scaling
    std::complex<double> carry(1.0, 0.0);
    const bool carry_on = !q->gmats;
    for (const PassOp &op : ops) {
        const TileSet &S = q->sets[op.set];
        {
            int rc = ensure_frame(q);  // a swap may have relabelled the qubits
            if (rc) return rc;
        }
        qk::PassParams P = base_params(q, S);
        std::complex<double> k1(1.0, 0.0), k2(1.0, 0.0);
        unsigned own = S.own;
        if (q->ls_now) {
            if (op.wmix) own |= wtile;
            if (S.full12) own &= ~wtile;
        }
        const unsigned m1 = op.mix1 & own, m2 = op.mix2 & own;
        P.c1 = mix_coef(op.b1, k1);
        P.c2 = mix_coef(op.b2, k2);
        P.mix1 = m1;
        P.mix2 = op.phase ? m2 : 0u;
        std::complex<double> sc = cpow_int(k1, __builtin_popcount(P.mix1)) * cpow_int(k2, __builtin_popcount(P.mix2));
        if (carry_on) {  // a plain pass defers its scalar to the next phase or reducing pass
            if (!op.phase && !op.reduce) {
                carry *= sc;
                sc = 1.0;
            } else {
                sc *= carry;
                carry = 1.0;
            }
        }
        P.scale = make_double2(sc.real(), sc.imag());
        set_gmix(q, P, S.L, op);
        // X gates of the |tan beta| > 1 form -> flip mask (energies of this pass use the
        // mask after mix1; the state after the pass carries the mask after mix2)
        auto posmask = [&](unsigned tm) {
            u64 r = 0;
            for (int i = 0; i < qk::KT; ++i)
                if ((tm >> i) & 1u) r |= 1ull << S.L[i];
            return r;
        };
        const u64 f1 = P.c1.form ? posmask(P.mix1) : 0ull;
        const u64 f2 = P.c2.form ? posmask(P.mix2) : 0ull;
        P.flip = q->flip ^ f1;
        q->flip = P.flip ^ f2;
        P.kind = S.full12 ? (op.phase ? qk::K_TURN12 : qk::K_PLAIN12) : (op.phase ? qk::K_TURN_RUN : qk::K_PLAIN_RUN);
        P.init = op.init;
        P.phase = op.phase;
        P.reduce = op.reduce;
        P.gamma = op.gamma;
        P.rec = q->d_rec;
        double2 *outbuf = nullptr;  // out-of-place output (moving passes of the fused swap)
        if (op.mv) {
            P.swap_store = op.mv == 2;
            P.mv = op.mv;
            P.gbits = q->g;
            P.rank = q->rank;
            P.mv_pshift = q->mv_pshift;
            P.mv_pbits = q->split ? q->mv_pbits : 0;
            P.mv_lo = op.lo;
            P.mv_hi = op.hi;
            if (op.mv == 3) {
                P.wsh = 3 - q->g;
                P.mv_pshift = op.gshift;
                P.mv_pbits = ls_gbits;
                if (ls_gbits > 0) {  // visit the tiles group bits first (moving and local tiles interleave)
                    P.ord_bits = q->m - qk::KT;
                    const int tpos = op.gshift - __builtin_popcountll(S.lmask & ((1ull << op.gshift) - 1ull));
                    P.ord_rot = tpos % P.ord_bits;
                }
            }
            if (q->ipfused) {  // in place: the peers' current buffers, after the per-slot handshake
                for (int c = 0; c < q->world; ++c) {
                    P.dst[c] = q->peer[0][c];
                    P.fl_peer[c] = q->fl_peer[c];
                }
                P.ip = 1;
                P.epoch = ++q->epoch;
                P.fl_own = q->d_flags;
                P.fl_stride = S.ntiles;
                P.err = q->d_err;
                const int cb = q->m - q->g;  // tile-id position of the swapped (top local) bits
                P.xor_cp = cb - __builtin_popcountll(S.lmask & ((1ull << cb) - 1ull));
            } else {
                for (int c = 0; c < q->world; ++c) P.dst[c] = q->peer[q->cur ^ 1][c];
                outbuf = q->bufs[q->cur ^ 1];
            }
            if (op.mv == 1 && q->tma_moves && P.tma_store) {
                // TMA tensor stores of the moving tiles: one map per destination buffer
                int rc = encode_dest_maps(q, S, P);
                if (rc) return rc;
            }
            if (op.mv == 1 && P.mv_pbits > 0) {
                // the group bits are tile-id bits of every non-boundary set; their tile-id position
                // = non-tile bits below them
                const int tpos = q->mv_pshift - __builtin_popcountll(S.lmask & ((1ull << q->mv_pshift) - 1ull));
                const int cb = q->m - q->g;
                const int dpos = cb - __builtin_popcountll(S.lmask & ((1ull << cb) - 1ull));
                const u64 fields = (((1ull << P.mv_pbits) - 1ull) << q->mv_pshift) | (((1ull << q->g) - 1ull) << cb);
                const int gmax = q->ipfused ? q->grid_cap : 0;  // as launch_pass sizes the grid
                const int grid = (int)std::min<u64>((u64)(gmax > 0 ? gmax : q->num_sms), S.ntiles);
                // (measured: helps on 2 GPUs at m = 30, 32 and on 4 at m = 30; hurts on 4 GPUs with four
                // or more sets, m = 31: 54.3 -> 57.4-64.8 ms per layer at every share, also with the
                // 256-byte promotion; an explicit QSIM_SP share in (0, 1) still forces it there)
                const bool sp_ok = !(q->world >= 4 && q->sets.size() >= 4) || (q->sp_frac > 0.0 && q->sp_frac < 1.0);
                if (sp_ok && !q->ipfused && !S.full12 && q->sp_frac > 0.0 && !(S.lmask & fields) &&
                    tpos + P.mv_pbits <= dpos && grid >= 2) {
                    // spatial split: a share of the CTAs visits the moving tiles, the rest the
                    // local ones, both in natural order.  Default share = the fraction of tiles
                    // that move (a moving tile takes about as long as a local one at these
                    // concurrencies); QSIM_SP=<share> overrides.  Measured optima on the run
                    // pass: 0.18 at G = 2 (fraction 1/6), 0.25 at G = 4 (1/4); DESIGN §8
                    P.sp = 1;
                    P.sp_gpos = tpos;
                    P.sp_dpos = dpos;
                    const double G = (double)(1 << q->g);
                    const double fm = (double)(op.hi - op.lo) * (G - 1.0) / ((double)(1 << P.mv_pbits) * G);
                    const double share = q->sp_frac >= 1.0 ? fm : q->sp_frac;
                    P.sp_ctas = std::max(1, std::min(grid - 1, (int)std::lround(share * grid)));
                } else {
                    // visit the tiles group bits first (moving and local tiles interleave in time)
                    P.ord_bits = q->m - qk::KT;
                    P.ord_rot = tpos % P.ord_bits;
                }
            }
        }
        P.pw = pw_eligible(q, S, P);  // after the swap setup: moving passes keep the group kernel
        if (op.phase || op.reduce) {
            CK(qk::launch_tile_fields(P, q->d_rec, q->st));
            q->launches++;
        }
        int grid = 0;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (q->prof) {
            int rc = prof_events(q, &e0, &e1);
            if (rc) return rc;
            CK(cudaEventRecord(e0, q->st));
        }
        {
            int rc = launch_pass(q, S, P, &grid, outbuf, op.mv && q->ipfused ? q->grid_cap : 0);
            if (rc) return rc;
        }
        if (q->prof) {
            CK(cudaEventRecord(e1, q->st));
            // algorithmic HBM bytes: read + write of the shard, write only for the init pass
            q->prof_bytes.push_back((op.init ? 1.0 : 2.0) * (double)q->es * (double)(1ull << q->m));
            q->prof_kind.push_back(P.kind | (op.mv ? QSIM_PASS_MOVING : 0) | (op.init ? QSIM_PASS_INIT : 0) |
                                   (op.reduce ? QSIM_PASS_REDUCE : 0));
        }
        last_grid = grid;
        if (op.mv) {
            int rc = finish_fused_swap(q, op.swap_done);
            if (rc) return rc;
        }
        if (op.swap_after) {
            int rc = do_swap(q);
            if (rc) return rc;
        }
    }
    q->pending_plus = false;
    q->ls_now = false;
    if (q->gmats) return QSIM_OK;  // J-only frame: <H_C> is recomputed on demand
    return finish_reduce(q, last_grid);
}

int check_angles(const double *a, int p) {
    for (int i = 0; i < p; ++i)
        if (!std::isfinite(a[i])) return QSIM_EINVAL;
    return QSIM_OK;
}

int run_reduce(qsim *q) {
    int rc = materialize_plus(q);
    if (rc) return rc;
    rc = ensure_frame(q);
    if (rc) return rc;
    if (q->res_valid) return QSIM_OK;
    if (q->m <= qk::KT) {
        qk::SmallParams S{};
        S.f32 = q->f32;
        S.psi = q->psi;
        S.hp = q->cur_hp;
        S.Jp = q->cur_Jp;
        S.ang = nullptr;
        S.n = q->n;
        S.p = 0;
        S.init = 0;
        S.reduce = 1;
        S.res = q->d_res;
        CK(qk::launch_small(S, q->st));
        q->launches++;
        q->res_valid = true;
        return QSIM_OK;
    }
    const TileSet &S = q->sets[0];
    qk::PassParams P = base_params(q, S);
    P.rec = q->d_rec;
    P.flip = q->flip;
    CK(qk::launch_tile_fields(P, q->d_rec, q->st));
    q->launches++;
    int grid = grid_for(q, S.ntiles);
    CK(qk::launch_reduce(P, grid, q->st));
    q->launches++;
    return finish_reduce(q, grid);
}

qk::GatherParams gather_params(const qsim *q, u64 first, u64 count, const u64 *list) {
    qk::GatherParams G{};
    G.n = q->n;
    G.m = q->m;
    G.rank = (u64)q->rank;
    G.first = first;
    G.count = count;
    G.list = list;
    G.flip = q->flip;
    for (int b = 0; b < q->n; ++b) G.pos[b] = (unsigned char)q->pos[b];
    return G;
}

// gather logical amplitudes (explicit list or range) into host memory; collective
int gather_host(qsim *q, u64 first, u64 count, const uint64_t *hlist, double *out) {
    int rc = materialize_plus(q);
    if (rc) return rc;
    const u64 CH = 1ull << 22;  // 64 MiB of amplitudes per round
    for (u64 done = 0; done < count; done += CH) {
        u64 c = std::min(CH, count - done);
        size_t need = c * sizeof(double2) + (hlist ? c * sizeof(u64) : 0);
        rc = scratch(q, need);
        if (rc) return rc;
        double2 *dout = (double2 *)q->d_scratch;
        u64 *dlist = nullptr;
        if (hlist) {
            dlist = (u64 *)((char *)q->d_scratch + c * sizeof(double2));
            CK(cudaMemcpyAsync(dlist, hlist + done, c * sizeof(u64), cudaMemcpyHostToDevice, q->st));
        }
        qk::GatherParams G = gather_params(q, first + done, c, dlist);
        CK(qk::launch_gather(G, q->psi, dout, (int)std::min<u64>((c + 255) / 256, 4096), q->st, q->f32));
        q->launches++;
        if (q->world > 1) CM(q->comm->allreduce((double *)dout, c * 2, qc::Op::Sum, q->st));
        CK(cudaMemcpyAsync(out + 2 * done, dout, c * sizeof(double2), cudaMemcpyDeviceToHost, q->st));
        SYNC(q);
    }
    return QSIM_OK;
}

int create_common(qsim *q, int n, int precision, int rank, int world, const void *uid, void *buf,
                  size_t buf_bytes, void *stream) {
    if (precision != QSIM_FP64 && precision != QSIM_FP32) return fail(q, QSIM_EINVAL, "unknown precision");
    q->f32 = precision == QSIM_FP32;
    q->es = q->f32 ? 8 : 16;
    if (n < 1 || n > qk::NMAX) return fail(q, QSIM_EINVAL, "n out of range [1, 40]");
    int g = ilog2(world);
    if (world < 1 || world > 8 || g < 0) return fail(q, QSIM_EINVAL, "world must be 1, 2, 4 or 8");
    if (rank < 0 || rank >= world) return fail(q, QSIM_EINVAL, "rank out of range");
    q->n = n;
    q->g = g;
    q->m = n - g;
    q->rank = rank;
    q->world = world;
    if (world > 1 && q->m < qk::KT + 3) return fail(q, QSIM_EUNSUPPORTED, "multi-GPU needs n - log2(world) >= 15");
    CK(cudaGetDevice(&q->dev));
    CK(cudaDeviceGetAttribute(&q->num_sms, cudaDevAttrMultiProcessorCount, q->dev));
    CK(qk::setup_kernels());
    if (stream) {
        q->st = (cudaStream_t)stream;
    } else {
        CK(cudaStreamCreateWithFlags(&q->st, cudaStreamNonBlocking));
        q->own_stream = true;
    }
    const size_t bytes = q->es << q->m;
    if (buf) {
        if (buf_bytes < bytes) return fail(q, QSIM_EINVAL, "state_buf too small");
        q->psi = (double2 *)buf;
        q->user_buf = buf;
    } else {
        cudaError_t e = cudaMalloc(&q->psi, bytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(q, QSIM_ENOMEM, "cannot allocate " + std::to_string(bytes) + " bytes for 2^" +
                                            std::to_string(q->m) + " amplitudes");
        }
        q->own_psi = true;
    }
    for (int k = 0; k < qsim::NFR; ++k) CK(cudaMalloc(&q->d_fr[k], sizeof(double) * ((size_t)n + (size_t)n * n)));
    CK(cudaMalloc(&q->d_hlog, sizeof(double) * ((size_t)n + (size_t)n * n)));
    reset_perm(q);
    CK(cudaMalloc(&q->d_part, sizeof(double) * 2 * 4 * q->num_sms));
    CK(cudaMalloc(&q->d_res, sizeof(double) * 2));
    if (q->m > qk::KT) {
        q->sets = build_sets(q->m, (int)q->es);
        // Split runs (one GPU, two 9-bit runs, i.e. m = 30): run 1 takes the bits [12, 12+a) and
        // the top 9-a bits, run 2 the 9 bits between.  With 128-byte rows a run on the top
        // bits [21, 30) streams at 61-69 % of HBM even for reads alone (the run on [12, 21) at
        // 97 %); with a = 4 both runs stream like the low one (passbench, profiles/r1_runsplit.txt).
        // QSIM_RUNSPLIT=a overrides a (0 = contiguous runs).
        int split_a = 4;
        if (const char *e = std::getenv("QSIM_RUNSPLIT")) split_a = std::max(0, std::min(8, std::atoi(e)));
        // One GPU only: on 2 and 4 GPUs the split layout (top set {12..15, 25..29}, swap groups
        // on bits 12..15) made the 12-bit pass's share of the swap slower (G = 2: 22.8 vs 22.5 ms
        // per layer, G = 4: 24.4-27.9 vs 21.7), so the multi-GPU schedules keep contiguous runs.
        // (an explicit QSIM_RUNSPLIT=a applies it on any world, for measurements)
        const bool rs_forced = std::getenv("QSIM_RUNSPLIT") && std::atoi(std::getenv("QSIM_RUNSPLIT")) > 0;
        if (split_a > 0 && split_a <= 6 && (world == 1 || rs_forced) && q->sets.size() == 3 && q->m == qk::KT + 18) {
            const int a = split_a;
            std::vector<int> L1, L2;
            for (int i = 0; i < 3; ++i) { L1.push_back(i); L2.push_back(i); }
            for (int i = 0; i < a; ++i) L1.push_back(qk::KT + i);
            for (int i = 0; i < 9 - a; ++i) L1.push_back(q->m - (9 - a) + i);
            for (int i = 0; i < 9; ++i) L2.push_back(qk::KT + a + i);
            q->sets[1] = make_set(q->m, L2, ((1u << 9) - 1) << 3, (int)q->es);
            q->sets[2] = make_set(q->m, L1, ((1u << 9) - 1) << 3, (int)q->es);
            q->sets[1].full12 = q->sets[2].full12 = false;
        }
        CK(cudaMalloc(&q->d_rec, qk::TILE_REC_BYTES << (q->m - qk::KT)));
    }
    if (world > 1) {
        {
            std::string cerr;
            q->comm = qc::make_comm(uid, world, rank, &cerr);
            if (!q->comm) return fail(q, QSIM_ENCCL, "communicator: " + cerr);
        }
        // out-of-place swap buffer when it leaves >= 8 GiB free on EVERY rank, else in-place
        // staging (QSIM_SWAP_INPLACE=1 forces the in-place path, for tests).  The ranks agree
        // before branching: the schedules differ in their collectives.
        size_t fr = 0, tot = 0;
        CK(cudaMemGetInfo(&fr, &tot));
        const char *ip = std::getenv("QSIM_SWAP_INPLACE");
        if (fr > bytes + (8ull << 30) && !(ip && std::atoi(ip) == 1)) {
            if (cudaMalloc(&q->tmp, bytes) != cudaSuccess) {
                cudaGetLastError();
                q->tmp = nullptr;
            }
        }
        long long all_tmp = 0;
        CM(q->comm->agree_min(q->tmp ? 1 : 0, &all_tmp, q->st));
        if (!all_tmp && q->tmp) {
            cudaFree(q->tmp);
            q->tmp = nullptr;
        }
        // fused swap: map every rank's two state buffers (CUDA IPC, or the loopback's pointers);
        // if any rank cannot map, all keep the separate swap
        const char *fz = std::getenv("QSIM_FUSED_SWAP");
        bool fuse = q->tmp && !q->user_buf && !(fz && std::atoi(fz) == 0);
        if (fuse) {
            q->bufs[0] = q->psi;
            q->bufs[1] = q->tmp;
            void *mp[2][8] = {};
            fuse = q->comm->share(q->bufs[0], bytes, mp[0], q->st);
            if (fuse && !q->comm->share(q->bufs[1], bytes, mp[1], q->st)) {
                q->comm->unshare(mp[0]);
                fuse = false;
            }
            for (int b = 0; b < 2 && fuse; ++b)
                for (int c = 0; c < world; ++c) q->peer[b][c] = (double2 *)mp[b][c];
        }
        // in-place fused swap: no second buffer (the n = 36 shape), peer stores into the peers'
        // current buffers after a per-slot handshake (PassParams::ip).  QSIM_FUSED_SWAP=0 keeps
        // the staged collective swap instead.
        if (!fuse && !q->tmp && !q->user_buf && q->m > qk::KT && !(fz && std::atoi(fz) == 0)) {
            const u64 nt = 1ull << (q->m - qk::KT);
            void *mp[8] = {}, *fp[8] = {};
            CK(cudaMalloc(&q->d_flags, sizeof(unsigned) * nt * world));
            CK(cudaMemsetAsync(q->d_flags, 0, sizeof(unsigned) * nt * world, q->st));
            CK(cudaHostAlloc(&q->h_err, sizeof(int), cudaHostAllocMapped));
            *q->h_err = 0;
            CK(cudaHostGetDevicePointer(&q->d_err, q->h_err, 0));
            CK(cudaStreamSynchronize(q->st));
            bool ok = q->comm->share(q->psi, bytes, mp, q->st);
            if (ok && !q->comm->share(q->d_flags, sizeof(unsigned) * nt * world, fp, q->st)) {
                q->comm->unshare(mp);
                ok = false;
            }
            if (ok) {
                for (int c = 0; c < world; ++c) {
                    q->peer[0][c] = (double2 *)mp[c];
                    q->fl_peer[c] = (unsigned *)fp[c];
                }
                q->bufs[0] = q->psi;
                q->ipfused = fuse = true;
                // loopback ranks on one device: the moving passes of all ranks must be resident
                // at once (they wait on each other's loads), so each takes 1/world of the SMs
                if (q->comm->shared_device()) q->grid_cap = std::max(1, q->num_sms / world);
            }
        }
        if (fuse) {
            q->fused_swap = true;
            q->cur = 0;
            // split swap: groups from the top run's bits below the swapped ones
            const TileSet &T = q->sets.back();
            int a_top = q->m;
            u64 tbits = 0;
            for (int i = 0; i < qk::KT; ++i)
                if ((T.own >> i) & 1u) {
                    a_top = std::min(a_top, T.L[i]);
                    tbits |= 1ull << T.L[i];
                }
            int seg = 0;  // contiguous top-set bits from a_top (a split top run has two segments)
            while (a_top + seg < q->m && ((tbits >> (a_top + seg)) & 1ull)) ++seg;
            q->mv_pshift = a_top;
            q->mv_pbits = std::min(std::min(10, seg), std::max(0, q->m - q->g - a_top));
            q->split = q->mv_pbits > 0 && q->sets.size() > 1;
            // default weights: equal shares for every pass of the layer (boundary turning run,
            // plain runs, the 12-bit set).  A non-boundary pass moves its share at almost no cost
            // when the moving tiles are interleaved with local ones; the boundary pass moves per
            // element (STG).  An earlier kernel made the boundary pass's STG stores cost ~1.7 ms
            // whatever its share, so G = 2 used "0,1,1" -- no longer the better choice (below).
            {
                q->lowswap = !q->ipfused && lowswap_layout(q->m, q->g) && q->sets.size() >= 3;
            }
            // (re-measured with the final pass kernels: equal shares are best at G = 2 too,
            // 20.7-20.9 vs 22.5 ms per layer with "0,1,1"; profiles/r1_mgpu2_split_weights.jsonl).
            // With four or more sets (m >= 31) the boundary pass moves nothing: a moving boundary
            // pass stores every element from registers (no TMA store), which cost ~20 ms of its
            // ~51 at n = 34 (in place, 2 B200s: 219 ms per layer with equal shares, 204 with
            // "0,1,1,1"; profiles/r2_mgpu2_split_weights.jsonl)
            q->split_w.clear();
            q->split_w.push_back(q->sets.size() >= 4 ? 0.0 : 1.0);
            for (int s2 = (int)q->sets.size() - 2; s2 >= 0; --s2) q->split_w.push_back(1.0);
            if (const char *w = std::getenv("QSIM_SPLIT_W")) {
                std::vector<double> ws;
                const char *c = w;
                while (*c) {
                    char *e = nullptr;
                    double v = std::strtod(c, &e);
                    if (e == c) break;
                    ws.push_back(v);
                    c = (*e == ',') ? e + 1 : e;
                }
                if (ws.size() == q->sets.size()) q->split_w = ws;
            }
        }
    }
    q->pending_plus = true;
    if (const char *e = std::getenv("QSIM_TMA_STORE")) q->tma_store = std::atoi(e) != 0;
    if (const char *e = std::getenv("QSIM_SP")) q->sp_frac = std::atof(e);
    if (const char *e = std::getenv("QSIM_L2PROMO")) {
        const int v = std::atoi(e);
        q->l2promo_run = v == 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                   : v == 64  ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                   : v == 0   ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                              : CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    }
    if (const char *e = std::getenv("QSIM_TMA_MOVES")) q->tma_moves = std::atoi(e) != 0;


    CK(qk::setup_tma_kernels());
    for (const TileSet &S : q->sets)
        if (!S.tm_ok) return fail(q, QSIM_EUNSUPPORTED, "tile set without a 5-D TMA view");
    return QSIM_OK;
}

}  // namespace

// =========================================================================== C-ABI
extern "C" {

int qsim_create(int n, int precision, qsim_t **out) {
    return qsim_create_ex(n, precision, 0, 1, nullptr, nullptr, 0, nullptr, out);
}

int qsim_create_ex(int n, int precision, int rank, int world, const void *nccl_unique_id, void *state_buf,
                   size_t buf_bytes, void *cuda_stream, qsim_t **out) {
    if (!out) return fail(nullptr, QSIM_EINVAL, "out is NULL");
    *out = nullptr;
    if (world > 1 && !nccl_unique_id) return fail(nullptr, QSIM_EINVAL, "nccl_unique_id is NULL");
    qsim *q = new qsim();
    int rc = create_common(q, n, precision, rank, world, nccl_unique_id, state_buf, buf_bytes, cuda_stream);
    if (rc != QSIM_OK) {
        g_create_error = q->err;
        qsim_destroy(q);
        return rc;
    }
    *out = q;
    return QSIM_OK;
}

int qsim_destroy(qsim_t *q) {
    if (!q) return QSIM_EINVAL;
    if (q->st) cudaStreamSynchronize(q->st);
    if (q->fused_swap) {
        if (q->comm) {  // no rank may unmap while a peer could still write into it
            q->comm->barrier(q->st);
            cudaStreamSynchronize(q->st);
            for (int b = 0; b < (q->ipfused ? 1 : 2); ++b) q->comm->unshare(reinterpret_cast<void **>(q->peer[b]));
            if (q->ipfused) q->comm->unshare(reinterpret_cast<void **>(q->fl_peer));
        }
    }
    if (q->d_flags) cudaFree(q->d_flags);
    if (q->d_maps) cudaFree(q->d_maps);
    if (q->h_err) cudaFreeHost(q->h_err);
    delete q->comm;
    if (q->psi && q->psi != q->user_buf) cudaFree(q->psi);
    if (q->tmp && q->tmp != q->user_buf) cudaFree(q->tmp);
    for (int k = 0; k < qsim::NFR; ++k)
        if (q->d_fr[k]) cudaFree(q->d_fr[k]);
    if (q->d_hlog) cudaFree(q->d_hlog);
    if (q->d_part) cudaFree(q->d_part);
    if (q->d_res) cudaFree(q->d_res);
    if (q->d_ang) cudaFree(q->d_ang);
    if (q->d_scratch) cudaFree(q->d_scratch);
    if (q->d_rec) cudaFree(q->d_rec);
    for (cudaEvent_t e : q->ev_pool) cudaEventDestroy(e);
    if (q->own_stream && q->st) cudaStreamDestroy(q->st);
    delete q;
    return QSIM_OK;
}

int qsim_set_ising(qsim_t *q, const double *h, const double *J) {
    if (!q) return QSIM_EINVAL;
    if (!h || !J) return fail(q, QSIM_EINVAL, "h or J is NULL");
    const int n = q->n;
    std::vector<double> hh(h, h + n), JJ((size_t)n * n, 0.0);
    for (int i = 0; i < n; ++i) {
        if (!std::isfinite(hh[i])) return fail(q, QSIM_EINVAL, "h contains NaN/Inf");
        if (J[(size_t)i * n + i] != 0.0) return fail(q, QSIM_EINVAL, "J has a non-zero (or NaN) diagonal entry");
        for (int j = i + 1; j < n; ++j) {
            double v = J[(size_t)i * n + j];
            if (!std::isfinite(v)) return fail(q, QSIM_EINVAL, "J contains NaN/Inf");
            JJ[(size_t)i * n + j] = v;
            JJ[(size_t)j * n + i] = v;
        }
    }
    q->h = hh;
    q->J = JJ;
    {
        std::vector<double> lg((size_t)n + (size_t)n * n);
        std::copy(hh.begin(), hh.end(), lg.begin());
        std::copy(JJ.begin(), JJ.end(), lg.begin() + n);
        CK(cudaMemcpyAsync(q->d_hlog, lg.data(), sizeof(double) * lg.size(), cudaMemcpyHostToDevice, q->st));
    }
    q->fr_valid = false;
    int rc = ensure_frame(q);
    if (rc) return rc;
    q->has_ising = true;
    q->res_valid = false;
    return QSIM_OK;
}

int qsim_init_plus(qsim_t *q) {
    if (!q) return QSIM_EINVAL;
    q->pending_plus = true;
    q->res_valid = false;
    return QSIM_OK;
}

int qsim_apply_qaoa(qsim_t *q, const double *gamma, const double *beta, int p) {
    if (!q) return QSIM_EINVAL;
    if (!gamma || !beta || p < 1) return fail(q, QSIM_EINVAL, "need gamma, beta and p >= 1");
    if (check_angles(gamma, p) || check_angles(beta, p)) return fail(q, QSIM_EINVAL, "angles contain NaN/Inf");
    if (!q->has_ising) return fail(q, QSIM_ESTATE, "qsim_set_ising not called");
    q->res_valid = false;
    return apply_layers(q, gamma, beta, p);
}

int qsim_aqa_angles(double T, int p, const double *s, const double *A, const double *B, int n_knots,
                    double *gamma_out, double *beta_out) {
    if (p < 2 || n_knots < 2 || !s || !A || !B || !gamma_out || !beta_out) return QSIM_EINVAL;
    if (!std::isfinite(T)) return QSIM_EINVAL;
    for (int j = 0; j < n_knots; ++j) {
        if (!std::isfinite(s[j]) || !std::isfinite(A[j]) || !std::isfinite(B[j])) return QSIM_EINVAL;
        if (j > 0 && !(s[j] > s[j - 1])) return QSIM_EINVAL;
    }
    if (s[0] != 0.0 || s[n_knots - 1] != 1.0) return QSIM_EINVAL;
    const double tau = T / p;  // t_anneal = (n_steps + 1) tau = p tau = T
    for (int k = 1; k <= p; ++k) {
        const double sk = (double)(k - 1) / (double)(p - 1);  // s_k = (k-1)/(p-1)
        gamma_out[k - 1] = tau * pwl(s, B, n_knots, sk);    // eq:gamma_k
        if (k < p) {
            const double sk1 = (double)k / (double)(p - 1);
            beta_out[k - 1] = -tau * (pwl(s, A, n_knots, sk1) + pwl(s, A, n_knots, sk)) / 2.0;  // eq:beta_k
        } else {
            beta_out[k - 1] = -tau * pwl(s, A, n_knots, sk) / 2.0;  // beta_p
        }
    }
    return QSIM_OK;
}

int qsim_apply_aqa(qsim_t *q, double T, int p, const double *s, const double *A, const double *B, int n_knots) {
    if (!q) return QSIM_EINVAL;
    if (p < 2) return fail(q, QSIM_EINVAL, "AQA needs p >= 2 (s_k = (k-1)/(p-1))");
    std::vector<double> g(p), b(p);
    if (qsim_aqa_angles(T, p, s, A, B, n_knots, g.data(), b.data()) != QSIM_OK)
        return fail(q, QSIM_EINVAL, "invalid schedule (knots must rise strictly from s=0 to s=1)");
    return qsim_apply_qaoa(q, g.data(), b.data(), p);
}

int qsim_apply_qsds(qsim_t *q, double tau, int n_steps, const double *s, const double *A, const double *B,
                    int n_knots) {
    if (!q) return QSIM_EINVAL;
    if (!q->has_ising) return fail(q, QSIM_ESTATE, "qsim_set_ising not called");
    if (n_steps < 0 || !s || !A || !B || n_knots < 2 || !std::isfinite(tau))
        return fail(q, QSIM_EINVAL, "need tau, n_steps >= 0 and a schedule");
    for (int j = 0; j < n_knots; ++j) {
        if (!std::isfinite(s[j]) || !std::isfinite(A[j]) || !std::isfinite(B[j])) return fail(q, QSIM_EINVAL, "NaN in schedule");
        if (j > 0 && !(s[j] > s[j - 1])) return fail(q, QSIM_EINVAL, "knots must rise strictly");
    }
    if (s[0] != 0.0 || s[n_knots - 1] != 1.0) return fail(q, QSIM_EINVAL, "knots must span [0, 1]");
    const int n = q->n, L = n_steps + 1;  // step operators l = 0..n_steps (eq. AQA4)
    // exact half-step exp[i tau/2 (A X - B h_q Z)] per qubit (AQA3), Z = diag(-1, +1)
    auto half = [&](int l, int a, std::complex<double> (&U)[4]) {
        const double sl = (double)l / (double)L;
        const double al = 0.5 * tau * pwl(s, A, n_knots, sl), bl = -0.5 * tau * pwl(s, B, n_knots, sl) * q->h[a];
        const double w = std::sqrt(al * al + bl * bl), c = std::cos(w), sw = w > 0.0 ? std::sin(w) / w : 1.0;
        U[0] = {c, -sw * bl};
        U[1] = {0.0, sw * al};
        U[2] = {0.0, sw * al};
        U[3] = {c, sw * bl};
    };
    // layers k = 0..L: mixer M_k (k = 0: U(0); 0 < k < L: U(k) U(k-1); k = L: U(L-1)), phase
    // gamma_k = tau B(s_{k-1}) on the J-only energy before mixer k (gamma_0 = 0)
    const int p = L + 1;
    std::vector<double2> G((size_t)p * n * 4);
    std::vector<double> gam(p, 0.0), bet(p, 0.0);
    for (int k = 0; k < p; ++k) {
        if (k > 0) gam[k] = tau * pwl(s, B, n_knots, (double)(k - 1) / (double)L);
        for (int a = 0; a < n; ++a) {
            std::complex<double> M[4];
            if (k == 0 || k == L) {
                half(k == 0 ? 0 : L - 1, a, M);
            } else {
                std::complex<double> Ua[4], Ub[4];
                half(k - 1, a, Ua);
                half(k, a, Ub);
                M[0] = Ub[0] * Ua[0] + Ub[1] * Ua[2];
                M[1] = Ub[0] * Ua[1] + Ub[1] * Ua[3];
                M[2] = Ub[2] * Ua[0] + Ub[3] * Ua[2];
                M[3] = Ub[2] * Ua[1] + Ub[3] * Ua[3];
            }
            for (int e = 0; e < 4; ++e) G[((size_t)k * n + a) * 4 + e] = make_double2(M[e].real(), M[e].imag());
        }
    }
    q->gmats = &G;
    q->frame_noh = true;
    q->res_valid = false;
    int rc = apply_layers(q, gam.data(), bet.data(), p);
    if (rc == QSIM_OK) rc = qsim_sync(q) == QSIM_OK ? QSIM_OK : QSIM_ECUDA;  // G must outlive the launches
    q->gmats = nullptr;
    q->frame_noh = false;
    q->res_valid = false;
    return rc;
}

int qsim_qaoa_batch(qsim_t *q, const double *gamma, const double *beta, int p, int count, double *out) {
    if (!q) return QSIM_EINVAL;
    if (!gamma || !beta || !out || p < 1 || count < 0) return fail(q, QSIM_EINVAL, "need gamma, beta, out, p >= 1, count >= 0");
    if (!q->has_ising) return fail(q, QSIM_ESTATE, "qsim_set_ising not called");
    if (q->world != 1 || q->n > qk::KT) return fail(q, QSIM_EUNSUPPORTED, "qsim_qaoa_batch needs n <= 12 on one GPU");
    if (check_angles(gamma, p * count) || check_angles(beta, p * count)) return fail(q, QSIM_EINVAL, "angles contain NaN/Inf");
    if (count == 0) return QSIM_OK;
    {
        int rc = ensure_frame(q);
        if (rc) return rc;
    }
    const size_t np = (size_t)p * count, dim = (size_t)1 << q->n;
    int rc = scratch(q, sizeof(double) * (2 * np + count + dim));
    if (rc) return rc;
    double *dg = (double *)q->d_scratch, *db = dg + np, *dout = db + np, *det = dout + count;
    CK(cudaMemcpyAsync(dg, gamma, sizeof(double) * np, cudaMemcpyHostToDevice, q->st));
    CK(cudaMemcpyAsync(db, beta, sizeof(double) * np, cudaMemcpyHostToDevice, q->st));
    qk::BatchParams B{};
    B.hp = q->cur_hp;
    B.Jp = q->cur_Jp;
    B.gamma = dg;
    B.beta = db;
    B.etab = det;
    B.out = dout;
    B.n = q->n;
    B.p = p;
    B.count = count;
    B.a0 = std::pow(2.0, -0.5 * q->n);
    CK(qk::launch_qaoa_batch(B, det, q->st));
    q->launches += 2;
    CK(cudaMemcpyAsync(out, dout, sizeof(double) * count, cudaMemcpyDeviceToHost, q->st));
    SYNC(q);
    return QSIM_OK;
}

int qsim_apply_hadamard(qsim_t *q, int reps) {
    if (!q) return QSIM_EINVAL;
    if (reps < 1) return fail(q, QSIM_EINVAL, "reps >= 1");
    if (!q->has_ising && q->J.empty()) {  // no problem data needed: the phase frame is all zero
        q->h.assign(q->n, 0.0);
        q->J.assign((size_t)q->n * q->n, 0.0);
        q->fr_valid = false;
    }
    const int n = q->n;
    const double r = std::sqrt(0.5);
    std::vector<double2> G((size_t)reps * n * 4);
    for (size_t i = 0; i < (size_t)reps * n; ++i) {
        G[4 * i + 0] = make_double2(r, 0.0);
        G[4 * i + 1] = make_double2(r, 0.0);
        G[4 * i + 2] = make_double2(r, 0.0);
        G[4 * i + 3] = make_double2(-r, 0.0);
    }
    std::vector<double> zero(reps, 0.0);
    q->gmats = &G;
    q->hmode = q->m > qk::KT;  // the tile kernels have a dedicated Hadamard butterfly
    q->frame_noh = true;
    q->res_valid = false;
    int rc = apply_layers(q, zero.data(), zero.data(), reps);
    if (rc == QSIM_OK) rc = qsim_sync(q) == QSIM_OK ? QSIM_OK : QSIM_ECUDA;
    q->gmats = nullptr;
    q->hmode = false;
    q->frame_noh = false;
    q->res_valid = false;
    return rc;
}

int qsim_expect_hc(qsim_t *q, double *out) {
    if (!q) return QSIM_EINVAL;
    if (!out) return fail(q, QSIM_EINVAL, "out is NULL");
    if (!q->has_ising) return fail(q, QSIM_ESTATE, "qsim_set_ising not called");
    int rc = run_reduce(q);
    if (rc) return rc;
    double r[2];
    CK(cudaMemcpyAsync(r, q->d_res, sizeof(r), cudaMemcpyDeviceToHost, q->st));
    SYNC(q);
    *out = r[0];
    return QSIM_OK;
}

int qsim_norm2(qsim_t *q, double *out) {
    if (!q) return QSIM_EINVAL;
    if (!out) return fail(q, QSIM_EINVAL, "out is NULL");
    if (!q->has_ising) return fail(q, QSIM_ESTATE, "qsim_set_ising not called");
    int rc = run_reduce(q);
    if (rc) return rc;
    double r[2];
    CK(cudaMemcpyAsync(r, q->d_res, sizeof(r), cudaMemcpyDeviceToHost, q->st));
    SYNC(q);
    *out = r[1];
    return QSIM_OK;
}

int qsim_success_prob(qsim_t *q, const uint64_t *gs, int count, double *out) {
    if (!q) return QSIM_EINVAL;
    if (!gs || count < 1 || !out) return fail(q, QSIM_EINVAL, "need ground_states, count >= 1, out");
    for (int i = 0; i < count; ++i)
        if (gs[i] >> q->n) return fail(q, QSIM_ERANGE, "ground state label >= 2^n");
    std::vector<double> amp(2 * (size_t)count);
    int rc = gather_host(q, 0, (u64)count, gs, amp.data());
    if (rc) return rc;
    double acc = 0.0;
    for (int i = 0; i < count; ++i) acc += amp[2 * i] * amp[2 * i] + amp[2 * i + 1] * amp[2 * i + 1];
    *out = acc;
    return QSIM_OK;
}

int qsim_get_amplitudes(qsim_t *q, uint64_t first, uint64_t count, double *out) {
    if (!q) return QSIM_EINVAL;
    if (!out && count) return fail(q, QSIM_EINVAL, "out is NULL");
    if (count == 0) return QSIM_OK;
    if (first >> q->n || count > (1ull << q->n) - first) return fail(q, QSIM_ERANGE, "range exceeds 2^n");
    return gather_host(q, first, count, nullptr, out);
}

int qsim_energies(qsim_t *q, uint64_t first, uint64_t count, double *out) {
    if (!q) return QSIM_EINVAL;
    if (!out && count) return fail(q, QSIM_EINVAL, "out is NULL");
    if (!q->has_ising) return fail(q, QSIM_ESTATE, "qsim_set_ising not called");
    if (count == 0) return QSIM_OK;
    if (first >> q->n || count > (1ull << q->n) - first) return fail(q, QSIM_ERANGE, "range exceeds 2^n");
    {
        int rc = ensure_frame(q);
        if (rc) return rc;
    }
    // the hot path's arithmetic: tile records of set 0 (flip 0: energies at the physical labels)
    // from tile_fields_kernel, then the frame-Z sums of the reducing pass (energy_dump_kernel)
    qk::PassParams P{};
    if (q->m > qk::KT) {
        P = base_params(q, q->sets[0]);
        P.flip = 0;
        P.rec = q->d_rec;
        CK(qk::launch_tile_fields(P, q->d_rec, q->st));
        q->launches++;
    } else {
        P.hp = q->cur_hp;
        P.Jp = q->cur_Jp;
    }
    const u64 CH = 1ull << 23;
    for (u64 done = 0; done < count; done += CH) {
        u64 c = std::min(CH, count - done);
        int rc = scratch(q, c * sizeof(double));
        if (rc) return rc;
        qk::GatherParams G = gather_params(q, first + done, c, nullptr);
        CK(qk::launch_energy_dump(G, P, (double *)q->d_scratch, (int)std::min<u64>((c + 255) / 256, 4096), q->st));
        q->launches++;
        if (q->world > 1) CM(q->comm->allreduce((double *)q->d_scratch, c, qc::Op::Sum, q->st));
        CK(cudaMemcpyAsync(out + done, q->d_scratch, c * sizeof(double), cudaMemcpyDeviceToHost, q->st));
        SYNC(q);
    }
    return QSIM_OK;
}

int qsim_spin_expectations(qsim_t *q, double *out) {
    if (!q) return QSIM_EINVAL;
    if (!out) return fail(q, QSIM_EINVAL, "out is NULL");
    if (q->m <= qk::KT) {  // small states: amplitudes are few; gather and sum in the fixed order
        const u64 dim = 1ull << q->n;
        std::vector<double> amp(2 * dim);
        int rc = gather_host(q, 0, dim, nullptr, amp.data());
        if (rc) return rc;
        for (int i = 0; i < q->n; ++i) {
            double acc = 0.0;
            for (u64 z = 0; z < dim; ++z)
                acc += (amp[2 * z] * amp[2 * z] + amp[2 * z + 1] * amp[2 * z + 1]) * (((z >> i) & 1) ? 1.0 : -1.0);
            out[i] = acc;
        }
        return QSIM_OK;
    }
    int rc = materialize_plus(q);
    if (rc) return rc;
    const TileSet &S = q->sets[0];
    qk::PassParams P = base_params(q, S);
    P.flip = q->flip;
    const int grid = grid_for(q, S.ntiles);
    rc = scratch(q, sizeof(double) * ((size_t)grid * q->n + q->n));
    if (rc) return rc;
    double *part = (double *)q->d_scratch, *vec = part + (size_t)grid * q->n;
    CK(qk::launch_spin(P, part, grid, q->st));
    CK(qk::launch_sum_vec(part, grid, q->n, vec, q->st));
    q->launches += 2;
    if (q->world > 1) CM(q->comm->allreduce(vec, q->n, qc::Op::Sum, q->st));
    std::vector<double> phys(q->n);
    CK(cudaMemcpyAsync(phys.data(), vec, sizeof(double) * q->n, cudaMemcpyDeviceToHost, q->st));
    SYNC(q);
    for (int a = 0; a < q->n; ++a) out[a] = phys[q->pos[a]];  // flips already folded in
    return QSIM_OK;
}

int qsim_apply_aqa_traced(qsim_t *q, double T, int p, const double *s, const double *A, const double *B,
                          int n_knots, double *trace) {
    if (!q) return QSIM_EINVAL;
    if (p < 2) return fail(q, QSIM_EINVAL, "AQA needs p >= 2 (s_k = (k-1)/(p-1))");
    if (!trace) return fail(q, QSIM_EINVAL, "trace is NULL");
    std::vector<double> g(p), b(p);
    if (qsim_aqa_angles(T, p, s, A, B, n_knots, g.data(), b.data()) != QSIM_OK)
        return fail(q, QSIM_EINVAL, "invalid schedule (knots must rise strictly from s=0 to s=1)");
    for (int k = 0; k < p; ++k) {
        int rc = qsim_apply_qaoa(q, &g[k], &b[k], 1);
        if (rc) return rc;
        rc = qsim_spin_expectations(q, trace + (size_t)k * q->n);
        if (rc) return rc;
    }
    return QSIM_OK;
}

int qsim_ground_states(qsim_t *q, uint64_t *out, int max_out, double *emin_out, uint64_t *count_out) {
    if (!q) return QSIM_EINVAL;
    if (!emin_out || !count_out || max_out < 0 || (max_out > 0 && !out)) return fail(q, QSIM_EINVAL, "bad outputs");
    if (!q->has_ising) return fail(q, QSIM_ESTATE, "qsim_set_ising not called");
    if (q->n < qk::KT) return fail(q, QSIM_EUNSUPPORTED, "enumeration needs n >= 12");
    const u64 ntiles = 1ull << (q->n - qk::KT);
    const u64 u0 = ntiles * (u64)q->rank / (u64)q->world, u1 = ntiles * (u64)(q->rank + 1) / (u64)q->world;
    const int grid = (int)std::max<u64>(1, std::min<u64>((u64)q->num_sms * 8, u1 - u0));
    const int cap = std::max(max_out, 1);
    // collect pass: every CTA keeps the first `cap` minimisers of its tiles (ascending); the
    // merged lists contain the global first `cap` (per-CTA slots bounded to 2^24 labels)
    const int cgrid = (int)std::max<u64>(1, std::min<u64>((u64)grid, (1ull << 24) / (u64)cap));
    int rc = scratch(q, sizeof(double) * (grid + 1) + sizeof(unsigned long long) * 2 + sizeof(unsigned) * cgrid +
                            sizeof(u64) * (size_t)cap * cgrid + 16);
    if (rc) return rc;
    double *part = (double *)q->d_scratch, *res = part + grid;
    unsigned long long *cnt = (unsigned long long *)(res + 1);
    unsigned *ccnt = (unsigned *)(cnt + 2);
    u64 *lst = (u64 *)(((uintptr_t)(ccnt + cgrid) + 15) & ~(uintptr_t)15);
    qk::EnumParams E{};
    E.h = q->d_hlog;
    E.J = q->d_hlog + q->n;
    E.n = q->n;
    E.u0 = u0;
    E.u1 = u1;
    E.part = part;
    E.collect = 0;
    CK(qk::launch_enum(E, grid, q->st));
    CK(qk::launch_min_partials(part, grid, res, q->st));
    q->launches += 2;
    if (q->world > 1) CM(q->comm->allreduce(res, 1, qc::Op::Min, q->st));
    double emin = 0.0;
    CK(cudaMemcpyAsync(&emin, res, sizeof(double), cudaMemcpyDeviceToHost, q->st));
    CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), q->st));
    CK(cudaStreamSynchronize(q->st));
    E.collect = 1;
    E.emin = emin;
    E.out = lst;
    E.cta_cnt = ccnt;
    E.count = cnt;
    E.max_out = cap;
    CK(qk::launch_enum(E, cgrid, q->st));
    q->launches++;
    unsigned long long c = 0;
    std::vector<unsigned> cc(cgrid);
    std::vector<u64> lists((size_t)cap * cgrid);
    CK(cudaMemcpyAsync(&c, cnt, sizeof(c), cudaMemcpyDeviceToHost, q->st));
    CK(cudaMemcpyAsync(cc.data(), ccnt, sizeof(unsigned) * cgrid, cudaMemcpyDeviceToHost, q->st));
    CK(cudaMemcpyAsync(lists.data(), lst, sizeof(u64) * lists.size(), cudaMemcpyDeviceToHost, q->st));
    CK(cudaStreamSynchronize(q->st));
    std::vector<u64> mine;
    for (int b = 0; b < cgrid; ++b)
        for (unsigned k = 0; k < std::min<unsigned>(cc[b], (unsigned)cap); ++k) mine.push_back(lists[(size_t)b * cap + k]);
    std::sort(mine.begin(), mine.end());
    if (mine.size() > (size_t)cap) mine.resize(cap);
    std::vector<u64> all = mine;
    unsigned long long total = c;
    if (q->world > 1) {  // gather every rank's (count, first cap labels)
        const size_t rec = 1 + (size_t)cap;
        std::vector<u64> sendv(rec, ~0ull), recv(rec * q->world);
        sendv[0] = c;
        std::copy(mine.begin(), mine.end(), sendv.begin() + 1);
        u64 *d = nullptr;
        CK(cudaMalloc(&d, sizeof(u64) * rec * (1 + q->world)));
        CK(cudaMemcpyAsync(d, sendv.data(), sizeof(u64) * rec, cudaMemcpyHostToDevice, q->st));
        CM(q->comm->allgather(d, d + rec, rec * sizeof(u64), q->st));
        CK(cudaMemcpyAsync(recv.data(), d + rec, sizeof(u64) * rec * q->world, cudaMemcpyDeviceToHost, q->st));
        CK(cudaStreamSynchronize(q->st));
        cudaFree(d);
        all.clear();
        total = 0;
        for (int r = 0; r < q->world; ++r) {
            total += recv[r * rec];
            for (size_t k = 0; k < (size_t)std::min<u64>(recv[r * rec], (u64)cap); ++k) all.push_back(recv[r * rec + 1 + k]);
        }
        std::sort(all.begin(), all.end());
    }
    for (int k = 0; k < max_out && k < (int)all.size(); ++k) out[k] = all[k];
    *emin_out = emin;
    *count_out = total;
    return QSIM_OK;
}

int qsim_enumerate(int n, const double *h, const double *J, uint64_t *out, int max_out, double *emin_out,
                   uint64_t *count_out, double *ms_out) {
    if (n < qk::KT || n > 48 || !h || !J || !emin_out || !count_out || max_out < 0 || (max_out > 0 && !out))
        return fail(nullptr, QSIM_EINVAL, "qsim_enumerate: bad arguments (12 <= n <= 48)");
    qsim *q = new qsim();  // a state-less handle: frames and scratch only
    q->n = n;
    q->m = n;
    int rc = QSIM_OK;
    auto body = [&]() -> int {
        CK(cudaGetDevice(&q->dev));
        CK(cudaDeviceGetAttribute(&q->num_sms, cudaDevAttrMultiProcessorCount, q->dev));
        CK(cudaStreamCreateWithFlags(&q->st, cudaStreamNonBlocking));
        q->own_stream = true;
        std::vector<double> lg((size_t)n + (size_t)n * n, 0.0);
        for (int i = 0; i < n; ++i) {
            if (!std::isfinite(h[i])) return fail(q, QSIM_EINVAL, "h contains NaN/Inf");
            lg[i] = h[i];
            for (int j = i + 1; j < n; ++j) {
                const double v = J[(size_t)i * n + j];
                if (!std::isfinite(v)) return fail(q, QSIM_EINVAL, "J contains NaN/Inf");
                lg[n + (size_t)i * n + j] = lg[n + (size_t)j * n + i] = v;
            }
        }
        CK(cudaMalloc(&q->d_hlog, sizeof(double) * lg.size()));
        CK(cudaMemcpyAsync(q->d_hlog, lg.data(), sizeof(double) * lg.size(), cudaMemcpyHostToDevice, q->st));
        q->has_ising = true;
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0, q->st));
        int r = qsim_ground_states(q, out, max_out, emin_out, count_out);
        CK(cudaEventRecord(e1, q->st));
        CK(cudaEventSynchronize(e1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (ms_out) *ms_out = ms;
        return r;
    };
    rc = body();
    if (rc != QSIM_OK) g_create_error = q->err;
    qsim_destroy(q);
    return rc;
}

int qsim_sync(qsim_t *q) {
    if (!q) return QSIM_EINVAL;
    SYNC(q);
    return QSIM_OK;
}

int qsim_plan_counts(int n, int world, int p, int *passes_out, int *swaps_out, uint64_t *amps_sent_out) {
    int g = ilog2(world);
    if (n < 1 || n > qk::NMAX || world < 1 || world > 8 || g < 0 || p < 1) return QSIM_EINVAL;
    int m = n - g;
    if (world > 1 && m < qk::KT + 3) return QSIM_EINVAL;
    int passes = 0, swaps = 0;
    if (m <= qk::KT) {
        passes = 1;
    } else {
        std::vector<double> z(p, 0.0);
        const int ns = (int)build_sets(m).size();
        auto ops = build_schedule(ns, g, p, z.data(), z.data(), true, g > 0, nullptr, lowswap_layout(m, g) && ns >= 3);
        passes = (int)ops.size();
        for (auto &o : ops) swaps += (o.swap_after || o.swap_fused) ? 1 : 0;
    }
    if (passes_out) *passes_out = passes;
    if (swaps_out) *swaps_out = swaps;
    if (amps_sent_out) *amps_sent_out = g ? (uint64_t)(world - 1) << (m - g) : 0;
    return QSIM_OK;
}

int qsim_plan_positions(int n, int world, int layers, int *pos_out) {
    int g = ilog2(world);
    if (n < 1 || n > qk::NMAX || g < 0 || world > 8 || layers < 0 || !pos_out) return QSIM_EINVAL;
    int m = n - g;
    const bool low = lowswap_layout(m, g) && build_sets(m).size() >= 3;
    for (int qb = 0; qb < n; ++qb)
        pos_out[qb] = low ? phys_pos_low(n, m, g, layers & 1, qb) : phys_pos(n, m, g, layers & 1, qb);
    return QSIM_OK;
}

int qsim_bench_pass(qsim_t *q, int set, int phase, int reps, double *ms_out) {
    if (!q || !ms_out || reps < 1) return QSIM_EINVAL;
    const int ns = (int)q->sets.size();
    if (q->m <= qk::KT || set < 0 || set >= ns) return fail(q, QSIM_EINVAL, "no such tile set");
    if (!q->has_ising) return fail(q, QSIM_ESTATE, "qsim_set_ising not called");
    int rc = materialize_plus(q);
    if (rc) return rc;
    rc = ensure_frame(q);
    if (rc) return rc;
    const TileSet &S = q->sets[set];
    qk::PassParams P = base_params(q, S);
    std::complex<double> k1, k2;
    P.c1 = mix_coef(0.3, k1);
    P.c2 = mix_coef(-0.2, k2);
    // phase < 0: memory-pattern probes: -1 copy, -2 read only, -3 write only (no butterflies)
    P.mix1 = phase < 0 ? 0u : S.own;
    P.mix2 = phase > 0 ? S.own : 0u;
    P.dbg = phase == -2 ? 1 : (phase == -3 ? 2 : 0);
    if (phase < 0) phase = 0;
    std::complex<double> sc = cpow_int(k1, __builtin_popcount(P.mix1)) * cpow_int(k2, __builtin_popcount(P.mix2));
    P.scale = make_double2(sc.real(), sc.imag());
    P.kind = S.full12 ? (phase ? qk::K_TURN12 : qk::K_PLAIN12) : (phase ? qk::K_TURN_RUN : qk::K_PLAIN_RUN);
    P.phase = phase;
    P.gamma = 0.1;
    P.rec = q->d_rec;
    P.flip = q->flip;
    P.pw = P.dbg ? 0 : pw_eligible(q, S, P);
    CK(qk::launch_tile_fields(P, q->d_rec, q->st));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    int grid = 0;
    rc = launch_pass(q, S, P, &grid);  // warm-up
    if (rc) return rc;
    CK(cudaEventRecord(e0, q->st));
    for (int r = 0; r < reps; ++r) {
        rc = launch_pass(q, S, P, &grid);
        if (rc) return rc;
    }
    CK(cudaEventRecord(e1, q->st));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    q->res_valid = false;
    *ms_out = ms / reps;
    return QSIM_OK;
}

int qsim_profile_enable(qsim_t *q, int on) {
    if (!q) return QSIM_EINVAL;
    q->prof = on != 0;
    q->ev_used = 0;
    q->prof_bytes.clear();
    q->prof_kind.clear();
    return QSIM_OK;
}

int qsim_profile_read(qsim_t *q, double *ms_sum, uint64_t *count, double *bytes_sum) {
    if (!q || !ms_sum || !count || !bytes_sum) return QSIM_EINVAL;
    CK(cudaStreamSynchronize(q->st));
    double ms = 0.0, by = 0.0;
    size_t npass = q->ev_used / 2;
    for (size_t i = 0; i < npass; ++i) {
        float t = 0.f;
        CK(cudaEventElapsedTime(&t, q->ev_pool[2 * i], q->ev_pool[2 * i + 1]));
        ms += t;
        by += q->prof_bytes[i];
    }
    *ms_sum = ms;
    *count = npass;
    *bytes_sum = by;
    q->ev_used = 0;
    q->prof_bytes.clear();
    q->prof_kind.clear();
    return QSIM_OK;
}

int qsim_profile_passes(qsim_t *q, double *ms_out, int *kind_out, int cap) {
    if (!q || (cap > 0 && !ms_out)) return QSIM_EINVAL;
    CK(cudaStreamSynchronize(q->st));
    const int npass = (int)(q->ev_used / 2);
    for (int i = 0; i < npass && i < cap; ++i) {
        float t = 0.f;
        CK(cudaEventElapsedTime(&t, q->ev_pool[2 * i], q->ev_pool[2 * i + 1]));
        ms_out[i] = t;
        if (kind_out) kind_out[i] = q->prof_kind[i];
    }
    q->ev_used = 0;
    q->prof_bytes.clear();
    q->prof_kind.clear();
    return npass;
}

uint64_t qsim_kernel_launches(const qsim_t *q) { return q ? q->launches : 0; }

int qsim_num_qubits(const qsim_t *q) { return q ? q->n : QSIM_EINVAL; }

int qsim_swap_path(const qsim_t *q) {
    if (!q) return QSIM_EINVAL;
    if (q->world == 1) return QSIM_SWAP_NONE;
    if (q->ipfused) return QSIM_SWAP_FUSED_INPLACE;
    if (q->fused_swap) return q->lowswap ? QSIM_SWAP_LOWBIT : (q->split ? QSIM_SWAP_FUSED_SPLIT : QSIM_SWAP_FUSED);
    return q->tmp ? QSIM_SWAP_COLLECTIVE : QSIM_SWAP_INPLACE_STAGED;
}

const char *qsim_last_error(const qsim_t *q) { return q ? q->err.c_str() : g_create_error.c_str(); }

const char *qsim_version(void) { return "qsim-b200 0.2 (sm_100a, FP64 + FP32 mode)"; }

int qsim_loopback_id(int world, void *out128) {
    if (!out128 || world < 1 || world > 8 || ilog2(world) < 0) return QSIM_EINVAL;
    return qc::make_loopback_id(world, out128) == 0 ? QSIM_OK : QSIM_EINVAL;
}

int qsim_nccl_unique_id(void *out128) {
    if (!out128) return QSIM_EINVAL;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return QSIM_ENCCL;
    std::memcpy(out128, &id, sizeof(id));
    return QSIM_OK;
}

}  // extern "C"
