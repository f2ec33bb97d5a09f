/*
 * qsim.h -- C-ABI of the B200-native (sm_100a) FP64 state-vector engine for the
 * QAOA / AQA hot path of arXiv:2104.03293 ("GPU-accelerated simulations of quantum
 * annealing and the quantum approximate optimization algorithm", JUQCS-G).
 *
 * Citations "P:<line>" refer to the paper's LaTeX source, equation labels
 * are the paper's (eq:HC, eq:QAOA_state, eq:beta_k, eq:gamma_k, ...).
 *
 * Conventions shared by every call (readings R1-R4):
 *   - n qubits; basis label z in [0, 2^n); qubit j <-> bit j of z (little endian).
 *   - spin s_j(z) = 2 bit_j(z) - 1: |0> is the -1 and |1> the +1 eigenstate of
 *     sigma^z_j.
 *   - H_C = sum_i h_i sigma^z_i + sum_{i<j} J_ij sigma^z_i sigma^z_j (eq:HC):
 *     E(z) = sum_i h_i s_i + sum_{i<j} J_ij s_i s_j.  The constant C of eq:HCC is not
 *     part of H_C (global phase) and never enters any result.
 *   - H_D = sum_i sigma^x_i.
 *   - amplitudes are complex128, passed as interleaved (re, im) doubles.
 *
 * Ownership and threading:
 *   - a qsim_t* is owned by the caller from create until destroy; all pointer
 *     arguments are host pointers unless stated otherwise, read (or written) during
 *     the call only, never retained.
 *   - single writer per handle: calls on one handle must not run concurrently.
 *   - qsim_apply_* and qsim_init_plus enqueue work on the handle's CUDA stream and
 *     may return before it completes; calls that return values to the host
 *     (expect_hc, norm2, success_prob, get_amplitudes, energies, sync) synchronise.
 *   - multi-GPU handles (world > 1) are SPMD collectives: every rank makes the same
 *     calls with the same arguments, and scalar / gathered results are returned on
 *     every rank.
 *
 * Errors: every int-returning call returns QSIM_OK (0) or a negative QSIM_E* code;
 * qsim_last_error() describes the most recent failure on that handle.  A call that
 * fails with QSIM_EINVAL / QSIM_ERANGE / QSIM_ESTATE leaves the state unchanged.
 * QSIM_ECUDA / QSIM_ENCCL leave the handle unusable except for destroy.
 */
#ifndef QSIM_H
#define QSIM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct qsim qsim_t; /* opaque */

enum {
    QSIM_OK = 0,
    QSIM_EINVAL = -1,      /* bad argument: NULL pointer, NaN/Inf, p < 1, n out of range */
    QSIM_ENOMEM = -2,      /* device memory capacity exceeded for 2^n amplitudes */
    QSIM_ERANGE = -3,      /* basis index out of [0, 2^n) */
    QSIM_ESTATE = -4,      /* qsim_set_ising not called yet */
    QSIM_EUNSUPPORTED = -5,/* configuration not supported (e.g. QSIM_FP32 without the TMA kernel) */
    QSIM_ECUDA = -6,       /* CUDA runtime error (message in qsim_last_error) */
    QSIM_ENCCL = -7        /* NCCL error (multi-GPU handles) */
};

/* Amplitude precision.  QSIM_FP64 is the north-star path (complex128 amplitudes).  QSIM_FP32
 * (the precision of the paper's Table I GPU timings) stores
 * complex64 amplitudes (8 bytes each, half the HBM traffic) and runs the butterflies and phase
 * multiplications in FP32; energies E(z), tile fields and phase tables stay FP64 (E is still
 * exact), reductions accumulate in FP64, and readback converts to FP64.  Error bound and
 * tests: DESIGN.md §9. */
enum { QSIM_FP64 = 0, QSIM_FP32 = 1 };

/* Create a single-GPU handle on the current CUDA device for an n-qubit state
 * (1 <= n <= 40; the library allocates 16 * 2^n bytes of device memory (8 * 2^n for
 * QSIM_FP32), QSIM_ENOMEM if that fails).  The state starts as |+>^n.  precision is
 * QSIM_FP64 or QSIM_FP32 (else QSIM_EINVAL). */
int qsim_create(int n, int precision, qsim_t **out);

/* Multi-GPU / embedding variant.  The state is partitioned over `world` = 2^g ranks
 * on its top g physical qubits (the "global" qubits): rank r holds the
 * 2^(n-g) amplitudes whose global bits equal r.  `nccl_unique_id` points to 128 bytes
 * identifying the rank group (ignored when world == 1); a group id initialises exactly one
 * communicator, so use a fresh id per handle.  Two kinds:
 *   - an ncclUniqueId from qsim_nccl_unique_id (rank 0 creates it and broadcasts the bytes):
 *     one process per GPU, NCCL over NVLink, peer buffers mapped with CUDA IPC;
 *   - a loopback id from qsim_loopback_id: the `world` ranks are threads of ONE process, each
 *     creating its handle with the same id on its thread's current device and driving it from
 *     its own thread (every call is still a collective).  All ranks on one device = the one-GPU
 *     test mode of every multi-GPU swap path; one device per rank = a single-process multi-GPU
 *     run (peer access enabled between the devices; e.g. for ncu, which cannot follow a
 *     multi-process NCCL job).  Each rank owns its shard buffers and stream; collectives are
 *     stream-ordered with CUDA events and a host barrier; the pass kernels store into the
 *     peers' buffers exactly as over NVLink with IPC mappings.
 * `state_buf` (device pointer, optional) provides caller-owned storage of buf_bytes >= 16 *
 * 2^(n-g) bytes (the library then does not allocate the state); `cuda_stream` (cudaStream_t,
 * optional) is the stream all work is enqueued on.  world must be a power of two <= 8 with
 * n - g >= 15 (QSIM_EUNSUPPORTED otherwise).  Every rank takes the same swap path: the ranks
 * agree (minimum over ranks) on whether a second shard buffer fits and whether the peer
 * mappings succeeded. */
int qsim_create_ex(int n, int precision, int rank, int world, const void *nccl_unique_id,
                   void *state_buf, size_t buf_bytes, void *cuda_stream, qsim_t **out);

int qsim_destroy(qsim_t *q);

/* Upload the Ising problem (eq:HC): h[n] and J[n*n] row-major, of which the entries with
 * i < j are read (the lower triangle is ignored).  Values must be finite and the diagonal
 * J[i*n + i] zero (QSIM_EINVAL otherwise; eq:HC has no self-coupling).
 * E(z) is bit-exact when every h_i, J_ij is a multiple of 2^-m with
 * sum |coef| 2^m < 2^53 (dyadic data such as the paper's half-integer exact-cover
 * fields); other data is accepted without the bit-exactness claim. */
int qsim_set_ising(qsim_t *q, const double *h, const double *J);

/* Reset the state to |+>^n: psi_z = 2^(-n/2).  Applied lazily: the
 * first pass of the next qsim_apply_* writes it instead of reading the state. */
int qsim_init_plus(qsim_t *q);

/* Apply p QAOA layers to the current state (eq:QAOA_state, with the order
 * of Appendix A): for k = 1..p, psi <- e^{-i beta_k H_D} e^{-i gamma_k H_C} psi,
 * i.e. the cost phase psi_z <- e^{-i gamma_k E(z)} psi_z followed by the mixer
 * e^{-i beta_k sigma^x} on every qubit ("rotations around the x axis with angle
 * 2 beta_k").  gamma[p], beta[p] are used as given (never reduced modulo
 * pi / 2 pi).  p >= 1. */
int qsim_apply_qaoa(qsim_t *q, const double *gamma, const double *beta, int p);

/* AQA / second-order QAOA initialisation (eq:beta_k, eq:gamma_k,
 * P:338-347): tau = T/p (t_anneal = (n_steps + 1) tau = T), s_k = (k-1)/(p-1)
 * for k = 1..p (== k'/n_steps, k' = 0..n_steps, n_steps = p-1), A and B piecewise
 * linear through the n_knots knots (s[0] = 0 < ... < s[n_knots-1] = 1),
 *   beta_k = -tau (A(s_{k+1}) + A(s_k)) / 2 (k < p),  beta_p = -tau A(s_p) / 2,
 *   gamma_k = tau B(s_k),
 * then exactly qsim_apply_qaoa(gamma, beta, p).  A, B are in angular units per unit
 * of T (no 2 pi applied; reading R7).  p >= 2 (reading R8). */
int qsim_apply_aqa(qsim_t *q, double T, int p, const double *s, const double *A, const double *B,
                   int n_knots);

/* the QSDS "combined" second-order Suzuki-Trotter stepping of eq. AQA4
 * applied to the current state for l = 0..n_steps:
 *   exp[i tau/2 sum_i (A sigma^x_i - B h_i sigma^z_i)] exp[-i tau B sum_{i<j} J_ij s_i s_j]
 *   exp[i tau/2 sum_i (A sigma^x_i - B h_i sigma^z_i)],  A, B at s_l = l / (n_steps + 1)
 * (AQA0-AQA3: h~x = A, h~z_i = -B h_i, J~z = -B J; t_anneal = (n_steps + 1) tau), each
 * single-spin exponential exact.  Consecutive half-steps are merged into one per-qubit
 * 2x2 unitary, so n_steps + 2 general-mixer layers run on the tile-pass kernels.  A, B in
 * angular units per unit of tau. */
int qsim_apply_qsds(qsim_t *q, double tau, int n_steps, const double *s, const double *A, const double *B,
                    int n_knots);

/* apply `reps` layers of H on every qubit, (H^{otimes n})^reps -- the paper's
 * Hadamard benchmark circuit (H^N)^11 (Table I) -- with the general-mixer tile passes
 * (12 gates per HBM sweep); no phase, so no qsim_set_ising is needed. */
int qsim_apply_hadamard(qsim_t *q, int reps);

/* Batched QAOA expectation values for small problems (n <= 12, one GPU): for each of the `count`
 * angle sets b, <H_C> of |beta_b, gamma_b> (eq:QAOA_state, p layers from |+>)
 * into out[b]; gamma, beta are [count][p] row-major host arrays.  One CTA per angle set with the
 * whole state in shared memory -- the parameter-grid scans of the paper's Fig. 3 in one
 * launch.  The handle's state is not touched.  QSIM_EUNSUPPORTED for n > 12 or world > 1. */
int qsim_qaoa_batch(qsim_t *q, const double *gamma, const double *beta, int p, int count, double *out);

/* Host-only helper (no device work): the angles qsim_apply_aqa uses. */
int qsim_aqa_angles(double T, int p, const double *s, const double *A, const double *B,
                    int n_knots, double *gamma_out, double *beta_out);

/* <H_C> = sum_z |psi_z|^2 E(z) (E_p(beta, gamma)), constant C excluded. */
int qsim_expect_hc(qsim_t *q, double *out);

/* ||psi||^2 = sum_z |psi_z|^2. */
int qsim_norm2(qsim_t *q, double *out);

/* Success probability sum_{z in ground_states} |psi_z|^2.  count >= 1,
 * every label < 2^n (QSIM_ERANGE otherwise). */
int qsim_success_prob(qsim_t *q, const uint64_t *ground_states, int count, double *out);

/* Copy amplitudes psi_z for z = first .. first+count-1 in LOGICAL order (any qubit
 * relabelling done by the multi-GPU engine is undone) to out[2*count]. */
int qsim_get_amplitudes(qsim_t *q, uint64_t first, uint64_t count, double *out);

/* Test / diagnostic: E(z) for z = first .. first+count-1, computed on the device with the hot
 * path's own arithmetic: the per-tile records of tile_fields_kernel (12-bit set) and the register
 * tree of the reducing pass (frame Z), in the same summation order (for n <= 12 the small-state
 * kernel's direct sum).  Multi-GPU: the rank owning each label computes it, the others add zero. */
int qsim_energies(qsim_t *q, uint64_t first, uint64_t count, double *out);

/* spin expectations <sigma^z_i> = sum_z |psi_z|^2 s_i(z), i = 0..n-1 in
 * logical order ("spin expectation values during the time evolution"; Fig. 5). */
int qsim_spin_expectations(qsim_t *q, double *out);

/* qsim_apply_aqa that also records <sigma^z_i> after every layer k into trace[k*n + i]
 * (p*n doubles).  Layers are applied one at a time (P passes per layer instead of P-1). */
int qsim_apply_aqa_traced(qsim_t *q, double T, int p, const double *s, const double *A, const double *B,
                          int n_knots, double *trace);

/* full enumeration of E(z) over all 2^n labels on the GPU(s) (the paper's
 * t_FE): the minimum energy, the number of minimisers, and the first
 * max_out minimisers in ascending label order.  Needs n >= 12.  Independent of the state. */
int qsim_ground_states(qsim_t *q, uint64_t *out, int max_out, double *emin, uint64_t *count);

/* State-less variant on the current device (no 2^n state is allocated, so n may exceed
 * what fits in memory, 12 <= n <= 48): same results as qsim_ground_states, plus the
 * device time in *ms_out (optional).  Errors are reported by qsim_last_error(NULL). */
int qsim_enumerate(int n, const double *h, const double *J, uint64_t *out, int max_out, double *emin,
                   uint64_t *count, double *ms_out);

/* Wait for all work enqueued on the handle's stream. */
int qsim_sync(qsim_t *q);

/* Host-only planner introspection (no device work): for an n-qubit state on `world`
 * GPUs and p layers, the number of full HBM passes over the local shard and of
 * global-qubit swaps one qsim_apply_qaoa performs, and the amplitudes each rank
 * sends per swap.  Returns QSIM_EINVAL for unsupported layouts. */
int qsim_plan_counts(int n, int world, int p, int *passes_out, int *swaps_out,
                     uint64_t *amps_sent_per_swap_out);

/* Host-only: the physical bit positions of the qubits after `layers` swaps of the
 * multi-GPU schedule (pos_out[q] = physical position of logical qubit q). */
int qsim_plan_positions(int n, int world, int layers, int *pos_out);

/* Multi-GPU bootstrap helper: write a fresh ncclUniqueId (128 bytes) to out128 (call on
 * rank 0, broadcast the bytes, pass them to qsim_create_ex on every rank). */
int qsim_nccl_unique_id(void *out128);

/* Loopback test transport: write a fresh 128-byte group id for `world` in-process ranks to
 * out128 (host only; the group is freed when its last handle is destroyed).  QSIM_EINVAL
 * unless world is 1, 2, 4 or 8. */
int qsim_loopback_id(int world, void *out128);

/* Which global-qubit swap path the handle runs (collective choice, identical on every rank):
 *   QSIM_SWAP_NONE            world == 1;
 *   QSIM_SWAP_FUSED_SPLIT     the passes of a layer store the swapped amplitudes straight into
 *                             the peers' second buffers (split over the layer's passes);
 *   QSIM_SWAP_FUSED           the same, all moved by the boundary pass;
 *   QSIM_SWAP_LOWBIT          fused, low-bit swap schedule (QSIM_LOWSWAP=1, G = 2);
 *   QSIM_SWAP_COLLECTIVE      out of place through the transport's grouped send/recv;
 *   QSIM_SWAP_INPLACE_STAGED  in place through a bounded staging ring (no second buffer;
 *                             QSIM_FUSED_SWAP=0);
 *   QSIM_SWAP_FUSED_INPLACE   no second buffer (the n = 36 shape): the passes of a layer store the
 *                             swapped amplitudes into the peers' current buffers, each tile after
 *                             its partner tile on the peer has been loaded (per-tile handshake
 *                             flags over NVLink).
 * The default is the fused split swap when a second shard buffer fits on every rank with 8 GiB to
 * spare, else the fused in-place swap; QSIM_SWAP_INPLACE=1 forces the no-second-buffer paths. */
enum { QSIM_SWAP_NONE = 0, QSIM_SWAP_FUSED_SPLIT = 1, QSIM_SWAP_FUSED = 2, QSIM_SWAP_LOWBIT = 3,
       QSIM_SWAP_COLLECTIVE = 4, QSIM_SWAP_INPLACE_STAGED = 5, QSIM_SWAP_FUSED_INPLACE = 6 };
int qsim_swap_path(const qsim_t *q);

/* Number of qubits of the handle (QSIM_EINVAL for NULL). */
int qsim_num_qubits(const qsim_t *q);

/* Diagnostics for benchmarking: when enabled, every tile-pass kernel launch is bracketed
 * by CUDA events on the handle's stream.  qsim_profile_read synchronises and returns the
 * summed pass-kernel time (ms), the number of pass launches and their summed algorithmic
 * HBM bytes (32 B per amplitude read+written, 16 B for the write-only init pass) since the
 * last enable/read, then resets the counters. */
int qsim_profile_enable(qsim_t *q, int on);
int qsim_profile_read(qsim_t *q, double *ms_sum, uint64_t *count, double *bytes_sum);
/* Per-pass variant: writes the duration (ms) of each recorded pass, in launch order, into
 * ms_out[0 .. min(count, cap)) and (if kind_out is not NULL) its pass program into kind_out:
 * bits 0-1 = QSIM_PASS_PLAIN12 / _PLAIN_RUN / _TURN12 / _TURN_RUN (12-bit set or run set, without
 * or with the cost phase = a "turning" pass), plus the flags QSIM_PASS_MOVING (carries part of a
 * global-qubit swap), QSIM_PASS_INIT (writes |+> instead of reading), QSIM_PASS_REDUCE (fused
 * <H_C> / norm).  Returns the number of recorded passes (>= 0) or a negative error code; clears
 * the record like qsim_profile_read.  Synchronises. */
enum { QSIM_PASS_PLAIN12 = 0, QSIM_PASS_PLAIN_RUN = 1, QSIM_PASS_TURN12 = 2, QSIM_PASS_TURN_RUN = 3,
       QSIM_PASS_MOVING = 4, QSIM_PASS_INIT = 8, QSIM_PASS_REDUCE = 16 };
int qsim_profile_passes(qsim_t *q, double *ms_out, int *kind_out, int cap);

/* Diagnostic micro-benchmark (modifies the state): time `reps` back-to-back launches of the tile
 * pass over tile set `set` (0 = bits 0..11, 1.. = the run sets in ascending bit order) with phase
 * on (1) / off (0), or, for phase < 0, a memory-pattern probe without butterflies (-1 copy, -2 read
 * only, -3 write only), on the handle's stream; *ms_out = mean ms per launch.  The pass program is
 * the one the schedules would use for that set (per-warp turning kernel where eligible). */
int qsim_bench_pass(qsim_t *q, int set, int phase, int reps, double *ms_out);

/* Number of kernels the library has launched on this handle (for bench reporting). */
uint64_t qsim_kernel_launches(const qsim_t *q);

/* Message for the last error on q (or for the last failed create when q is NULL). */
const char *qsim_last_error(const qsim_t *q);

const char *qsim_version(void);

#ifdef __cplusplus
}
#endif
#endif /* QSIM_H */
