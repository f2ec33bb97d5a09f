/*
 * oracle.c -- plain, slow, obviously-correct CPU state-vector simulator for the
 * QAOA / AQA hot path of arXiv:2104.03293 (JUQCS-G paper).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  The product path
 * (paper_2104_03293_b200/) never imports, links or executes anything here, and
 * this file shares no code, header, table or constant with the CUDA path.
 *
 * Citations: "P:<line>" = /root/reference/PAPER.md line (LaTeX source), labels
 * as in the paper (eq:HC, eq:QAOA_state, eq:beta_k, ...).
 *
 * Conventions (readings R1, R2, R4, R5):
 *   - basis label z, qubit j <-> bit j of z (little-endian), "psi_{q_{N-1}...q_0}".
 *   - spin s_j(z) = 2*bit_j(z) - 1 : |0> is the -1 eigenstate, |1> the +1
 *     eigenstate of sigma^z (eq:xtosigma context).
 *   - E(z) = sum_i h_i s_i + sum_{i<j} J_ij s_i s_j (eq:HC); the
 *     additive constant C is not part of H_C (global phase).
 *   - J is an n*n row-major array; only entries with i<j are read.
 *   - state psi: interleaved complex128, psi[2z] = Re, psi[2z+1] = Im.
 *
 * Compile: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC
 * (no fused multiply-add contraction, glibc sin/cos).
 *
 * Every function has a pin in tests/test_oracle_pins.py (none is "parity unpinned").
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* spin value of qubit i in basis state z: P:303 ("-1 (+1) eigenstate ... |0> (|1>)") */
static double spin(uint64_t z, int i) { return ((z >> i) & 1ull) ? 1.0 : -1.0; }

/* E(z) = sum_i h_i s_i + sum_{i<j} J_ij s_i s_j  -- eq:HC.
 * Canonical order: fields i ascending, then couplings (i,j) row-major, i<j. */
double oracle_energy(int n, const double *h, const double *J, uint64_t z) {
    double e = 0.0;
    for (int i = 0; i < n; ++i) e += h[i] * spin(z, i);
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j) e += J[(size_t)i * n + j] * spin(z, i) * spin(z, j);
    return e;
}

/* E(z) for z = first .. first+count-1 */
void oracle_energies(int n, const double *h, const double *J, uint64_t first, uint64_t count,
                     double *out) {
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < (int64_t)count; ++k) out[k] = oracle_energy(n, h, J, first + (uint64_t)k);
}

/* |+>^{otimes n}: psi_z = 2^{-n/2} for all z  (eq:HI ground state) */
void oracle_init_plus(int n, double *psi) {
    uint64_t dim = 1ull << n;
    /* exact power of two when n is even; correctly rounded libm pow otherwise */
    double a = pow(2.0, -0.5 * n);
#pragma omp parallel for schedule(static)
    for (int64_t z = 0; z < (int64_t)dim; ++z) { psi[2 * z] = a; psi[2 * z + 1] = 0.0; }
}

/* e^{-i gamma H_C}: psi_z <- (cos(gamma E(z)) - i sin(gamma E(z))) psi_z
 * (eq:QAOA_state; H_C diagonal in the computational basis).
 * If `etab` is non-NULL it holds E(z) for all z (computed by oracle_energies). */
void oracle_apply_phase(int n, const double *h, const double *J, const double *etab, double gamma,
                        double *psi) {
    uint64_t dim = 1ull << n;
#pragma omp parallel for schedule(static)
    for (int64_t z = 0; z < (int64_t)dim; ++z) {
        double e = etab ? etab[z] : oracle_energy(n, h, J, (uint64_t)z);
        double th = gamma * e;
        double c = cos(th), s = sin(th);
        double re = psi[2 * z], im = psi[2 * z + 1];
        /* (c - i s)(re + i im) = (c re + s im) + i (c im - s re) */
        psi[2 * z] = c * re + s * im;
        psi[2 * z + 1] = c * im - s * re;
    }
}

/* single-qubit 2-component update on qubit q (eq:twocomponentupdates)
 * with the Rx matrix e^{-i beta sigma^x} = [[c, -i s], [-i s, c]], c = cos beta, s = sin beta. */
void oracle_apply_rx(int n, int q, double beta, double *psi) {
    uint64_t dim = 1ull << n, bit = 1ull << q;
    double c = cos(beta), s = sin(beta);
#pragma omp parallel for schedule(static)
    for (int64_t z = 0; z < (int64_t)dim; ++z) {
        if ((uint64_t)z & bit) continue;
        uint64_t z1 = (uint64_t)z | bit;
        double ar = psi[2 * z], ai = psi[2 * z + 1];
        double br = psi[2 * z1], bi = psi[2 * z1 + 1];
        /* a' = c a - i s b ; b' = -i s a + c b ; (-i s)(x + i y) = s y - i s x */
        psi[2 * z] = c * ar + s * bi;
        psi[2 * z + 1] = c * ai - s * br;
        psi[2 * z1] = s * ai + c * br;
        psi[2 * z1 + 1] = -s * ar + c * bi;
    }
}

/* e^{-i beta H_D}, H_D = sum_i sigma^x_i = prod_i e^{-i beta sigma^x_i}
 * ("rotations around the x axis with angle 2 beta_k"; H_D P:272-274) */
void oracle_apply_mixer(int n, double beta, double *psi) {
    for (int q = 0; q < n; ++q) oracle_apply_rx(n, q, beta, psi);
}

/* |beta,gamma> = prod_{k=1}^p e^{-i beta_k H_D} e^{-i gamma_k H_C} |+>^n
 * (eq:QAOA_state P:265-268; explicit order from Appendix A: layer 1 first,
 * phase before mixer).  psi must hold 2*2^n doubles; it is (re)initialised. */
void oracle_apply_qaoa(int n, const double *h, const double *J, const double *gamma,
                       const double *beta, int p, double *psi) {
    uint64_t dim = 1ull << n;
    double *etab = (double *)malloc(sizeof(double) * dim);
    if (etab) oracle_energies(n, h, J, 0, dim, etab);
    oracle_init_plus(n, psi);
    for (int k = 0; k < p; ++k) {
        oracle_apply_phase(n, h, J, etab, gamma[k], psi);
        oracle_apply_mixer(n, beta[k], psi);
    }
    free(etab);
}

/* same as oracle_apply_qaoa but continuing from the given psi (no init) */
void oracle_apply_layers(int n, const double *h, const double *J, const double *gamma,
                         const double *beta, int p, double *psi) {
    for (int k = 0; k < p; ++k) {
        oracle_apply_phase(n, h, J, NULL, gamma[k], psi);
        oracle_apply_mixer(n, beta[k], psi);
    }
}

/* piecewise-linear schedule value at s (knots s_0=0 < ... < s_{m-1}=1); the
 * schedule data of Fig. 1 (DW_2000Q_6) is not printed in the paper (reading R10). */
static double pwl(const double *ks, const double *kv, int m, double s) {
    if (s <= ks[0]) return kv[0];
    for (int j = 0; j + 1 < m; ++j)
        if (s <= ks[j + 1]) return kv[j] + (kv[j + 1] - kv[j]) * (s - ks[j]) / (ks[j + 1] - ks[j]);
    return kv[m - 1];
}

/* AQA / QAOA-initialisation angles, eq:beta_k / eq:gamma_k:
 *   beta_k  = -tau (A(s_{k+1}) + A(s_k)) / 2,  k = 1..p-1
 *   beta_p  = -tau A(s_p) / 2
 *   gamma_k =  tau B(s_k)
 * with s_k = (k-1)/(p-1), identical to the AQA convention s_k = k/n,
 * k = 0..n, n = p-1.  tau = T/p so that t_anneal = (n+1) tau = T
 * (reading R9).  Returns 0, or -1 if p < 2 or the knots are invalid. */
int oracle_aqa_angles(double T, int p, const double *ks, const double *A, const double *B, int m,
                      double *gamma, double *beta) {
    if (p < 2 || m < 2) return -1;
    double tau = T / p;
    for (int k = 1; k <= p; ++k) {
        double sk = (double)(k - 1) / (double)(p - 1);
        gamma[k - 1] = tau * pwl(ks, B, m, sk);
        if (k < p) {
            double sk1 = (double)k / (double)(p - 1);
            beta[k - 1] = -tau * (pwl(ks, A, m, sk1) + pwl(ks, A, m, sk)) / 2.0;
        } else {
            beta[k - 1] = -tau * pwl(ks, A, m, sk) / 2.0;
        }
    }
    return 0;
}

/* QSDS "combined" second-order step, eq. AQA4, applied for l = 0..nsteps:
 *   exp[i tau/2 sum_i (ht^x sigma^x_i + ht^z_i sigma^z_i)] exp[i tau sum_{i<j} Jt_ij s_i s_j]
 *   exp[i tau/2 sum_i (...)]  with ht^x = A(s_l), ht^z_i = -B(s_l) h_i, Jt_ij = -B(s_l) J_ij
 * (AQA0-AQA3), s_l = l tau / t_anneal, t_anneal = (nsteps+1) tau.
 * Each single-spin exponential exactly: exp[i(a X + b Z)] = cos w I + i sin w / w (a X + b Z),
 * w = sqrt(a^2 + b^2); sigma^z = diag(-1, +1) on (|0>, |1>).  psi is updated in place
 * (the caller supplies |+>^n for Psi(0)). */
static void qsds_half(int n, const double *h, double a_coef, double b_scale, double *psi) {
    uint64_t dim = 1ull << n;
    for (int q = 0; q < n; ++q) {
        double a = a_coef, b = b_scale * h[q];
        double w = sqrt(a * a + b * b);
        double c = cos(w), sw = (w > 0.0) ? sin(w) / w : 1.0;
        /* U = [[c - i sw b, i sw a], [i sw a, c + i sw b]] on (|0>, |1>) */
        double u00r = c, u00i = -sw * b, u01r = 0.0, u01i = sw * a;
        double u11r = c, u11i = sw * b;
        uint64_t bit = 1ull << q;
#pragma omp parallel for schedule(static)
        for (int64_t z = 0; z < (int64_t)dim; ++z) {
            if ((uint64_t)z & bit) continue;
            uint64_t z1 = (uint64_t)z | bit;
            double ar = psi[2 * z], ai = psi[2 * z + 1], br = psi[2 * z1], bi = psi[2 * z1 + 1];
            psi[2 * z] = u00r * ar - u00i * ai + u01r * br - u01i * bi;
            psi[2 * z + 1] = u00r * ai + u00i * ar + u01r * bi + u01i * br;
            psi[2 * z1] = u01r * ar - u01i * ai + u11r * br - u11i * bi;
            psi[2 * z1 + 1] = u01r * ai + u01i * ar + u11r * bi + u11i * br;
        }
    }
}

void oracle_apply_qsds(int n, const double *h, const double *J, double tau, int nsteps, const double *ks,
                       const double *A, const double *B, int m, double *psi) {
    uint64_t dim = 1ull << n;
    double *zeros = (double *)calloc((size_t)n, sizeof(double));
    for (int l = 0; l <= nsteps; ++l) {
        double sl = (double)l / (double)(nsteps + 1);
        double Al = pwl(ks, A, m, sl), Bl = pwl(ks, B, m, sl);
        qsds_half(n, h, 0.5 * tau * Al, -0.5 * tau * Bl, psi);
        /* exp[i tau sum Jt s s] = exp[-i tau B E_J(z)], E_J = sum_{i<j} J_ij s_i s_j */
#pragma omp parallel for schedule(static)
        for (int64_t z = 0; z < (int64_t)dim; ++z) {
            double e = oracle_energy(n, zeros, J, (uint64_t)z);
            double th = tau * Bl * e, c = cos(th), s = sin(th);
            double re = psi[2 * z], im = psi[2 * z + 1];
            psi[2 * z] = c * re + s * im;
            psi[2 * z + 1] = c * im - s * re;
        }
        qsds_half(n, h, 0.5 * tau * Al, -0.5 * tau * Bl, psi);
    }
    free(zeros);
}

/* <H_C> = sum_z |psi_z|^2 E(z)  (E_p(beta,gamma)), constant C excluded (R4).
 * Also returns sum_z |psi_z|^2 |E(z)| in *abs_out (tolerance scale, reading R12). */
double oracle_expect_hc(int n, const double *h, const double *J, const double *psi,
                        double *abs_out) {
    uint64_t dim = 1ull << n;
    double acc = 0.0, acc_abs = 0.0;
#pragma omp parallel for schedule(static) reduction(+ : acc, acc_abs)
    for (int64_t z = 0; z < (int64_t)dim; ++z) {
        double pz = psi[2 * z] * psi[2 * z] + psi[2 * z + 1] * psi[2 * z + 1];
        double e = oracle_energy(n, h, J, (uint64_t)z);
        acc += pz * e;
        acc_abs += pz * fabs(e);
    }
    if (abs_out) *abs_out = acc_abs;
    return acc;
}

/* ||psi||^2 = sum_z |psi_z|^2  (normalisation) */
double oracle_norm2(int n, const double *psi) {
    uint64_t dim = 1ull << n;
    double acc = 0.0;
#pragma omp parallel for schedule(static) reduction(+ : acc)
    for (int64_t z = 0; z < (int64_t)dim; ++z)
        acc += psi[2 * z] * psi[2 * z] + psi[2 * z + 1] * psi[2 * z + 1];
    return acc;
}

/* spin expectations <sigma^z_i> = sum_z |psi_z|^2 s_i(z) for i = 0..n-1
 * ("spin expectation values during the time evolution"; Fig. 5) */
void oracle_spin_expectations(int n, const double *psi, double *out) {
    uint64_t dim = 1ull << n;
    for (int i = 0; i < n; ++i) {
        double acc = 0.0;
#pragma omp parallel for schedule(static) reduction(+ : acc)
        for (int64_t z = 0; z < (int64_t)dim; ++z)
            acc += (psi[2 * z] * psi[2 * z] + psi[2 * z + 1] * psi[2 * z + 1]) * spin((uint64_t)z, i);
        out[i] = acc;
    }
}

/* success probability: sum over the listed ground states of |psi_z|^2 */
double oracle_success_prob(int n, const double *psi, const uint64_t *gs, int count) {
    (void)n;
    double acc = 0.0;
    for (int k = 0; k < count; ++k) {
        uint64_t z = gs[k];
        acc += psi[2 * z] * psi[2 * z] + psi[2 * z + 1] * psi[2 * z + 1];
    }
    return acc;
}

/* brute-force ground states: enumerate all 2^n energies (cf. "full enumeration",
 * P:535).  Writes up to max_out minimisers in ascending z into out, the minimum
 * energy into *emin, and returns the total number of minimisers. */
int oracle_ground_states(int n, const double *h, const double *J, uint64_t *out, int max_out,
                         double *emin) {
    uint64_t dim = 1ull << n;
    double best = INFINITY;
    for (uint64_t z = 0; z < dim; ++z) {
        double e = oracle_energy(n, h, J, z);
        if (e < best) best = e;
    }
    int cnt = 0;
    for (uint64_t z = 0; z < dim; ++z) {
        if (oracle_energy(n, h, J, z) == best) {
            if (cnt < max_out) out[cnt] = z;
            ++cnt;
        }
    }
    *emin = best;
    return cnt;
}

/* number of OpenMP threads the oracle runs with (for the cpu_baseline "cores" key) */
#ifdef _OPENMP
#include <omp.h>
int oracle_num_threads(void) { return omp_get_max_threads(); }
#else
int oracle_num_threads(void) { return 1; }
#endif
