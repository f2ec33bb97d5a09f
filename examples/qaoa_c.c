/* qaoa_c.c -- the C-ABI (include/qsim.h) used from plain C, no Python: a p-layer QAOA evaluation
 * of a small dense Ising problem on one GPU, <H_C>, the norm, one amplitude, the enumeration of the
 * ground state and its success probability, with every return code checked.
 *
 *   gcc -O2 -I include examples/qaoa_c.c -L paper_2104_03293_b200 -lqsim \
 *       -Wl,-rpath,$PWD/paper_2104_03293_b200 -o examples/qaoa_c && examples/qaoa_c 18 3
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "qsim.h"

#define CHECK(call)                                                                              \
    do {                                                                                         \
        int rc_ = (call);                                                                        \
        if (rc_ != QSIM_OK) {                                                                    \
            fprintf(stderr, "%s -> %d (%s)\n", #call, rc_, qsim_last_error(q));                   \
            return 1;                                                                            \
        }                                                                                        \
    } while (0)

int main(int argc, char **argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 18, p = argc > 2 ? atoi(argv[2]) : 3;
    qsim_t *q = NULL;
    double *h = calloc((size_t)n, sizeof(double)), *J = calloc((size_t)n * n, sizeof(double));
    double *gamma = malloc(sizeof(double) * p), *beta = malloc(sizeof(double) * p);
    uint64_t seed = 12345;
    for (int i = 0; i < n; ++i) {  /* half-integer fields and couplings (dyadic: exact energies) */
        seed = seed * 6364136223846793005ull + 1442695040888963407ull;
        h[i] = (double)((int)((seed >> 33) % 9) - 4) / 2.0;
        for (int j = i + 1; j < n; ++j) {
            seed = seed * 6364136223846793005ull + 1442695040888963407ull;
            J[(size_t)i * n + j] = (double)((int)((seed >> 33) % 5) - 2) / 2.0;
        }
    }
    for (int k = 0; k < p; ++k) {
        gamma[k] = 0.8 * (k + 1) / (p + 1);
        beta[k] = -0.6 * (1.0 - (double)(k + 1) / (p + 1));
    }
    if (qsim_create(n, QSIM_FP64, &q) != QSIM_OK) {
        fprintf(stderr, "qsim_create: %s\n", qsim_last_error(NULL));
        return 1;
    }
    CHECK(qsim_set_ising(q, h, J));
    CHECK(qsim_init_plus(q));
    CHECK(qsim_apply_qaoa(q, gamma, beta, p));
    double e = 0.0, nrm = 0.0, amp[2] = {0.0, 0.0}, emin = 0.0, ps = 0.0;
    uint64_t gs[4], cnt = 0;
    CHECK(qsim_expect_hc(q, &e));
    CHECK(qsim_norm2(q, &nrm));
    CHECK(qsim_get_amplitudes(q, 0, 1, amp));
    CHECK(qsim_ground_states(q, gs, 4, &emin, &cnt));
    CHECK(qsim_success_prob(q, gs, cnt < 4 ? (int)cnt : 4, &ps));
    printf("qaoa_c n=%d p=%d <H_C>=%.12f norm=%.15f psi_0=(%.3e,%.3e) E_min=%.1f minimisers=%llu P_gs=%.6e launches=%llu\n",
           n, p, e, nrm, amp[0], amp[1], emin, (unsigned long long)cnt, ps,
           (unsigned long long)qsim_kernel_launches(q));
    CHECK(qsim_destroy(q));
    free(h);
    free(J);
    free(gamma);
    free(beta);
    return (nrm > 1.0 - 1e-12 && nrm < 1.0 + 1e-12) ? 0 : 2;
}
