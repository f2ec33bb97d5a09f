"""Product-side problem preparation (host, harness): reductions of the paper's problem
classes to Ising fields and the rescale factor.  Not on the GPU hot path; written
independently of oracle/problems.py (tests compare both to brute-force objectives).
"""
from __future__ import annotations

import numpy as np


def ising_from_exact_cover(a: np.ndarray):
    """eq:HChi / eq:HCJij / eq:HCC with b = 1_F:
    h_i = sum_j (a a^T)_ij / 2 - (a b)_i, J_ij = (a a^T)_ij / 2 for i<j,
    C = F + sum_{i<j} (a a^T)_ij / 2 + sum_i ((a a^T)_ii - 2 (a b)_i) / 2.
    Returns (h, J upper-triangular n x n, C); all values are half-integers."""
    A = np.asarray(a, dtype=np.int64)
    N, F = A.shape
    G = A @ A.T                      # (a a^T), integer
    rowsum = A.sum(axis=1)           # (a b)_i
    h = G.sum(axis=1) / 2.0 - rowsum
    J = np.triu(G, 1) / 2.0
    C = F + np.triu(G, 1).sum() / 2.0 + (np.diag(G) - 2 * rowsum).sum() / 2.0
    return h.astype(np.float64), J.astype(np.float64), float(C)


def ising_from_2sat(n: int, clauses):
    """Clause (i, a, j, b) is violated iff a s_i = -1 and b s_j = -1 (s = 2x - 1,
    eq:xtosigma); its indicator (1 - a s_i)(1 - b s_j)/4 gives h, J, C."""
    h = np.zeros(n)
    J = np.zeros((n, n))
    C = 0.0
    for (i, a, j, b) in clauses:
        h[i] += -0.25 * a
        h[j] += -0.25 * b
        J[min(i, j), max(i, j)] += 0.25 * a * b
        C += 0.25
    return h, J, C


def rescale_r(h, J) -> float:
    """eq:rescale with h_max = -h_min = 2 and J_max = -J_min = 1.
    The library keeps (h, J) unscaled and the harness divides gamma by r instead
    (reading R6), which leaves E(z) exactly representable."""
    h = np.asarray(h, dtype=np.float64)
    n = h.shape[0]
    iu = np.triu_indices(n, 1)
    Jv = np.asarray(J, dtype=np.float64).reshape(n, n)[iu]
    cands = [h.max() / 2.0, h.min() / -2.0, 0.0]
    if Jv.size:
        cands += [Jv.max() / 1.0, Jv.min() / -1.0]
    return float(max(cands))
