"""Oracle-side problem reductions (TEST INFRASTRUCTURE ONLY, see oracle/oracle.py).

Written from the paper independently of the product harness
(paper_2104_03293_b200/problems.py); tests check both against brute-force
objectives.
"""
from __future__ import annotations

import numpy as np


def exact_cover_objective(a: np.ndarray, x: np.ndarray) -> float:
    """sum_f (sum_i a_if x_i - 1)^2  -- eq:exactcover."""
    cov = np.asarray(x, dtype=np.float64) @ np.asarray(a, dtype=np.float64)
    return float(np.sum((cov - 1.0) ** 2))


def exact_cover_to_ising(a: np.ndarray):
    """h_i = sum_j 1/2 (a a^T)_ij - (a b)_i ; J_ij = 1/2 (a a^T)_ij (i<j) ;
    C = b^T b + 1/2 sum_{i<j} (a a^T)_ij + 1/2 sum_i ((a a^T)_ii - (2 a b)_i)
    -- eq:HChi, eq:HCJij, eq:HCC, with x_i -> (1 + s_i)/2 (eq:xtosigma)."""
    a = np.asarray(a, dtype=np.float64)
    n, F = a.shape
    b = np.ones(F)
    aat = a @ a.T
    ab = a @ b
    h = 0.5 * aat.sum(axis=1) - ab
    J = np.triu(0.5 * aat, 1)
    iu = np.triu_indices(n, 1)
    C = b @ b + 0.5 * aat[iu].sum() + 0.5 * np.sum(np.diag(aat) - 2.0 * ab)
    return h, J, float(C)


def two_sat_violations(clauses, x) -> int:
    """number of violated 2-clauses; clause (i, a, j, b): literal (x_i if a=+1 else not x_i)
    OR (x_j if b=+1 else not x_j)."""
    v = 0
    for (i, a, j, b) in clauses:
        li = x[i] if a > 0 else 1 - x[i]
        lj = x[j] if b > 0 else 1 - x[j]
        v += int(li == 0 and lj == 0)
    return v


def two_sat_to_ising(n: int, clauses):
    """Penalty of clause (i,a,j,b) = (1 - a s_i)(1 - b s_j)/4 with s = 2x - 1 (eq:xtosigma):
    h_i -= a/4, h_j -= b/4, J_ij += a b/4 (i<j), C += 1/4 (quarter-integer data)."""
    h = np.zeros(n)
    J = np.zeros((n, n))
    C = 0.0
    for (i, a, j, b) in clauses:
        h[i] -= a / 4.0
        h[j] -= b / 4.0
        lo, hi = (i, j) if i < j else (j, i)
        J[lo, hi] += a * b / 4.0
        C += 0.25
    return h, J, C


def rescale_factor(h, J, hmax=2.0, jmax=1.0) -> float:
    """r of eq:rescale, h_max = -h_min = 2, J_max = -J_min = 1."""
    h = np.asarray(h, dtype=np.float64)
    n = h.shape[0]
    Ju = np.asarray(J, dtype=np.float64).reshape(n, n)[np.triu_indices(n, 1)]
    return float(max(max(h.max() / hmax, 0.0), max(h.min() / -hmax, 0.0),
                     max(Ju.max() / jmax, 0.0), max(Ju.min() / -jmax, 0.0)))
