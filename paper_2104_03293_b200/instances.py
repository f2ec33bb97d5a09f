"""Seeded synthetic input generators shared by the product harness, bench.py and the
tests.  This module holds NO arithmetic of the method (no energies, phases, mixers,
angles or reductions): it only draws problem data.  The reductions of problem data
to Ising fields (eq:HChi..eq:HCC) are written twice, independently, in
paper_2104_03293_b200/problems.py (product harness) and oracle/problems.py (oracle).

Recipes:
  * random_ising: dense Ising, h_i uniform half-integers in [-2, 2], J_ij uniform in
    {-1, -1/2, 0, 1/2, 1} (i<j) -- inside the eq:rescale bounds.
  * planted_2sat: random 2-clauses satisfied by a planted x*, added until x* is the
    unique minimiser of the violated-clause count (brute force over 2^n).
  * exact_cover: N x F boolean matrix, F = 472; 8 planted rows partition the
    F columns; the other rows are random weight-53 subsets (shaped to give r~36-37,
    cf. r = 36.75 for instance 30(0)).
  * cluster_ising / product_ising: structured instances for large-n pins (P8, P9).
  * dw_like_schedule: synthetic piecewise-linear A(s), B(s) in GHz shaped like the
    DW_2000Q_6 schedule of Fig. 1 (values not printed in the paper; reading R10).
"""
from __future__ import annotations

import numpy as np


def random_ising(n: int, seed: int = 1):
    rng = np.random.default_rng(seed)
    h = rng.integers(-4, 5, size=n).astype(np.float64) / 2.0
    J = np.zeros((n, n))
    iu = np.triu_indices(n, 1)
    J[iu] = rng.integers(-2, 3, size=iu[0].shape[0]).astype(np.float64) / 2.0
    return h, J


def planted_2sat(n: int, seed: int = 0, max_clauses: int = 100000):
    """Return (clauses, x_star).  clause = (i, a, j, b) with a, b in {+1, -1}:
    literal i is x_i if a = +1 else (not x_i)."""
    rng = np.random.default_rng(seed)
    x_star = rng.integers(0, 2, size=n)
    dim = 1 << n
    zs = np.arange(dim, dtype=np.int64)
    bits = ((zs[:, None] >> np.arange(n)[None, :]) & 1).astype(np.int8)
    viol = np.zeros(dim, dtype=np.int64)
    z_star = int(sum(int(x_star[i]) << i for i in range(n)))
    clauses = []
    while len(clauses) < max_clauses:
        i, j = rng.choice(n, size=2, replace=False)
        a = int(rng.choice([-1, 1]))
        b = int(rng.choice([-1, 1]))
        li = x_star[i] if a > 0 else 1 - x_star[i]
        lj = x_star[j] if b > 0 else 1 - x_star[j]
        if li == 0 and lj == 0:
            continue  # x* must satisfy every clause
        clauses.append((int(i), a, int(j), b))
        vi = bits[:, i] if a > 0 else 1 - bits[:, i]
        vj = bits[:, j] if b > 0 else 1 - bits[:, j]
        viol += ((vi == 0) & (vj == 0)).astype(np.int64)
        if viol[z_star] == 0 and np.count_nonzero(viol == 0) == 1:
            break
    return clauses, x_star


def exact_cover(N: int, F: int = 472, seed: int = 0, planted_rows: int = 8, weight: int = 53):
    """Return (a, x_star): a in {0,1}^{N x F}; x_star selects the planted rows."""
    rng = np.random.default_rng(seed)
    k = min(planted_rows, N)
    rows = rng.permutation(N)[:k]
    a = np.zeros((N, F), dtype=np.uint8)
    cols = rng.permutation(F)
    for r, chunk in zip(rows, np.array_split(cols, k)):
        a[r, chunk] = 1
    for r in range(N):
        if r in rows:
            continue
        a[r, rng.choice(F, size=min(weight, F), replace=False)] = 1
    x_star = np.zeros(N, dtype=np.int64)
    x_star[rows] = 1
    return a, x_star


def product_ising(n: int, seed: int = 0):
    """J = 0 instance (pin P8)."""
    rng = np.random.default_rng(seed)
    h = rng.integers(-4, 5, size=n).astype(np.float64) / 2.0
    return h, np.zeros((n, n))


def cluster_ising(n: int, clusters, seed: int = 0):
    """Block-diagonal J over the given disjoint qubit clusters (pin P9)."""
    rng = np.random.default_rng(seed)
    h = rng.integers(-4, 5, size=n).astype(np.float64) / 2.0
    J = np.zeros((n, n))
    for c in clusters:
        c = sorted(c)
        for x in range(len(c)):
            for y in range(x + 1, len(c)):
                J[c[x], c[y]] = rng.integers(-2, 3) / 2.0
    return h, J


def spread_clusters(n: int, size: int, seed: int = 0):
    """Partition range(n) into clusters of `size` qubits whose members are spread over
    low, middle and high bit positions (so that tile, passenger and global bits mix)."""
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n)
    return [sorted(int(q) for q in perm[i:i + size]) for i in range(0, n, size)]


def dw_like_schedule():
    """(s, A, B) knots in GHz; A(0)~5.6, A(1)~0, B(0)~0.1, B(1)~12 (reading R10)."""
    s = np.linspace(0.0, 1.0, 11)
    A = np.array([5.6, 3.9, 2.6, 1.6, 0.95, 0.5, 0.25, 0.1, 0.04, 0.01, 0.0])
    B = np.array([0.1, 0.5, 1.1, 1.9, 2.9, 4.0, 5.3, 6.7, 8.3, 10.0, 12.0])
    return s, A, B


def toy_schedule():
    """A(s) = 1 - s, B(s) = s (dimensionless; SPEC S:341 example schedule)."""
    return np.array([0.0, 1.0]), np.array([1.0, 0.0]), np.array([0.0, 1.0])


def sample_indices(n: int, count: int, seed: int = 0):
    """Seeded sample of basis labels in [0, 2^n) (always includes 0 and 2^n - 1)."""
    rng = np.random.default_rng(seed)
    zs = rng.integers(0, 1 << n, size=count, dtype=np.uint64)
    zs[0] = 0
    zs[-1] = (1 << n) - 1
    return zs
