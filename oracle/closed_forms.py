"""Closed forms and structured compositions used to pin the oracle and to check the
CUDA path at sizes where a flat 2^n oracle state does not fit (SURVEY §8c pins P2,
P3, P4, P8, P9).

TEST INFRASTRUCTURE ONLY (see oracle/oracle.py).  Plain numpy; every function
cites the passage it follows and is pinned in tests/test_oracle_pins.py against
the full-state oracle and/or a dense matrix exponential.

Spin convention: s = 2 z - 1, |0> <-> -1, |1> <-> +1.
"""
from __future__ import annotations

import itertools

import numpy as np

from . import oracle as _o


def _energy_np(h: np.ndarray, J: np.ndarray, z: int) -> float:
    """E(z) of eq:HC written out again in numpy (independent of oracle.c)."""
    n = h.shape[0]
    s = np.array([1.0 if (z >> i) & 1 else -1.0 for i in range(n)])
    iu = np.triu_indices(n, 1)
    return float(h @ s + np.sum(J[iu] * s[iu[0]] * s[iu[1]]))


# ---------------------------------------------------------------------------------
# P2: n = 1 closed form.  psi_0 = (c e^{i g h} - i s e^{-i g h})/sqrt2,
#                         psi_1 = (-i s e^{i g h} + c e^{-i g h})/sqrt2   (p = 1)
# derived from eq:QAOA_state with E(0) = -h, E(1) = +h.
# ---------------------------------------------------------------------------------
def n1_state(h: float, gamma: float, beta: float) -> np.ndarray:
    c, s = np.cos(beta), np.sin(beta)
    e0 = np.exp(1j * gamma * h)  # e^{-i gamma E(0)}, E(0) = -h
    e1 = np.exp(-1j * gamma * h)  # e^{-i gamma E(1)}, E(1) = +h
    return np.array([c * e0 - 1j * s * e1, -1j * s * e0 + c * e1]) / np.sqrt(2.0)


def n1_spin(h: float, gamma: float, beta: float) -> float:
    """<sigma^z> = P(1) - P(0) = sin 2beta sin 2 gamma h (p = 1, n = 1)."""
    return float(np.sin(2 * beta) * np.sin(2 * gamma * h))


# ---------------------------------------------------------------------------------
# P3: p = 1 path sum, any single amplitude:
#   psi'_z = 2^{-n/2} sum_y cos^{n-|y|}(beta) (-i sin beta)^{|y|} e^{-i gamma E(z xor y)}
# (tensor product of the 2x2 Rx matrices of P:349 applied to the phased |+>^n).
# ---------------------------------------------------------------------------------
def p1_path_amplitude(h, J, gamma: float, beta: float, z: int) -> complex:
    h = np.asarray(h, dtype=np.float64)
    n = h.shape[0]
    J = np.asarray(J, dtype=np.float64).reshape(n, n)
    c, s = np.cos(beta), np.sin(beta)
    acc = 0.0 + 0.0j
    for y in range(1 << n):
        w = bin(y).count("1")
        acc += c ** (n - w) * (-1j * s) ** w * np.exp(-1j * gamma * _energy_np(h, J, z ^ y))
    return complex(acc * 2.0 ** (-n / 2))


# ---------------------------------------------------------------------------------
# P4: p = 1 <H_C> closed form, any n (O(n^3)).  Derived in these conventions
# (same structure as the standard light-cone result for p = 1 QAOA):
#   <s_u> = sin2b sin(2g h_u) prod_{w != u} cos(2g J_uw)
#   <s_u s_v> = 1/2 sin4b sin(2g J_uv) [cos(2g h_u) prod_{w!=u,v} cos(2g J_uw)
#                                     + cos(2g h_v) prod_{w!=u,v} cos(2g J_vw)]
#             + 1/2 sin^2(2b) [cos(2g(h_u-h_v)) prod_{w!=u,v} cos(2g(J_uw-J_vw))
#                              - cos(2g(h_u+h_v)) prod_{w!=u,v} cos(2g(J_uw+J_vw))]
# <H_C> = sum_u h_u <s_u> + sum_{u<v} J_uv <s_u s_v>.
# ---------------------------------------------------------------------------------
def p1_spins(h, J, gamma: float, beta: float) -> np.ndarray:
    """p = 1: <s_u> = sin 2b sin(2 g h_u) prod_{w != u} cos(2 g J_uw) for every u."""
    h = np.asarray(h, dtype=np.float64)
    n = h.shape[0]
    Js = np.triu(np.asarray(J, dtype=np.float64).reshape(n, n), 1)
    Js = Js + Js.T
    out = np.empty(n)
    for u in range(n):
        others = [w for w in range(n) if w != u]
        out[u] = np.sin(2 * beta) * np.sin(2 * gamma * h[u]) * np.prod(np.cos(2 * gamma * Js[u, others]))
    return out


def p1_expect_hc(h, J, gamma: float, beta: float) -> float:
    h = np.asarray(h, dtype=np.float64)
    n = h.shape[0]
    J = np.asarray(J, dtype=np.float64).reshape(n, n)
    Js = np.triu(J, 1)
    Js = Js + Js.T  # symmetric couplings, zero diagonal
    g2 = 2.0 * gamma
    s2b, s4b = np.sin(2 * beta), np.sin(4 * beta)
    total = 0.0
    for u in range(n):
        others = [w for w in range(n) if w != u]
        zu = s2b * np.sin(g2 * h[u]) * np.prod(np.cos(g2 * Js[u, others]))
        total += h[u] * zu
    for u in range(n):
        for v in range(u + 1, n):
            if Js[u, v] == 0.0:
                continue
            ws = [w for w in range(n) if w != u and w != v]
            cu = np.prod(np.cos(g2 * Js[u, ws]))
            cv = np.prod(np.cos(g2 * Js[v, ws]))
            term1 = 0.5 * s4b * np.sin(g2 * Js[u, v]) * (np.cos(g2 * h[u]) * cu + np.cos(g2 * h[v]) * cv)
            cm = np.prod(np.cos(g2 * (Js[u, ws] - Js[v, ws])))
            cp = np.prod(np.cos(g2 * (Js[u, ws] + Js[v, ws])))
            term2 = 0.5 * s2b ** 2 * (np.cos(g2 * (h[u] - h[v])) * cm - np.cos(g2 * (h[u] + h[v])) * cp)
            total += Js[u, v] * (term1 + term2)
    return float(total)


# ---------------------------------------------------------------------------------
# P8: product state (J = 0).  Each qubit evolves independently with field h_q:
# per layer diag(e^{+i g h}, e^{-i g h}) (E = -h, +h for bits 0, 1) then Rx(2 beta).
# psi_z = prod_q phi_q[z_q].
# ---------------------------------------------------------------------------------
def single_qubit_evolution(hq: float, gammas, betas) -> np.ndarray:
    phi = np.array([1.0, 1.0], dtype=np.complex128) / np.sqrt(2.0)
    for g, b in zip(gammas, betas):
        phi = phi * np.array([np.exp(1j * g * hq), np.exp(-1j * g * hq)])
        c, s = np.cos(b), np.sin(b)
        phi = np.array([c * phi[0] - 1j * s * phi[1], -1j * s * phi[0] + c * phi[1]])
    return phi


def product_amplitudes(h, gammas, betas, zs) -> np.ndarray:
    h = np.asarray(h, dtype=np.float64)
    phis = [single_qubit_evolution(float(hq), gammas, betas) for hq in h]
    out = np.empty(len(zs), dtype=np.complex128)
    for k, z in enumerate(zs):
        a = 1.0 + 0.0j
        for q, phi in enumerate(phis):
            a *= phi[(int(z) >> q) & 1]
        out[k] = a
    return out


# ---------------------------------------------------------------------------------
# P9: cluster instances.  If J is block-diagonal over disjoint qubit clusters, H_C is
# a sum of commuting cluster terms and H_D factorises, so the QAOA state is the
# tensor product of the cluster states (each computed by the full-state oracle on
# its own |c| qubits); <H_C> is the sum of cluster expectations.
# ---------------------------------------------------------------------------------
class ClusterComposition:
    def __init__(self, h, J, clusters, gammas, betas):
        h = np.asarray(h, dtype=np.float64)
        n = h.shape[0]
        J = np.asarray(J, dtype=np.float64).reshape(n, n)
        seen = sorted(itertools.chain.from_iterable(clusters))
        assert seen == list(range(n)), "clusters must partition the qubits"
        Ju = np.triu(J, 1)
        for a in range(len(clusters)):
            for b in range(len(clusters)):
                if a != b:
                    assert not np.any(Ju[np.ix_(clusters[a], clusters[b])]), "J not block-diagonal"
        self.clusters = [list(c) for c in clusters]
        self.states = []
        self.expect = 0.0
        for c in self.clusters:
            hc = h[c]
            Jc = Ju[np.ix_(c, c)]
            psi = _o.qaoa_state(hc, Jc, gammas, betas)
            self.states.append(psi)
            self.expect += _o.expect_hc(hc, Jc, psi)

    def amplitude(self, z: int) -> complex:
        a = 1.0 + 0.0j
        for c, psi in zip(self.clusters, self.states):
            zc = 0
            for k, q in enumerate(c):
                zc |= ((int(z) >> q) & 1) << k
            a *= psi[zc]
        return complex(a)

    def amplitudes(self, zs) -> np.ndarray:
        return np.array([self.amplitude(int(z)) for z in zs], dtype=np.complex128)
