"""Pins of the CPU oracle against things other than itself:
dense matrix exponentials (scipy), closed forms, brute force, symmetries, and the
worked values in tests/golden/ (each with its PAPER.md citation).

CPU only; no GPU.  A plausible mistake anywhere in oracle.c (dropped term, wrong
sign, wrong bit/index, transposed operand, wrong layer order) fails at least one.
"""
import json
import os

import numpy as np
import pytest
import scipy.linalg as sla
from scipy.integrate import solve_ivp

from oracle import closed_forms as cf
from oracle import oracle as o
from oracle import problems as op
from paper_2104_03293_b200 import instances as inst


# ----------------------------------------------------------------------------- dense helpers
def dense_energies(h, J):
    """E(z) for all z, straight from eq:HC with numpy broadcasting (no loops shared with oracle.c)."""
    n = len(h)
    z = np.arange(1 << n)
    S = np.where(((z[:, None] >> np.arange(n)[None, :]) & 1) == 1, 1.0, -1.0)
    Ju = np.triu(np.asarray(J, dtype=float), 1)
    return S @ np.asarray(h, dtype=float) + np.einsum("zi,ij,zj->z", S, Ju, S)


def dense_HD(n):
    """H_D = sum_i sigma^x_i as a dense 2^n x 2^n matrix (qubit i <-> bit i)."""
    X = np.array([[0.0, 1.0], [1.0, 0.0]])
    I2 = np.eye(2)
    H = np.zeros((1 << n, 1 << n))
    for i in range(n):
        op_ = np.array([[1.0]])
        for q in reversed(range(n)):  # kron ordering: leftmost factor = highest qubit
            op_ = np.kron(op_, X if q == i else I2)
        H += op_
    return H


def dense_qaoa(h, J, gammas, betas):
    n = len(h)
    E = dense_energies(h, J)
    HD = dense_HD(n)
    psi = np.full(1 << n, 2.0 ** (-n / 2), dtype=complex)
    for g, b in zip(gammas, betas):
        psi = np.exp(-1j * g * E) * psi
        psi = sla.expm(-1j * b * HD) @ psi
    return psi


def rand_angles(p, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(-2.0, 2.0, p), rng.uniform(-np.pi, np.pi, p)


# ----------------------------------------------------------------------------- E(z)
def test_energy_matches_independent_numpy_and_is_exact():
    for n, seed in [(1, 0), (5, 1), (9, 2), (12, 3)]:
        h, J = inst.random_ising(n, seed)
        e_or = o.energies(h, J)
        e_np = dense_energies(h, J)
        assert np.array_equal(e_or, e_np)  # dyadic data: exact in any order (reading R14)


def test_energy_sign_convention():
    # |0> is the -1, |1> the +1 eigenstate of sigma^z
    h = np.array([1.0, 0.0])
    J = np.zeros((2, 2))
    assert o.energy(h, J, 0) == -1.0 and o.energy(h, J, 1) == 1.0
    J[0, 1] = 1.0
    assert o.energy(np.zeros(2), J, 0b01) == -1.0 and o.energy(np.zeros(2), J, 0b11) == 1.0
    # only i<j is read
    J2 = J.copy()
    J2[1, 0] = 123.0
    assert o.energy(np.zeros(2), J2, 0b01) == -1.0


# ----------------------------------------------------------------------------- P1 dense expm
@pytest.mark.parametrize("n,p,seed", [(1, 3, 0), (2, 2, 1), (3, 4, 2), (5, 3, 3), (8, 2, 4)])
def test_P1_dense_expm(n, p, seed):
    h, J = inst.random_ising(n, seed)
    g, b = rand_angles(p, seed)
    ref = dense_qaoa(h, J, g, b)
    got = o.qaoa_state(h, J, g, b)
    assert np.max(np.abs(got - ref)) < 1e-13


@pytest.mark.parametrize("n,p,seed", [(1, 2, 20), (3, 3, 21), (6, 2, 22), (8, 3, 23)])
def test_P1_apply_layers_from_arbitrary_state(n, p, seed):
    """oracle_apply_layers (the continuation entry, which evaluates E(z) on the fly: the
    etab == NULL branch of oracle_apply_phase) from a random normalised state vs the dense
    expm product of eq:QAOA_state's factors (order of P:683)."""
    h, J = inst.random_ising(n, seed)
    g, b = rand_angles(p, seed)
    rng = np.random.default_rng(seed)
    psi0 = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    psi0 /= np.linalg.norm(psi0)
    E = dense_energies(h, J)
    HD = dense_HD(n)
    ref = psi0.copy()
    for gk, bk in zip(g, b):
        ref = sla.expm(-1j * bk * HD) @ (np.exp(-1j * gk * E) * ref)
    got = np.ascontiguousarray(psi0.copy())
    o.apply_layers(h, J, g, b, got)
    assert np.max(np.abs(got - ref)) < 1e-13


def test_P1_apply_layers_continues_qaoa_state():
    """apply_layers(qaoa_state(g[:k]), g[k:]) == qaoa_state(g) for every split k (the two
    entries reach the same |beta, gamma>), and the on-the-fly phase equals the
    table phase bit for bit (dyadic E, reading R14)."""
    n, p = 9, 5
    h, J = inst.random_ising(n, 31)
    g, b = rand_angles(p, 31)
    full = o.qaoa_state(h, J, g, b)
    for k in range(1, p):
        psi = o.qaoa_state(h, J, g[:k], b[:k])
        o.apply_layers(h, J, g[k:], b[k:], psi)
        assert np.max(np.abs(psi - full)) < 1e-14
    # phase alone: on the fly (etab NULL) vs the closed form e^{-i gamma E} psi
    psi = o.init_plus(n)
    o.apply_phase(h, J, 0.731, psi)
    ref = np.exp(-1j * 0.731 * dense_energies(h, J)) * 2.0 ** (-n / 2)
    assert np.max(np.abs(psi - ref)) < 1e-15


def test_P1_layer_order_matters():
    # a swapped order (mixer before phase) must NOT match -> the pin can see it
    h, J = inst.random_ising(4, 7)
    g, b = rand_angles(2, 7)
    n = 4
    E = dense_energies(h, J)
    HD = dense_HD(n)
    psi = np.full(1 << n, 0.25, dtype=complex)
    for gk, bk in zip(g, b):
        psi = sla.expm(-1j * bk * HD) @ psi
        psi = np.exp(-1j * gk * E) * psi
    assert np.max(np.abs(o.qaoa_state(h, J, g, b) - psi)) > 1e-3


# ----------------------------------------------------------------------------- P2 n=1
@pytest.mark.parametrize("hq,g,b", [(1.0, 0.3, 0.7), (-0.5, 1.9, -2.2), (2.0, 0.0, 1.1), (0.5, 3.0, np.pi / 2)])
def test_P2_single_qubit_closed_form(hq, g, b):
    psi = o.qaoa_state([hq], [[0.0]], [g], [b])
    assert np.max(np.abs(psi - cf.n1_state(hq, g, b))) < 1e-15
    pz = abs(psi[1]) ** 2 - abs(psi[0]) ** 2
    assert abs(pz - cf.n1_spin(hq, g, b)) < 1e-15


# ----------------------------------------------------------------------------- P3 path sum
def test_P3_p1_path_sum():
    for n, seed in [(2, 0), (2, 5), (6, 1), (9, 2)]:
        h, J = inst.random_ising(n, seed)
        g, b = 0.37 + 0.1 * seed, -1.3 + 0.2 * seed
        psi = o.qaoa_state(h, J, [g], [b])
        for z in [0, 1, (1 << n) - 1, (1 << n) // 3]:
            assert abs(psi[z] - cf.p1_path_amplitude(h, J, g, b, z)) < 1e-13


# ----------------------------------------------------------------------------- P4 p=1 <H_C>
@pytest.mark.parametrize("n,seed", [(2, 0), (3, 1), (6, 2), (10, 3), (12, 4)])
def test_P4_p1_expectation_closed_form(n, seed):
    h, J = inst.random_ising(n, seed)
    for g, b in [(0.21, 0.4), (1.7, -0.9), (0.05, 2.8)]:
        psi = o.qaoa_state(h, J, [g], [b])
        e, eabs = o.expect_hc(h, J, psi, with_abs=True)
        assert abs(e - cf.p1_expect_hc(h, J, g, b)) <= 1e-12 * max(1.0, eabs)


def test_expect_hc_matches_dense_quadratic_form():
    h, J = inst.random_ising(7, 9)
    g, b = rand_angles(3, 9)
    psi = o.qaoa_state(h, J, g, b)
    E = dense_energies(h, J)
    assert abs(o.expect_hc(h, J, psi) - np.vdot(psi, E * psi).real) < 1e-12


# ----------------------------------------------------------------------------- P5 Z2 symmetry
def test_P5_spin_flip():
    n = 9
    h, J = inst.random_ising(n, 11)
    g, b = rand_angles(4, 11)
    psi = o.qaoa_state(h, J, g, b)
    psi_f = o.qaoa_state(-h, J, g, b)
    comp = (1 << n) - 1
    idx = np.arange(1 << n) ^ comp
    assert np.array_equal(psi_f, psi[idx])
    psi0 = o.qaoa_state(np.zeros(n), J, g, b)
    assert np.array_equal(psi0, psi0[idx])


# ----------------------------------------------------------------------------- P6 beta + pi
def test_P6_beta_shift_by_pi():
    n = 7
    h, J = inst.random_ising(n, 12)
    g, b = rand_angles(3, 12)
    psi = o.qaoa_state(h, J, g, b)
    b2 = b.copy()
    b2[1] += np.pi
    psi2 = o.qaoa_state(h, J, g, b2)
    assert np.max(np.abs(psi2 - (-1) ** n * psi)) < 1e-14
    assert np.max(np.abs(np.abs(psi2) ** 2 - np.abs(psi) ** 2)) < 1e-15


# ----------------------------------------------------------------------------- P7 trivial problem
def test_P7_trivial_problem():
    n = 10
    g, b = rand_angles(5, 13)
    psi = o.qaoa_state(np.zeros(n), np.zeros((n, n)), g, b)
    ref = np.exp(-1j * n * np.sum(b)) * 2.0 ** (-n / 2)
    assert np.max(np.abs(psi - ref)) < 1e-14


# ----------------------------------------------------------------------------- P8 product state
def test_P8_product_state():
    n, p = 11, 5
    h, J = inst.product_ising(n, 3)
    g, b = rand_angles(p, 14)
    psi = o.qaoa_state(h, J, g, b)
    zs = np.arange(1 << n)
    assert np.max(np.abs(psi - cf.product_amplitudes(h, g, b, zs))) < 1e-14


# ----------------------------------------------------------------------------- P9 clusters
def test_P9_cluster_composition():
    n, p = 12, 3
    clusters = inst.spread_clusters(n, 4, seed=2)
    h, J = inst.cluster_ising(n, clusters, seed=5)
    g, b = rand_angles(p, 15)
    psi = o.qaoa_state(h, J, g, b)
    comp = cf.ClusterComposition(h, J, clusters, g, b)
    zs = np.arange(1 << n)
    assert np.max(np.abs(psi - comp.amplitudes(zs))) < 1e-14
    assert abs(o.expect_hc(h, J, psi) - comp.expect) < 1e-12


# ----------------------------------------------------------------------------- P11 brute force / reductions
def test_P11_exact_cover_reduction_and_ground_state():
    for seed in range(4):
        N, F = 10, 24
        a, x_star = inst.exact_cover(N, F=F, seed=seed, planted_rows=4, weight=5)
        h, J, C = op.exact_cover_to_ising(a)
        E = dense_energies(h, J)
        for z in range(1 << N):
            x = np.array([(z >> i) & 1 for i in range(N)])
            assert E[z] + C == op.exact_cover_objective(a, x)
        gs, emin, cnt = o.ground_states(h, J)
        z_star = int(sum(int(x_star[i]) << i for i in range(N)))
        assert z_star in gs and emin + C == 0.0


def test_P11_two_sat_reduction():
    n = 10
    clauses, x_star = inst.planted_2sat(n, seed=3)
    h, J, C = op.two_sat_to_ising(n, clauses)
    E = dense_energies(h, J)
    for z in range(1 << n):
        x = [(z >> i) & 1 for i in range(n)]
        assert E[z] + C == op.two_sat_violations(clauses, x)
    gs, emin, cnt = o.ground_states(h, J)
    assert cnt == 1 and gs[0] == int(sum(int(x_star[i]) << i for i in range(n)))


def test_golden_exact_cover_hand_case(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "exact_cover_hand.json")))
    h, J, C = op.exact_cover_to_ising(np.array(g["a"]))
    assert list(h) == g["h"] and J[0, 1] == g["J01"] and C == g["C"]
    assert op.rescale_factor(h, J) == g["r"]
    for key, val in g["objective_by_x"].items():
        assert op.exact_cover_objective(np.array(g["a"]), np.array([int(c) for c in key])) == val


# ----------------------------------------------------------------------------- P12 norm
def test_P12_norm_conservation():
    n = 14
    h, J = inst.random_ising(n, 16)
    g, b = rand_angles(10, 16)
    psi = o.qaoa_state(h, J, g, b)
    assert abs(o.norm2(psi) - 1.0) < 1e-12
    assert abs(np.sum(np.abs(psi) ** 2) - 1.0) < 1e-12


# ----------------------------------------------------------------------------- P13 Appendix A
@pytest.mark.parametrize("n,p", [(4, 3), (6, 5), (8, 2)])
def test_P13_appendix_A(n, p):
    h, J = inst.random_ising(n, 17 + p)
    s, A, B = inst.dw_like_schedule()
    A = 2 * np.pi * A
    B = 2 * np.pi * B / 8.0
    T = 0.05 * p
    psi = o.aqa_state(h, J, T, p, s, A, B)
    tau = T / p
    E = dense_energies(h, J)
    HD = dense_HD(n)
    sk = np.arange(p) / (p - 1)
    Ak = np.interp(sk, s, A)
    Bk = np.interp(sk, s, B)
    ref = np.full(1 << n, 2.0 ** (-n / 2), dtype=complex)
    for k in range(p):
        half = sla.expm(1j * tau * Ak[k] * HD / 2)
        ref = half @ (np.exp(-1j * tau * Bk[k] * E) * (half @ ref))
    ref *= np.exp(-1j * tau * Ak[0] * n / 2)
    assert np.max(np.abs(psi - ref)) < 1e-13


# ----------------------------------------------------------------------------- P14 angles
def test_P14_angle_worked_examples(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "aqa_angles_toy.json")))
    sch = g["schedule"]
    for case in g["cases"]:
        gam, bet = o.aqa_angles(case["T"], case["p"], sch["s"], sch["A"], sch["B"])
        assert list(bet) == case["beta"] and list(gam) == case["gamma"]


def test_P14_t_anneal(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "t_anneal.json")))
    # t_anneal = (n+1) tau = p tau
    assert abs((g["n_steps"] + 1) * g["tau_ns"] - g["t_anneal_ns"]) < 1e-12
    assert g["p"] == g["n_steps"] + 1


def test_aqa_angles_reject_p1():
    with pytest.raises(ValueError):
        o.aqa_angles(1.0, 1, [0.0, 1.0], [1.0, 0.0], [0.0, 1.0])


# ----------------------------------------------------------------------------- P15 AQA convergence
def test_P15_aqa_first_order_convergence():
    """AQA (paper grid s_k=(k-1)/(p-1)) converges to the continuous anneal
    H(s) = A(s)(-H_D) + B(s) H_C at FIRST order in tau = T/p (reading R9)."""
    n = 4
    h, J = inst.random_ising(n, 21)
    sA = np.array([0.0, 1.0])
    A = np.array([1.0, 0.0])
    B = np.array([0.0, 1.0])
    T = 3.0
    E = dense_energies(h, J)
    HD = dense_HD(n)

    def rhs(t, y):
        s = t / T
        H = (1 - s) * (-HD) + s * np.diag(E)
        return -1j * (H @ y)

    y0 = np.full(1 << n, 2.0 ** (-n / 2), dtype=complex)
    sol = solve_ivp(rhs, (0, T), y0, method="DOP853", rtol=1e-12, atol=1e-13)
    ref = sol.y[:, -1]
    errs = []
    for p in [16, 32, 64, 128]:
        psi = o.aqa_state(h, J, T, p, sA, A, B)
        ov = np.vdot(ref, psi)
        errs.append(np.linalg.norm(psi - ov / abs(ov) * ref))
    ratios = [errs[i] / errs[i + 1] for i in range(len(errs) - 1)]
    assert all(1.7 <= r <= 2.3 for r in ratios), ratios


# ----------------------------------------------------------------------------- P16 permutation covariance
def test_P16_qubit_permutation_covariance():
    n = 8
    h, J = inst.random_ising(n, 22)
    g, b = rand_angles(3, 22)
    perm = np.random.default_rng(22).permutation(n)
    hp = np.zeros(n)
    Jp = np.zeros((n, n))
    hp[perm] = h
    for i in range(n):
        for j in range(i + 1, n):
            a, c = sorted((perm[i], perm[j]))
            Jp[a, c] = J[i, j]
    psi = o.qaoa_state(h, J, g, b)
    psip = o.qaoa_state(hp, Jp, g, b)
    z = np.arange(1 << n)
    pz = np.zeros_like(z)
    for i in range(n):
        pz |= ((z >> i) & 1) << perm[i]
    assert np.max(np.abs(psip[pz] - psi)) < 1e-13


# ----------------------------------------------------------------------------- misc
def test_success_prob_and_init():
    n = 6
    psi = o.init_plus(n)
    assert np.all(psi == 0.125)
    assert o.success_prob(psi, [0, 5]) == 2 * 0.125 ** 2
    psi1 = o.init_plus(3)
    assert np.max(np.abs(psi1 - 2 ** -1.5)) < 1e-16


# ----------------------------------------------------------------------------- harness reductions vs oracle
def test_product_reductions_match_oracle_reductions():
    from paper_2104_03293_b200 import problems as pp
    for seed in range(3):
        a, _ = inst.exact_cover(12, F=40, seed=seed, planted_rows=4, weight=7)
        h1, J1, C1 = pp.ising_from_exact_cover(a)
        h2, J2, C2 = op.exact_cover_to_ising(a)
        assert np.array_equal(h1, h2) and np.array_equal(np.triu(J1, 1), np.triu(J2, 1)) and C1 == C2
        assert pp.rescale_r(h1, J1) == op.rescale_factor(h2, J2)
    clauses, _ = inst.planted_2sat(9, seed=4)
    h1, J1, C1 = pp.ising_from_2sat(9, clauses)
    h2, J2, C2 = op.two_sat_to_ising(9, clauses)
    assert np.array_equal(h1, h2) and np.array_equal(J1, J2) and C1 == C2


def test_exact_cover_instance_shape_matches_paper_r():
    """Generator calibration: N=30, F=472 instances give r near the paper's 36.75."""
    from paper_2104_03293_b200 import problems as pp
    rs = []
    for seed in range(4):
        a, x_star = inst.exact_cover(30, seed=seed)
        h, J, C = pp.ising_from_exact_cover(a)
        rs.append(pp.rescale_r(h, J))
        x = x_star
        assert op.exact_cover_objective(a, x) == 0.0
    assert 30.0 < np.mean(rs) < 45.0, rs


# ----------------------------------------------------------------------------- spin expectations (NEXT-2)
def test_spin_expectations_dense_and_closed_form():
    n = 8
    h, J = inst.random_ising(n, 23)
    g, b = rand_angles(3, 23)
    psi = o.qaoa_state(h, J, g, b)
    sz = o.spin_expectations(psi)
    # dense <psi| sigma^z_i |psi> with sigma^z_i = diag(s_i(z)), |1> <-> +1
    z = np.arange(1 << n)
    for i in range(n):
        si = np.where((z >> i) & 1, 1.0, -1.0)
        assert abs(sz[i] - np.vdot(psi, si * psi).real) < 1e-14
    # p = 1 closed form, and the n = 1 case of P2
    for n2, seed in [(1, 0), (5, 1), (11, 2)]:
        h2, J2 = inst.random_ising(n2, seed)
        psi1 = o.qaoa_state(h2, J2, [0.41], [-0.83])
        assert np.max(np.abs(o.spin_expectations(psi1) - cf.p1_spins(h2, J2, 0.41, -0.83))) < 1e-13
    assert abs(cf.p1_spins([0.5], [[0.0]], 0.41, -0.83)[0] - cf.n1_spin(0.5, 0.41, -0.83)) < 1e-15


# ----------------------------------------------------------------------------- QSDS combined step (NEXT-1)
def _dense_Z(n):
    z = np.arange(1 << n)
    return [np.where((z >> q) & 1, 1.0, -1.0) for q in range(n)]  # sigma^z_q = diag(s_q)


def test_qsds_matches_dense_exponentials():
    """Each factor of eq. AQA4 as a dense expm of its generator (AQA0-AQA3), n <= 5."""
    n, nsteps, tau = 5, 3, 0.37
    h, J = inst.random_ising(n, 31)
    s_, A, B = inst.dw_like_schedule()
    A, B = 0.3 * A, 0.3 * B
    HD = dense_HD(n)
    Zs = _dense_Z(n)
    EJ = dense_energies(np.zeros(n), J)
    psi = np.full(1 << n, 2.0 ** (-n / 2), dtype=complex)
    for l in range(nsteps + 1):
        sl = l / (nsteps + 1)
        Al, Bl = np.interp(sl, s_, A), np.interp(sl, s_, B)
        gen = Al * HD + np.diag(sum(-Bl * h[q] * Zs[q] for q in range(n)))  # sum_alpha ht^alpha sigma^alpha
        half = sla.expm(1j * tau / 2 * gen)
        psi = half @ (np.exp(-1j * tau * Bl * EJ) * (half @ psi))
    got = o.qsds_state(h, J, tau, nsteps, s_, A, B)
    assert np.max(np.abs(got - psi)) < 1e-13


def test_qsds_trivial_problem():
    n, nsteps, tau = 6, 4, 0.5
    s_, A, B = inst.toy_schedule()
    got = o.qsds_state(np.zeros(n), np.zeros((n, n)), tau, nsteps, s_, A, B)
    phase = sum(tau * np.interp(l / (nsteps + 1), s_, A) for l in range(nsteps + 1))
    assert np.max(np.abs(got - np.exp(1j * n * phase) * 2.0 ** (-n / 2))) < 1e-14


def test_qsds_first_order_convergence_and_forms_agree():
    """QSDS (left-endpoint s_l = l/(n+1)) converges to the TDSE of H(s) = A(s) H_I + B(s) H_C at
    first order (reading R9); the split (AQA) and combined (QSDS) forms approach each other."""
    n = 4
    h, J = inst.random_ising(n, 41)
    sA, A, B = np.array([0.0, 1.0]), np.array([1.0, 0.0]), np.array([0.0, 1.0])
    T = 3.0
    E = dense_energies(h, J)
    HD = dense_HD(n)

    def rhs(t, y):
        s = t / T
        return -1j * (((1 - s) * (-HD) + s * np.diag(E)) @ y)

    y0 = np.full(1 << n, 2.0 ** (-n / 2), dtype=complex)
    ref = solve_ivp(rhs, (0, T), y0, method="DOP853", rtol=1e-12, atol=1e-13).y[:, -1]
    errs, mutual = [], []
    for steps in [16, 32, 64, 128]:
        tau = T / steps
        psi = o.qsds_state(h, J, tau, steps - 1, sA, A, B)
        ov = np.vdot(ref, psi)
        errs.append(np.linalg.norm(psi - ov / abs(ov) * ref))
        aqa = o.aqa_state(h, J, T, steps, sA, A, B)
        ov2 = np.vdot(aqa, psi)
        mutual.append(np.linalg.norm(psi - ov2 / abs(ov2) * aqa))
    ratios = [errs[i] / errs[i + 1] for i in range(3)]
    assert all(1.7 <= r <= 2.3 for r in ratios), ratios
    assert all(mutual[i + 1] < mutual[i] for i in range(3)), mutual
