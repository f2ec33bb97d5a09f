"""GPU parity of the FP32 precision mode (QSIM_FP32) against the FP64 CPU
oracle.

The FP32 mode stores complex64 amplitudes and runs butterflies and phase products in FP32;
energies, fields and phase tables are FP64.  Every FP32 operation on the path of an amplitude
is unitary up to one rounding (relative error <= u = 2^-24 per operation, a few per butterfly
and per phase product), and unitary steps do not amplify earlier errors, so after p layers on n
qubits (n butterflies + phase + scale per layer):

    ||psi_fp32 - psi_exact||_2 <= p (2 n + 12) u          (reading R18)

which these tests enforce (max-abs is bounded by the same number); <H_C> within
2 * bound * max|E| (+ 1e-9 of the FP64 scale); norm within 2 * bound.  E(z) stays bit-exact.
"""
import numpy as np
import pytest

from oracle import closed_forms as cf
from oracle import oracle as o
from paper_2104_03293_b200 import instances as inst

pytestmark = pytest.mark.gpu

U32 = 2.0 ** -24


def bound(n, p):
    return p * (2 * n + 12) * U32


@pytest.fixture(scope="module")
def Q():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2104_03293_b200 import build

    build.build()
    from paper_2104_03293_b200 import qsim

    return qsim


def rand_angles(p, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(-2.0, 2.0, p), rng.uniform(-np.pi, np.pi, p)


def check_state(got, ref, tol):
    d = got - ref
    assert np.linalg.norm(d) <= tol, (np.linalg.norm(d), tol)
    assert np.max(np.abs(d)) <= tol


@pytest.mark.parametrize("n,p", [(6, 3), (10, 4), (13, 3), (16, 3), (20, 2), (22, 3)])
def test_fp32_qaoa_parity(Q, n, p):
    h, J = inst.random_ising(n, 300 + n)
    g, b = rand_angles(p, 310 + n)
    with Q.QSim(n, precision=Q.QSIM_FP32) as s:
        s.set_ising(h, J)
        s.init_plus()
        s.apply_qaoa(g, b)
        psi = s.amplitudes()
        e = s.expect_hc()
        nrm = s.norm2()
        en = s.energies(0, 1 << n)
    ref = o.qaoa_state(h, J, g, b)
    tol = bound(n, p)
    check_state(psi, ref, tol)
    er, sc = o.expect_hc(h, J, ref, with_abs=True)
    emax = np.max(np.abs(o.energies(h, J)))
    assert abs(e - er) <= 2 * tol * emax + 1e-9 * sc, (e, er)
    assert abs(nrm - 1.0) <= 2 * tol
    assert np.array_equal(en, o.energies(h, J))  # E(z) stays FP64 and exact


def test_fp32_continue_and_flips(Q):
    """Two apply calls (the second loads the FP32 state) with |tan beta| > 1 angles (flip mask)."""
    n = 19
    h, J = inst.random_ising(n, 77)
    g1, b1 = [0.4, -1.3], [1.3, 2.2]
    g2, b2 = [0.9], [-1.9]
    with Q.QSim(n, precision=Q.QSIM_FP32) as s:
        s.set_ising(h, J)
        s.init_plus()
        s.apply_qaoa(g1, b1)
        s.apply_qaoa(g2, b2)
        psi = s.amplitudes()
    ref = o.qaoa_state(h, J, g1 + g2, b1 + b2)
    check_state(psi, ref, bound(n, 3))


def test_fp32_aqa_exact_cover(Q):
    n, p = 18, 8
    a, x_star = inst.exact_cover(n, seed=2)
    from oracle import problems as op

    h, J, C = op.exact_cover_to_ising(a)
    r = op.rescale_factor(h, J)
    s_, A, B = inst.dw_like_schedule()
    A2, B2 = 2 * np.pi * np.asarray(A), 2 * np.pi * np.asarray(B) / r
    with Q.QSim(n, precision=Q.QSIM_FP32) as s:
        s.set_ising(h, J)
        s.init_plus()
        s.apply_aqa(0.4 * p, p, s_, A2, B2)
        psi = s.amplitudes()
        z_star = int(sum(int(x_star[i]) << i for i in range(n)))
        ps = s.success_prob([z_star])
    ref = o.aqa_state(h, J, 0.4 * p, p, s_, A2, B2)
    tol = bound(n, p)
    check_state(psi, ref, tol)
    pr = o.success_prob(ref, [z_star])
    assert abs(ps - pr) <= 2 * np.sqrt(pr) * tol + tol ** 2


def test_fp32_qsds_and_hadamard(Q):
    n = 16
    h, J = inst.random_ising(n, 5)
    s_, A, B = inst.toy_schedule()
    with Q.QSim(n, precision=Q.QSIM_FP32) as s:
        s.set_ising(h, J)
        s.init_plus()
        s.apply_qsds(0.3, 4, s_, A, B)
        psi = s.amplitudes()
        s.init_plus()
        s.apply_hadamard(11)
        psh = s.amplitudes()
    check_state(psi, o.qsds_state(h, J, 0.3, 4, s_, A, B), bound(n, 6))
    ref = np.zeros(1 << n, dtype=complex)
    ref[0] = 1.0
    check_state(psh, ref, bound(n, 11))


def test_fp32_spins(Q):
    n, p = 17, 3
    h, J = inst.random_ising(n, 9)
    g, b = rand_angles(p, 19)
    with Q.QSim(n, precision=Q.QSIM_FP32) as s:
        s.set_ising(h, J)
        s.init_plus()
        s.apply_qaoa(g, b)
        sz = s.spins()
    ref = o.spin_expectations(o.qaoa_state(h, J, g, b))
    assert np.max(np.abs(sz - ref)) <= 2 * bound(n, p)


def test_fp32_full_size_closed_forms(Q):
    """n = 30 in FP32 (the bench shard size): p = 1 closed-form <H_C> (pin P4) and sampled
    product-state amplitudes (pin P8) within the FP32 bound."""
    n = 30
    with Q.QSim(n, precision=Q.QSIM_FP32) as s:
        h, J = inst.random_ising(n, 31)
        s.set_ising(h, J)
        g, b = 0.23, 0.41
        s.init_plus()
        s.apply_qaoa([g], [b])
        e = s.expect_hc()
        ref = cf.p1_expect_hc(h, J, g, b)
        emax = np.sum(np.abs(h)) + np.sum(np.abs(np.triu(J, 1)))
        assert abs(e - ref) <= 2 * bound(n, 1) * emax, (e, ref)
        p = 6
        h, J = inst.product_ising(n, 5)
        g6, b6 = rand_angles(p, 55)
        s.set_ising(h, J)
        s.init_plus()
        s.apply_qaoa(g6, b6)
        zs = inst.sample_indices(n, 64, seed=3)
        got = np.array([s.amplitudes(int(z), 1)[0] for z in zs])
        refa = cf.product_amplitudes(h, g6, b6, zs)
        # per-amplitude relative error: each amplitude is a product of n single-qubit factors
        # rounded through p (2 n + 12) operations
        assert np.max(np.abs(got - refa)) <= bound(n, p) * np.max(np.abs(refa)) * 4


def test_fp32_register_stores_skewed_frames(Q, monkeypatch):
    """STG stores from registers (QSIM_TMA_STORE=0) out of the lane-skewed FP32 frame W."""
    monkeypatch.setenv("QSIM_TMA_STORE", "0")
    n, p = 23, 2
    h, J = inst.random_ising(n, 123)
    g, b = rand_angles(p, 124)
    with Q.QSim(n, precision=Q.QSIM_FP32) as s:
        s.set_ising(h, J)
        s.init_plus()
        s.apply_qaoa(g, b)
        psi = s.amplitudes()
    check_state(psi, o.qaoa_state(h, J, g, b), bound(n, p))
