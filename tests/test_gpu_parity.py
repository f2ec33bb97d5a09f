"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, element by
element, on seeded synthetic inputs.

Bars (BASELINE.json north_star; readings R12-R14):
  * amplitudes: max |psi_gpu - psi_oracle| <= 1e-10 and ||psi_gpu - psi_oracle||_2 <= 1e-12
  * <H_C>: |d| <= 1e-9 * max(|ref|, sum |psi|^2 |E|);  P_success, norm: relative 1e-9
  * E(z): bit-exact (dyadic instances)
"""
import numpy as np
import pytest

from oracle import closed_forms as cf
from oracle import oracle as o
from oracle import problems as op
from paper_2104_03293_b200 import instances as inst

pytestmark = pytest.mark.gpu

AMP_TOL = 1e-10
L2_TOL = 1e-12


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


def assert_state_close(got, ref):
    d = got - ref
    assert np.max(np.abs(d)) <= AMP_TOL, np.max(np.abs(d))
    assert np.linalg.norm(d) <= L2_TOL, np.linalg.norm(d)


def assert_expect_close(got, h, J, psi_ref):
    ref, scale = o.expect_hc(h, J, psi_ref, with_abs=True)
    assert abs(got - ref) <= 1e-9 * max(abs(ref), scale, 1e-300), (got, ref)


def run_gpu(Q, h, J, gam, bet, n=None):
    n = len(h) if n is None else n
    with Q.QSim(n) as s:
        s.set_ising(h, J)
        s.init_plus()
        s.apply_qaoa(gam, bet)
        return s.amplitudes(), s.expect_hc(), s.norm2(), s.launches


# ------------------------------------------------------------------ small states (one CTA)
@pytest.mark.parametrize("n,p", [(1, 3), (2, 2), (5, 4), (9, 3), (12, 5)])
def test_small_state_parity(Q, n, p):
    h, J = inst.random_ising(n, 100 + n)
    g, b = rand_angles(p, n)
    psi, e, nrm, _ = run_gpu(Q, h, J, g, b)
    ref = o.qaoa_state(h, J, g, b)
    assert_state_close(psi, ref)
    assert_expect_close(e, h, J, ref)
    assert abs(nrm - 1.0) <= 1e-12


# ------------------------------------------------------------------ tiled passes (m >= 13)
@pytest.mark.parametrize("n,p", [(13, 1), (13, 3), (14, 2), (16, 4), (20, 3), (21, 2), (22, 5), (24, 2)])
def test_tiled_parity(Q, n, p):
    h, J = inst.random_ising(n, 200 + n)
    g, b = rand_angles(p, 300 + n + p)
    psi, e, nrm, launches = run_gpu(Q, h, J, g, b)
    ref = o.qaoa_state(h, J, g, b)
    assert_state_close(psi, ref)
    assert_expect_close(e, h, J, ref)
    assert abs(nrm - 1.0) <= 1e-12
    assert launches > 0


def test_mixer_forms_and_edge_angles(Q):
    """beta where |tan beta| > 1 (form 1), exactly pi/4 and pi/2, beta = 0, gamma = 0."""
    n = 15
    h, J = inst.random_ising(n, 7)
    for bet in ([np.pi / 2, 0.0, np.pi / 4], [1.3, -1.3, 2.9], [0.0, 0.0, 0.0], [np.pi / 4, -np.pi / 4, 3 * np.pi / 4]):
        gam = [0.3, 0.0, -1.1]
        psi, e, _, _ = run_gpu(Q, h, J, gam, bet)
        ref = o.qaoa_state(h, J, gam, bet)
        assert_state_close(psi, ref)


def test_trivial_problem_P7(Q):
    n = 17
    g, b = rand_angles(4, 3)
    psi, e, _, _ = run_gpu(Q, np.zeros(n), np.zeros((n, n)), g, b)
    ref = np.exp(-1j * n * np.sum(b)) * 2.0 ** (-n / 2)
    assert np.max(np.abs(psi - ref)) <= AMP_TOL
    assert abs(e) <= 1e-12


def test_continue_without_init(Q):
    """apply(g1,b1) then apply(g2,b2) == apply(g1+g2, b1+b2) (second call loads the state)."""
    n = 18
    h, J = inst.random_ising(n, 9)
    g, b = rand_angles(5, 9)
    with Q.QSim(n) as s:
        s.set_ising(h, J)
        s.init_plus()
        s.apply_qaoa(g[:2], b[:2])
        s.apply_qaoa(g[2:], b[2:])
        psi = s.amplitudes()
        e = s.expect_hc()
    ref = o.qaoa_state(h, J, g, b)
    assert_state_close(psi, ref)
    assert_expect_close(e, h, J, ref)


def test_reinit_and_plus_state(Q):
    n = 16
    h, J = inst.random_ising(n, 10)
    with Q.QSim(n) as s:
        s.set_ising(h, J)
        s.apply_qaoa([0.4], [0.2])
        s.init_plus()
        psi = s.amplitudes()
        assert np.all(psi == 2.0 ** (-n / 2))
        assert abs(s.expect_hc()) <= 1e-12
        assert abs(s.norm2() - 1.0) <= 1e-13


def test_aqa_parity(Q):
    n = 20
    a, x_star = inst.exact_cover(n, F=60, seed=1, planted_rows=5, weight=9)
    h, J, C = op.exact_cover_to_ising(a)
    r = op.rescale_factor(h, J)
    s, A, B = inst.dw_like_schedule()
    A = 2 * np.pi * A
    B = 2 * np.pi * B / r
    p, T = 8, 0.4 * 8
    with Q.QSim(n) as sim:
        sim.set_ising(h, J)
        sim.init_plus()
        sim.apply_aqa(T, p, s, A, B)
        psi = sim.amplitudes()
        e = sim.expect_hc()
        z_star = int(sum(int(x_star[i]) << i for i in range(n)))
        ps = sim.success_prob([z_star])
    ref = o.aqa_state(h, J, T, p, s, A, B)
    assert_state_close(psi, ref)
    assert_expect_close(e, h, J, ref)
    pref = o.success_prob(ref, [z_star])
    assert abs(ps - pref) <= 1e-9 * pref


def test_energies_bit_exact(Q):
    for n, seed in [(6, 1), (12, 2), (13, 3), (20, 4), (22, 5)]:
        h, J = inst.random_ising(n, seed)
        with Q.QSim(n) as s:
            s.set_ising(h, J)
            e = s.energies()
        assert np.array_equal(e, o.energies(h, J))


def test_two_sat_config1_grid(Q):
    """configs[0]: n=12 planted 2-SAT, AQA p=5 and the p=1 64x64 grid."""
    n = 12
    clauses, x_star = inst.planted_2sat(n, seed=0)
    h, J, C = op.two_sat_to_ising(n, clauses)
    gs, emin, cnt = o.ground_states(h, J)
    assert cnt == 1
    s_, A, B = inst.toy_schedule()
    with Q.QSim(n) as sim:
        sim.set_ising(h, J)
        sim.init_plus()
        sim.apply_aqa(2.5, 5, s_, A, B)
        ref = o.aqa_state(h, J, 2.5, 5, s_, A, B)
        assert_state_close(sim.amplitudes(), ref)
        assert abs(sim.success_prob(gs) - o.success_prob(ref, gs)) <= 1e-9 * o.success_prob(ref, gs)
        betas = np.arange(64) * np.pi / 64
        gammas = np.arange(64) * 2 * np.pi / 64
        worst = 0.0
        for bi in range(0, 64, 3):
            for gi in range(0, 64, 3):
                sim.init_plus()
                sim.apply_qaoa([gammas[gi]], [betas[bi]])
                e = sim.expect_hc()
                ref = o.qaoa_state(h, J, [gammas[gi]], [betas[bi]])
                er, sc = o.expect_hc(h, J, ref, with_abs=True)
                worst = max(worst, abs(e - er) / max(abs(er), sc))
        assert worst <= 1e-9


# ------------------------------------------------------------------ errors
def test_error_codes(Q):
    with pytest.raises(Q.QsimError) as ei:
        Q.qsim_create(12, 7)  # unknown precision
    assert ei.value.code == Q.QSIM_EINVAL
    with Q.QSim(14) as s:
        with pytest.raises(Q.QsimError) as ei:
            s.apply_qaoa([0.1], [0.2])
        assert ei.value.code == Q.QSIM_ESTATE
        h, J = inst.random_ising(14, 1)
        with pytest.raises(Q.QsimError) as ei:
            s.set_ising(np.full(14, np.nan), J)
        assert ei.value.code == Q.QSIM_EINVAL
        s.set_ising(h, J)
        with pytest.raises(Q.QsimError) as ei:
            s.apply_qaoa([], [])
        assert ei.value.code == Q.QSIM_EINVAL
        with pytest.raises(Q.QsimError) as ei:
            s.apply_qaoa([np.inf], [0.1])
        assert ei.value.code == Q.QSIM_EINVAL
        with pytest.raises(Q.QsimError) as ei:
            Q.qsim_get_amplitudes(s.h, (1 << 14) - 1, 2)
        assert ei.value.code == Q.QSIM_ERANGE
        with pytest.raises(Q.QsimError) as ei:
            s.success_prob([1 << 14])
        assert ei.value.code == Q.QSIM_ERANGE
        with pytest.raises(Q.QsimError) as ei:
            s.apply_aqa(1.0, 1, [0, 1], [1, 0], [0, 1])
        assert ei.value.code == Q.QSIM_EINVAL


# ------------------------------------------------------------------ full size (bench config)
@pytest.fixture(scope="module")
def big30(Q):
    """The bench launch configuration (n=30, one GPU): one handle reused by the tests."""
    s = Q.QSim(30)
    yield s
    s.close()


def test_full_size_p1_closed_form_expectation(Q, big30):
    n = 30
    h, J = inst.random_ising(n, 31)
    big30.set_ising(h, J)
    for g, b in [(0.23, 0.41), (1.1, -0.7)]:
        big30.init_plus()
        big30.apply_qaoa([g], [b])
        e = big30.expect_hc()
        ref = cf.p1_expect_hc(h, J, g, b)
        scale = np.sum(np.abs(h)) + np.sum(np.abs(np.triu(J, 1)))
        assert abs(e - ref) <= 1e-9 * max(abs(ref), 1.0) + 1e-12 * scale, (e, ref)
        assert abs(big30.norm2() - 1.0) <= 1e-11


def test_full_size_product_state(Q, big30):
    n, p = 30, 6
    h, J = inst.product_ising(n, 5)
    g, b = rand_angles(p, 55)
    big30.set_ising(h, J)
    big30.init_plus()
    big30.apply_qaoa(g, b)
    zs = inst.sample_indices(n, 64, seed=3)
    got = np.array([big30.amplitudes(int(z), 1)[0] for z in zs])
    ref = cf.product_amplitudes(h, g, b, zs)
    assert np.max(np.abs(got - ref)) <= AMP_TOL
    assert np.max(np.abs(got - ref)) <= 1e-10 * np.max(np.abs(ref))


def test_full_size_cluster_instance(Q, big30):
    n, p = 30, 4
    clusters = inst.spread_clusters(n, 6, seed=4)
    h, J = inst.cluster_ising(n, clusters, seed=8)
    g, b = rand_angles(p, 66)
    big30.set_ising(h, J)
    big30.init_plus()
    big30.apply_qaoa(g, b)
    e = big30.expect_hc()
    comp = cf.ClusterComposition(h, J, clusters, g, b)
    assert abs(e - comp.expect) <= 1e-9 * max(abs(comp.expect), 1.0)
    zs = inst.sample_indices(n, 64, seed=5)
    got = np.array([big30.amplitudes(int(z), 1)[0] for z in zs])
    ref = comp.amplitudes(zs)
    assert np.max(np.abs(got - ref)) <= AMP_TOL
    # contiguous block read through the full gather path
    blk = big30.amplitudes(12345, 4096)
    assert np.max(np.abs(blk - comp.amplitudes(np.arange(12345, 12345 + 4096)))) <= AMP_TOL


def test_full_size_energies_sampled(Q, big30):
    n = 30
    a, x_star = inst.exact_cover(n, seed=0)
    h, J, C = op.exact_cover_to_ising(a)
    big30.set_ising(h, J)
    zs = inst.sample_indices(n, 20000, seed=6)
    first = int(zs[100])
    cnt = min(20000, (1 << n) - first)
    e = big30.energies(first, cnt)
    assert np.array_equal(e, o.energies(h, J, first, cnt))
    z_star = int(sum(int(x_star[i]) << i for i in range(n)))
    assert big30.energies(z_star, 1)[0] + C == 0.0


def test_full_size_energies_all_labels(Q, big30):
    """P10 at the bench size: E(z) of every one of the 2^30 labels of the bench's exact-cover
    instance, bit-exact against the oracle (dyadic data, reading R14), in chunks of 2^26."""
    n = 30
    a, _ = inst.exact_cover(n, seed=0)
    h, J, C = op.exact_cover_to_ising(a)
    big30.set_ising(h, J)
    CH = 1 << 26
    for first in range(0, 1 << n, CH):
        assert np.array_equal(big30.energies(first, CH), o.energies(h, J, first, CH)), first


@pytest.mark.parametrize("env", [{"QSIM_TURN_PW": "0"}, {"QSIM_RUNSPLIT": "0"}, {"QSIM_L2PROMO": "128"}])
def test_full_size_kernel_switches(Q, env, monkeypatch):
    """The documented switches of the single-GPU n = 30 path: QSIM_TURN_PW=0 runs the turning
    passes on the group-synchronous kernel instead of the per-warp one, QSIM_RUNSPLIT=0 uses
    contiguous runs instead of the split-run layout, QSIM_L2PROMO=128 keeps 128-byte L2 promotion
    on the run sets' tensor maps; each against the p = 1 closed form (P4) and the product-state
    amplitudes (P8) at p = 3."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    n = 30
    h, J = inst.random_ising(n, 77)
    with Q.QSim(n) as s:
        s.set_ising(h, J)
        s.init_plus()
        s.apply_qaoa([0.37], [-0.52])
        e = s.expect_hc()
        ref = cf.p1_expect_hc(h, J, 0.37, -0.52)
        assert abs(e - ref) <= 1e-9 * max(abs(ref), 1.0), (e, ref)
        hp, Jp = inst.product_ising(n, 9)
        g, b = rand_angles(3, 88)
        s.set_ising(hp, Jp)
        s.init_plus()
        s.apply_qaoa(g, b)
        zs = inst.sample_indices(n, 48, seed=8)
        got = np.array([s.amplitudes(int(z), 1)[0] for z in zs])
    assert np.max(np.abs(got - cf.product_amplitudes(hp, g, b, zs))) <= AMP_TOL


# ------------------------------------------------------------------ NEXT-2: <sigma^z_i>
@pytest.mark.parametrize("n,p", [(5, 3), (16, 3), (22, 2)])
def test_spin_expectations(Q, n, p):
    h, J = inst.random_ising(n, 500 + n)
    g, b = rand_angles(p, 600 + n)
    with Q.QSim(n) as s:
        s.set_ising(h, J)
        s.init_plus()
        s.apply_qaoa(g, b)
        sz = s.spins()
    ref = o.spin_expectations(o.qaoa_state(h, J, g, b))
    assert np.max(np.abs(sz - ref)) <= 1e-11


def test_spin_trace_aqa(Q):
    n, p = 17, 5
    h, J = inst.random_ising(n, 77)
    s_, A, B = inst.toy_schedule()
    with Q.QSim(n) as s:
        s.set_ising(h, J)
        s.init_plus()
        tr = s.apply_aqa_traced(2.5, p, s_, A, B)
        psi = s.amplitudes()
    g, b = o.aqa_angles(2.5, p, s_, A, B)
    ref = o.init_plus(n)
    for k in range(p):
        o.apply_layers(h, J, g[k:k + 1], b[k:k + 1], ref)
        assert np.max(np.abs(tr[k] - o.spin_expectations(ref))) <= 1e-11
    assert_state_close(psi, ref)


def test_full_size_spins_p1_closed_form(Q, big30):
    n = 30
    h, J = inst.random_ising(n, 35)
    big30.set_ising(h, J)
    big30.init_plus()
    big30.apply_qaoa([0.29], [-0.61])
    sz = big30.spins()
    assert np.max(np.abs(sz - cf.p1_spins(h, J, 0.29, -0.61))) <= 1e-10


# ------------------------------------------------------------------ NEXT-3: enumeration
@pytest.mark.parametrize("n,kind", [(12, "2sat"), (16, "ising"), (20, "cover"), (21, "ising")])
def test_ground_states_enumeration(Q, n, kind):
    if kind == "2sat":
        clauses, _ = inst.planted_2sat(n, seed=1)
        h, J, C = op.two_sat_to_ising(n, clauses)
    elif kind == "cover":
        a, _ = inst.exact_cover(n, F=80, seed=3, planted_rows=5, weight=13)
        h, J, C = op.exact_cover_to_ising(a)
    else:
        h, J = inst.random_ising(n, 900 + n)
    with Q.QSim(n) as s:
        s.set_ising(h, J)
        gs, emin, cnt = s.ground_states(max_out=16)
    rgs, remin, rcnt = o.ground_states(h, J, max_out=16)
    assert emin == remin and cnt == rcnt and gs == rgs[: len(gs)]


def test_ground_states_full_size_exact_cover(Q, big30):
    """n = 30 exact-cover-shaped instance: the planted cover is a ground state (E + C = 0)."""
    n = 30
    a, x_star = inst.exact_cover(n, seed=0)
    h, J, C = op.exact_cover_to_ising(a)
    big30.set_ising(h, J)
    gs, emin, cnt = big30.ground_states(max_out=8)
    z_star = int(sum(int(x_star[i]) << i for i in range(n)))
    assert emin + C == 0.0 and z_star in gs and cnt >= 1
    assert o.energy(h, J, gs[0]) == emin


# ------------------------------------------------------------------ NEXT-1: QSDS combined step
@pytest.mark.parametrize("n,steps", [(6, 4), (12, 3), (15, 5), (22, 3)])
def test_qsds_parity(Q, n, steps):
    h, J = inst.random_ising(n, 700 + n)
    s_, A, B = inst.dw_like_schedule()
    A, B = 2 * np.pi * A / 10, 2 * np.pi * B / 10
    tau = 0.4
    with Q.QSim(n) as s:
        s.set_ising(h, J)
        s.init_plus()
        s.apply_qsds(tau, steps, s_, A, B)
        psi = s.amplitudes()
        e = s.expect_hc()
    ref = o.qsds_state(h, J, tau, steps, s_, A, B)
    assert_state_close(psi, ref)
    assert_expect_close(e, h, J, ref)


def test_qsds_after_flipped_qaoa(Q):
    """QSDS continuing a state whose qubits carry X-gate flips (|tan beta| > 1 mixers)."""
    n = 16
    h, J = inst.random_ising(n, 55)
    s_, A, B = inst.toy_schedule()
    with Q.QSim(n) as s:
        s.set_ising(h, J)
        s.init_plus()
        s.apply_qaoa([0.7, -0.4], [1.3, 2.2])
        s.apply_qsds(0.3, 3, s_, A, B)
        psi = s.amplitudes()
    ref = o.qaoa_state(h, J, [0.7, -0.4], [1.3, 2.2])
    # continue the oracle state with the QSDS steps: compose via a fresh oracle run on |ref>
    import oracle.oracle as oo
    tau, steps = 0.3, 3
    cur = ref.copy()
    L = oo.lib()
    import ctypes
    L.oracle_apply_qsds(n, oo._dp(np.ascontiguousarray(h)), oo._dp(np.ascontiguousarray(J)), tau, steps,
                        oo._dp(np.ascontiguousarray(s_, dtype=float)), oo._dp(np.ascontiguousarray(A, dtype=float)),
                        oo._dp(np.ascontiguousarray(B, dtype=float)), len(s_), oo._dp(cur.view(np.float64)))
    assert_state_close(psi, cur)


# ------------------------------------------------------------------ NEXT-4: Hadamard circuits
@pytest.mark.parametrize("n", [8, 14, 21])
def test_hadamard_layers(Q, n):
    """(H^n)^11 |+> = |0>; (H^n)^2 = identity; a random state after 3 layers vs dense."""
    h, J = inst.random_ising(n, 3)
    with Q.QSim(n) as s:
        s.set_ising(h, J)
        s.init_plus()
        s.apply_hadamard(11)
        psi = s.amplitudes()
        ref = np.zeros(1 << n, dtype=complex)
        ref[0] = 1.0
        assert np.max(np.abs(psi - ref)) <= 1e-12
        g, b = rand_angles(2, n)
        s.init_plus()
        s.apply_qaoa(g, b)
        s.apply_hadamard(3)
        psi3 = s.amplitudes()
    st = o.qaoa_state(h, J, g, b)
    # H^{otimes n} = normalised Walsh-Hadamard transform (qubit j <-> bit j)
    wht = st.copy()
    for q in range(n):
        wht = wht.reshape(-1, 2, 1 << q)
        wht = np.stack([wht[:, 0] + wht[:, 1], wht[:, 0] - wht[:, 1]], axis=1).reshape(-1) / np.sqrt(2)
    assert np.max(np.abs(psi3 - wht)) <= 1e-12


def test_hadamard_after_flipped_qaoa(Q):
    """Hadamard layers on a state whose qubits carry X-gate flips (|tan beta| > 1 mixers)."""
    n = 17
    h, J = inst.random_ising(n, 4)
    g, b = [0.5, -0.9], [1.2, 2.4]
    with Q.QSim(n) as s:
        s.set_ising(h, J)
        s.init_plus()
        s.apply_qaoa(g, b)
        s.apply_hadamard(1)
        psi = s.amplitudes()
    wht = o.qaoa_state(h, J, g, b)
    for q in range(n):
        wht = wht.reshape(-1, 2, 1 << q)
        wht = np.stack([wht[:, 0] + wht[:, 1], wht[:, 0] - wht[:, 1]], axis=1).reshape(-1) / np.sqrt(2)
    assert np.max(np.abs(psi - wht)) <= 1e-12


# ------------------------------------------------------------------ edge cases
@pytest.mark.parametrize("n", [13, 15, 17, 19, 21])
def test_all_set_layouts_p1_p2(Q, n):
    """Every tile-set count (runs of 1..9 bits), p = 1 (no turning pass) and p = 2."""
    h, J = inst.random_ising(n, 1000 + n)
    for p in (1, 2):
        g, b = rand_angles(p, 1100 + n + p)
        psi, e, nrm, _ = run_gpu(Q, h, J, g, b)
        ref = o.qaoa_state(h, J, g, b)
        assert_state_close(psi, ref)
        assert_expect_close(e, h, J, ref)


def test_aqa_minimum_p(Q):
    n = 14
    h, J = inst.random_ising(n, 8)
    s_, A, B = inst.toy_schedule()
    with Q.QSim(n) as s:
        s.set_ising(h, J)
        s.init_plus()
        s.apply_aqa(1.0, 2, s_, A, B)
        psi = s.amplitudes()
    assert_state_close(psi, o.aqa_state(h, J, 1.0, 2, s_, A, B))


def test_degenerate_ground_states_and_chunked_readback(Q):
    """h = 0: z and its complement are both ground states (reading R11); the readback of
    2^23 amplitudes crosses the 2^22-amplitude gather chunk."""
    n = 23
    _, J = inst.random_ising(n, 12)
    h = np.zeros(n)
    g, b = rand_angles(2, 12)
    with Q.QSim(n) as s:
        s.set_ising(h, J)
        gs, emin, cnt = s.ground_states(max_out=8)
        s.init_plus()
        s.apply_qaoa(g, b)
        psi = s.amplitudes()
        ps = s.success_prob(gs)
        en = s.energies()  # 2^23 energies cross the 2^23-energy probe chunk boundary exactly
    assert cnt % 2 == 0 and all(((1 << n) - 1 - z) in gs for z in gs)
    ref = o.qaoa_state(h, J, g, b)
    assert_state_close(psi, ref)
    assert abs(ps - o.success_prob(ref, gs)) <= 1e-9 * o.success_prob(ref, gs)
    assert np.array_equal(en, o.energies(h, J))
    assert np.array_equal(psi, psi[(1 << n) - 1 - np.arange(1 << n)])  # P5 at the GPU


def test_set_ising_twice_and_reuse(Q):
    n = 16
    h1, J1 = inst.random_ising(n, 21)
    h2, J2 = inst.random_ising(n, 22)
    g, b = rand_angles(2, 23)
    with Q.QSim(n) as s:
        s.set_ising(h1, J1)
        s.init_plus()
        s.apply_qaoa(g, b)
        s.set_ising(h2, J2)
        s.init_plus()
        s.apply_qaoa(g, b)
        psi = s.amplitudes()
        e = s.expect_hc()
    ref = o.qaoa_state(h2, J2, g, b)
    assert_state_close(psi, ref)
    assert_expect_close(e, h2, J2, ref)


# ------------------------------------------------------------------ NEXT-3: more minimisers than max_out
@pytest.mark.parametrize("n,zeros,max_out", [(16, 6, 5), (20, 9, 37), (17, 17, 3)])
def test_ground_states_first_minimisers_when_count_exceeds_max_out(Q, n, zeros, max_out):
    """qsim.h promises the first max_out minimisers in ascending label order.  A product
    instance (J = 0) with `zeros` zero fields has 2^zeros minimisers (brute force by the
    oracle); the smallest max_out labels must come back whatever the CTA scheduling order."""
    rng = np.random.default_rng(n + zeros)
    h = rng.choice([-1.5, -0.5, 0.5, 1.0], size=n)
    h[rng.permutation(n)[:zeros]] = 0.0
    J = np.zeros((n, n))
    with Q.QSim(n) as s:
        s.set_ising(h, J)
        gs, emin, cnt = s.ground_states(max_out=max_out)
    rgs, remin, rcnt = o.ground_states(h, J, max_out=max_out)
    assert cnt == rcnt == 2 ** zeros and emin == remin == -np.sum(np.abs(h))
    assert gs == rgs == sorted(gs) and len(gs) == max_out


def test_enumerate_beyond_40_qubits(Q):
    """qsim_enumerate at n = 41 (the state-less entry accepts n <= 48): a J = 0 product instance
    has the unique minimiser z_i = [h_i < 0] and E_min = -sum |h| (closed form, brute force not
    needed); one coupled pair checks the couplings at positions >= 40."""
    n = 41
    rng = np.random.default_rng(41)
    h = rng.choice([-2.0, -1.0, -0.5, 0.5, 1.0, 2.0], size=n)
    J = np.zeros((n, n))
    gs, emin, cnt, ms = Q.qsim_enumerate(h, J, max_out=4)
    z = sum(1 << i for i in range(n) if h[i] < 0)
    assert cnt == 1 and gs == [z] and emin == -np.sum(np.abs(h))
    # couple qubits 39 and 40 antiferromagnetically with a field-free pair: E_min gains -|J|
    h2 = h.copy()
    h2[39] = h2[40] = 0.0
    J2 = np.zeros((n, n))
    J2[39, 40] = 3.0
    gs2, emin2, cnt2, _ = Q.qsim_enumerate(h2, J2, max_out=4)
    base = sum(1 << i for i in range(39) if h2[i] < 0)
    assert cnt2 == 2 and emin2 == -np.sum(np.abs(h2)) - 3.0
    assert gs2 == sorted([base | (1 << 39), base | (1 << 40)])


def test_boundary_errors_and_hadamard_without_problem(Q):
    """J with a non-zero diagonal is EINVAL (eq:HC has no self-coupling); the
    Hadamard benchmark needs no problem data."""
    n = 14
    h, J = inst.random_ising(n, 3)
    Jd = J.copy()
    Jd[2, 2] = 0.5
    with Q.QSim(n) as s:
        with pytest.raises(Q.QsimError) as ei:
            s.set_ising(h, Jd)
        assert ei.value.code == Q.QSIM_EINVAL
        s.init_plus()
        s.apply_hadamard(2)  # H^2 = I: |+> comes back
        psi = s.amplitudes()
        assert Q.qsim_num_qubits(s.h) == n and s.spins().shape == (n,)
    assert np.max(np.abs(psi - 2.0 ** (-n / 2))) <= 1e-14


@pytest.mark.parametrize("n", [13, 22])
def test_energies_are_the_reducing_pass_energies(Q, n):
    """qsim_energies returns E(z) from the hot path's own arithmetic (tile records + the frame-Z
    register tree of the reducing pass).  With a non-dyadic instance (bit-exactness not claimed,
    reading R14) the sum over |psi|^2 E of the returned energies must reproduce the fused
    <H_C> of the last pass to rounding, and every E(z) the oracle's to 1e-12 relative."""
    rng = np.random.default_rng(n)
    h = rng.normal(size=n)
    J = np.triu(rng.normal(size=(n, n)), 1)
    g, b = rand_angles(3, n)
    with Q.QSim(n) as s:
        s.set_ising(h, J)
        s.init_plus()
        s.apply_qaoa(g, b)
        e_fused = s.expect_hc()
        psi = s.amplitudes()
        en = s.energies()
    ref = o.energies(h, J)
    assert np.max(np.abs(en - ref)) <= 1e-12 * np.max(np.abs(ref))
    p = np.abs(psi) ** 2
    assert abs(np.dot(p, en) - e_fused) <= 1e-11 * np.dot(p, np.abs(en))


# ------------------------------------------------------------------ batched small-state QAOA (grid scans)
@pytest.mark.parametrize("n,p,count", [(8, 1, 37), (12, 3, 65), (5, 2, 1)])
def test_qaoa_batch_matches_oracle(Q, n, p, count):
    """qsim_qaoa_batch: <H_C> of |beta_b, gamma_b> for every angle set b (eq:QAOA_state),
    one CTA per set, against the oracle's state and expectation per set (reading R12 bar)."""
    rng = np.random.default_rng(n * 100 + p)
    if n == 12:
        clauses, _ = inst.planted_2sat(n, seed=2)
        h, J, C = op.two_sat_to_ising(n, clauses)
    else:
        h, J = inst.random_ising(n, n + 5)
    g = rng.uniform(-2, 2, (count, p))
    b = rng.uniform(-np.pi, np.pi, (count, p))
    with Q.QSim(n) as s:
        s.set_ising(h, J)
        got = s.qaoa_batch(g, b)
        s.init_plus()  # the batch leaves the handle's state alone
        assert np.max(np.abs(s.amplitudes() - 2.0 ** (-n / 2))) == 0.0
        assert s.qaoa_batch(np.zeros((0, p)), np.zeros((0, p))).shape == (0,)
    for k in range(count):
        psi = o.qaoa_state(h, J, g[k], b[k])
        assert_expect_close(got[k], h, J, psi)


def test_qaoa_batch_needs_small_state(Q):
    with Q.QSim(13) as s:
        h, J = inst.random_ising(13, 1)
        s.set_ising(h, J)
        with pytest.raises(Q.QsimError) as ei:
            s.qaoa_batch([[0.1]], [[0.2]])
        assert ei.value.code == Q.QSIM_EUNSUPPORTED


# ------------------------------------------------------------------ caller-owned state buffer
def test_caller_owned_state_buffer(Q):
    """qsim_create_ex with state_buf: the library computes in the caller's device memory (here a
    torch tensor) and never frees it; with |tan beta| < 1 no index flips occur, so the tensor holds
    the amplitudes in logical order after the call."""
    import torch

    n = 20
    h, J = inst.random_ising(n, 61)
    g, b = np.array([0.4, -0.3]), np.array([0.5, -0.6])
    buf = torch.zeros(1 << n, dtype=torch.complex128, device="cuda")
    st = torch.cuda.current_stream()
    with Q.QSim(n, state_buf=buf.data_ptr(), buf_bytes=buf.numel() * 16, cuda_stream=st.cuda_stream) as s:
        s.set_ising(h, J)
        s.init_plus()
        s.apply_qaoa(g, b)
        psi = s.amplitudes()
    ref = o.qaoa_state(h, J, g, b)
    assert_state_close(psi, ref)
    torch.cuda.synchronize()
    assert np.max(np.abs(buf.cpu().numpy() - ref)) <= AMP_TOL
    with pytest.raises(Q.QsimError) as ei:  # too small a buffer is EINVAL
        Q.QSim(n, state_buf=buf.data_ptr(), buf_bytes=buf.numel() * 8, cuda_stream=st.cuda_stream)
    assert ei.value.code == Q.QSIM_EINVAL


def test_c_example_runs_against_oracle(Q, tmp_path):
    """examples/qaoa_c.c (the C-ABI from plain C) on the GPU: its <H_C>, norm and ground-state energy
    against the oracle on the same instance."""
    import re
    import subprocess

    from tests.test_abi_host import _build_c_example, c_example_instance

    exe = _build_c_example(tmp_path)
    n, p = 18, 3
    out = subprocess.run([exe, str(n), str(p)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    m = re.search(r"<H_C>=(\S+) norm=(\S+) .* E_min=(\S+) minimisers=(\d+)", out.stdout)
    assert m, out.stdout
    h, J, g, b = c_example_instance(n, p)
    ref = o.qaoa_state(h, J, g, b)
    assert_expect_close(float(m.group(1)), h, J, ref)
    gs, emin, cnt = o.ground_states(h, J)
    assert float(m.group(3)) == emin and int(m.group(4)) == cnt
