"""GPU parity at the largest single-GPU size (BASELINE configs[3] at N = 1: n = 33, a 137 GB
state, four tile sets) through structured pins the oracle computes one by one (SURVEY §8c
P4, P8, P9, P10): p = 1 closed-form <H_C>, product-state amplitudes, cluster amplitudes and
expectation, sampled energies bit-exact, norm."""
import numpy as np
import pytest

from oracle import closed_forms as cf
from oracle import oracle as o
from oracle import problems as op
from paper_2104_03293_b200 import instances as inst

pytestmark = pytest.mark.gpu
N = 33


@pytest.fixture(scope="module")
def big33():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    free, _ = torch.cuda.mem_get_info()
    if free < (16 << N) + (4 << 30):
        pytest.skip("not enough device memory for n=33")
    from paper_2104_03293_b200 import build

    build.build()
    from paper_2104_03293_b200 import qsim

    s = qsim.QSim(N)
    yield s
    s.close()


def test_n33_p1_closed_form_and_norm(big33):
    h, J = inst.random_ising(N, 33)
    big33.set_ising(h, J)
    g, b = 0.31, -0.47
    big33.init_plus()
    big33.apply_qaoa([g], [b])
    e = big33.expect_hc()
    ref = cf.p1_expect_hc(h, J, g, b)
    assert abs(e - ref) <= 1e-9 * max(1.0, abs(ref)), (e, ref)
    assert abs(big33.norm2() - 1.0) <= 1e-11


def test_n33_product_state(big33):
    h, J = inst.product_ising(N, 7)
    rng = np.random.default_rng(33)
    g, b = rng.uniform(-2, 2, 3), rng.uniform(-np.pi, np.pi, 3)
    big33.set_ising(h, J)
    big33.init_plus()
    big33.apply_qaoa(g, b)
    zs = inst.sample_indices(N, 48, seed=9)
    got = np.array([big33.amplitudes(int(z), 1)[0] for z in zs])
    ref = cf.product_amplitudes(h, g, b, zs)
    assert np.max(np.abs(got - ref)) <= 1e-10 * np.max(np.abs(ref))


def test_n33_cluster_instance(big33):
    clusters = inst.spread_clusters(N, 6, seed=11)
    h, J = inst.cluster_ising(N, clusters, seed=12)
    rng = np.random.default_rng(34)
    g, b = rng.uniform(-2, 2, 2), rng.uniform(-np.pi, np.pi, 2)
    big33.set_ising(h, J)
    big33.init_plus()
    big33.apply_qaoa(g, b)
    e = big33.expect_hc()
    comp = cf.ClusterComposition(h, J, clusters, g, b)
    assert abs(e - comp.expect) <= 1e-9 * max(1.0, abs(comp.expect))
    zs = inst.sample_indices(N, 48, seed=13)
    got = np.array([big33.amplitudes(int(z), 1)[0] for z in zs])
    assert np.max(np.abs(got - comp.amplitudes(zs))) <= 1e-10 * 2.0 ** (-N / 2) * 1e4


def test_n33_energies_sampled(big33):
    a, x_star = inst.exact_cover(N, seed=2)
    h, J, C = op.exact_cover_to_ising(a)
    big33.set_ising(h, J)
    first = (1 << N) - 5000
    assert np.array_equal(big33.energies(first, 5000), o.energies(h, J, first, 5000))
    z_star = int(sum(int(x_star[i]) << i for i in range(N)))
    assert big33.energies(z_star, 1)[0] + C == 0.0
    # P10's 10^7 labels at n = 33: a contiguous block at a seeded offset (one gather, one oracle call)
    first = int(inst.sample_indices(N, 4, seed=21)[1]) % ((1 << N) - 10_000_000)
    assert np.array_equal(big33.energies(first, 10_000_000), o.energies(h, J, first, 10_000_000))
