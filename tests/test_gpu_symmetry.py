"""GPU symmetry pins at tiled sizes: relations the mathematics fixes
between two runs of the CUDA path, so they hold at any n without an oracle state.  The sizes
span several tile sets, the turning pass and a ragged last set.

  P5  (-h, J) gives psi'_z = psi_{~z}      (X^(x)n commutes with H_D and |+>, flips every s_i)
  P6  beta_k -> beta_k + pi multiplies every amplitude by (-1)^n   (R_x(2pi) = -I per qubit)
  P16 relabelling qubits by pi in (h, J) relabels the amplitude index bits by pi
"""
import numpy as np
import pytest

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


def run(Q, h, J, g, b):
    with Q.QSim(len(h)) as s:
        s.set_ising(h, J)
        s.init_plus()
        s.apply_qaoa(g, b)
        return s.amplitudes(), s.expect_hc()


def angles(p, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(-1.5, 1.5, p), rng.uniform(-np.pi, np.pi, p)


def close(a, b):
    d = a - b
    assert np.max(np.abs(d)) <= AMP_TOL, np.max(np.abs(d))
    assert np.linalg.norm(d) <= L2_TOL, np.linalg.norm(d)


@pytest.mark.parametrize("n", [21, 25])
def test_P5_spin_flip_gpu(Q, n):
    h, J = inst.random_ising(n, 40 + n)
    g, b = angles(3, n)
    psi, e = run(Q, h, J, g, b)
    psi_f, e_f = run(Q, -h, J, g, b)
    close(psi_f, psi[::-1])  # ~z = (2^n - 1) - z
    assert abs(e_f - e) <= 1e-9 * max(abs(e), 1.0)


@pytest.mark.parametrize("n", [22, 26])
def test_P6_beta_shift_gpu(Q, n):
    h, J = inst.random_ising(n, 50 + n)
    g, b = angles(3, 60 + n)
    psi, _ = run(Q, h, J, g, b)
    shifted = b.copy()
    shifted[1] += np.pi
    psi_s, _ = run(Q, h, J, g, shifted)
    close(psi_s, (-1.0) ** n * psi)


@pytest.mark.parametrize("n", [23, 27])
def test_P16_permutation_covariance_gpu(Q, n):
    h, J = inst.random_ising(n, 70 + n)
    g, b = angles(2, 80 + n)
    pi = np.random.default_rng(n).permutation(n)  # qubit i -> qubit pi[i]
    h2 = np.zeros(n)
    h2[pi] = h
    J2 = np.zeros((n, n))
    for i in range(n):
        for j in range(i + 1, n):
            a, c = sorted((pi[i], pi[j]))
            J2[a, c] = J[i, j]
    psi, e = run(Q, h, J, g, b)
    psi2, e2 = run(Q, h2, J2, g, b)
    z = np.arange(1 << n, dtype=np.int64)
    z2 = np.zeros_like(z)
    for i in range(n):
        z2 |= ((z >> i) & 1) << int(pi[i])
    close(psi2[z2], psi)
    assert abs(e2 - e) <= 1e-9 * max(abs(e), 1.0)
