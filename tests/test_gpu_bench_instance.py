"""Full-state parity on the bench's own workload: the dense n = 30
exact-cover-shaped instance (N x 472, seed 0, J ~93 % dense, r ~ 37) under the DW-like AQA
schedule at p = 8, every one of the 2^30 amplitudes against the full CPU oracle (16 GB state +
8 GB energy table on the host), with both bars of the north star / reading R13: max-abs <= 1e-10
and ||psi_gpu - psi_oracle||_2 <= 1e-12, plus <H_C> (R12) and P_success of the planted cover.

tau = 0.4 ns (the paper's step) rather than the bench's 0.02: gamma |E| then reaches
~10^3 rad, the hardest case for the phase arithmetic (factor products instead of one sincos per
amplitude).  Needs ~45 GB of host RAM and a few minutes of the host's cores."""
import numpy as np
import pytest

from oracle import oracle as o
from oracle import problems as op
from paper_2104_03293_b200 import instances as inst

pytestmark = pytest.mark.gpu
N, P, TAU = 30, 8, 0.4


def test_bench_instance_full_state_p8():
    import psutil
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if psutil.virtual_memory().available < (45 << 30):
        pytest.skip("needs ~45 GB of free host RAM for the n = 30 oracle")
    from paper_2104_03293_b200 import qsim as Q

    a, x_star = inst.exact_cover(N, seed=0)
    h, J, C = op.exact_cover_to_ising(a)
    r = op.rescale_factor(h, J)
    s, A, B = inst.dw_like_schedule()
    A_ang, B_ang = 2 * np.pi * A, 2 * np.pi * B / r
    T = TAU * P
    z_star = int(sum(int(x_star[i]) << i for i in range(N)))
    g, _ = o.aqa_angles(T, P, s, A_ang, B_ang)
    emax = float(np.max(np.abs(h)) * N + np.sum(np.abs(J)))
    assert np.max(np.abs(g)) * emax > 100.0  # the large-angle regime this test is about

    with Q.QSim(N) as sim:
        sim.set_ising(h, J)
        sim.init_plus()
        sim.apply_aqa(T, P, s, A_ang, B_ang)
        e_gpu = sim.expect_hc()
        p_gpu = sim.success_prob([z_star])
        ref = o.aqa_state(h, J, T, P, s, A_ang, B_ang)
        CH = 1 << 26
        dmax, d2 = 0.0, 0.0
        for first in range(0, 1 << N, CH):
            got = sim.amplitudes(first, CH)
            d = got - ref[first:first + CH]
            dmax = max(dmax, float(np.max(np.abs(d))))
            d2 += float(np.vdot(d, d).real)
    er, sc = o.expect_hc(h, J, ref, with_abs=True)
    pr = o.success_prob(ref, [z_star])
    assert dmax <= 1e-10, dmax
    assert np.sqrt(d2) <= 1e-12, np.sqrt(d2)
    assert abs(e_gpu - er) <= 1e-9 * max(abs(er), sc), (e_gpu, er)
    assert abs(p_gpu - pr) <= 1e-9 * pr, (p_gpu, pr)
