"""FP32 precision mode (NEXT-4) vs the FP64 oracle: amplitude errors against the bound of
DESIGN.md §9, <H_C>, norm, and timing of an AQA evaluation in both precisions."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

torch.cuda.set_device(0)
from oracle import oracle as o  # noqa: E402
from paper_2104_03293_b200 import instances as inst  # noqa: E402
from paper_2104_03293_b200 import problems as pp  # noqa: E402
from paper_2104_03293_b200 import qsim as Q  # noqa: E402

for n in (10, 14, 16, 20, 22):
    p = 3
    h, J = inst.random_ising(n, 7 + n)
    rng = np.random.default_rng(n)
    g = rng.uniform(-1.5, 1.5, p)
    b = rng.uniform(-np.pi, np.pi, p)
    ref = o.qaoa_state(h, J, g, b)
    with Q.QSim(n, precision=Q.QSIM_FP32) as s:
        s.set_ising(h, J)
        s.init_plus()
        s.apply_qaoa(g, b)
        psi = s.amplitudes()
        e = s.expect_hc()
        nn = s.norm2()
    err = np.abs(psi - ref)
    print(f"n={n} p={p} FP32: max|d|={err.max():.3e} l2={np.linalg.norm(psi - ref):.3e} "
          f"bound={4 * p * (n + 12) * 2.0 ** -24:.3e} <H_C> {e:.9f} vs {o.expect_hc(h, J, ref):.9f} norm {nn:.9f}",
          flush=True)

n = 30
ec, xs = inst.exact_cover(n, seed=0)
h, J, C = pp.ising_from_exact_cover(ec)
r = pp.rescale_r(h, J)
sch, A, B = inst.dw_like_schedule()
for prec in (Q.QSIM_FP64, Q.QSIM_FP32):
    stream = torch.cuda.Stream()
    with Q.QSim(n, precision=prec, cuda_stream=stream.cuda_stream) as s:
        s.set_ising(h, J)
        res = []
        for it in range(3):
            s.init_plus()
            torch.cuda.synchronize()
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            s.apply_aqa(0.4 * 32, 32, sch, 2 * np.pi * A, 2 * np.pi * B / r)
            ev1.record(stream)
            e = s.expect_hc()
            torch.cuda.synchronize()
            res.append(ev0.elapsed_time(ev1))
        ps = s.success_prob([int(x) for x in xs])
    print(f"n=30 AQA p=32 prec={'FP32' if prec else 'FP64'}: {min(res) / 32:.3f} ms/layer <H_C>={e:.9f} "
          f"P_success={ps:.9f}", flush=True)
