"""Per-pass times of one AQA evaluation (n qubits, p layers, 1 GPU), in schedule order, with the
pass program of each (qsim_profile_passes): python tools/pass_times.py --n 30 --p 8"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=30)
ap.add_argument("--p", type=int, default=8)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
import torch  # noqa: E402

torch.cuda.set_device(0)
from paper_2104_03293_b200 import instances as inst  # noqa: E402
from paper_2104_03293_b200 import problems as pp  # noqa: E402
from paper_2104_03293_b200 import qsim as Q  # noqa: E402

ec, xs = inst.exact_cover(a.n, seed=0)
h, J, C = pp.ising_from_exact_cover(ec)
r = pp.rescale_r(h, J)
s, A, B = inst.dw_like_schedule()
print("env:", {k: v for k, v in os.environ.items() if k.startswith("QSIM_")}, flush=True)
with Q.QSim(a.n) as sim:
    sim.set_ising(h, J)
    for rep in range(a.reps):
        Q.qsim_profile_enable(sim.h, 1)
        sim.init_plus()
        sim.apply_aqa(0.02 * a.p, a.p, s, 2 * np.pi * A, 2 * np.pi * B / r)
        e = sim.expect_hc()
        ms, kinds = Q.qsim_profile_passes(sim.h, kinds=True)
        Q.qsim_profile_enable(sim.h, 0)
    print("expect_hc", e)
    print(" ".join(f"{k}:{t:.3f}" for t, k in zip(ms, kinds)))
    for par in (0, 1):
        for k in sorted(set(kinds)):
            sel = [t for i, (t, kk) in enumerate(zip(ms, kinds)) if kk == k and i % 2 == par and i > 0]
            if sel:
                print(f"kind {k} pass parity {par}: {len(sel)} passes, mean {np.mean(sel):.3f} ms")
