"""Small driver for ncu captures: one AQA evaluation at n qubits, p layers (1 GPU)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=30)
ap.add_argument("--p", type=int, default=4)
ap.add_argument("--reps", type=int, default=1)
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
with Q.QSim(a.n) as sim:
    sim.set_ising(h, J)
    for _ in range(a.reps):
        sim.init_plus()
        sim.apply_aqa(0.02 * a.p, a.p, s, 2 * np.pi * A, 2 * np.pi * B / r)
        e = sim.expect_hc()
    print("expect_hc", e, "launches", sim.launches)
