"""Time each tile-set pass type in isolation: python tools/passbench.py --n 30"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, nargs="+", default=[30])
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--f32", action="store_true", help="FP32 state (8 B per amplitude)")
a = ap.parse_args()
print("env:", {k: v for k, v in os.environ.items() if k.startswith("QSIM_")}, flush=True)
torch.cuda.set_device(0)
from paper_2104_03293_b200 import instances as inst  # noqa: E402
from paper_2104_03293_b200 import qsim as Q  # noqa: E402

for n in a.n:
    h, J = inst.random_ising(n, 1)
    with Q.QSim(n, precision=Q.QSIM_FP32 if a.f32 else Q.QSIM_FP64) as s:
        s.set_ising(h, J)
        nsets = 16  # upper bound; qsim_bench_pass rejects indices past the last set
        ideal = (16 if a.f32 else 32) * 2.0 ** n / 6455.9e9 * 1e3
        for k in range(nsets):
            for ph in (-3, -2, -1, 0, 1):
                try:
                    ms = Q.qsim_bench_pass(s.h, k, ph, a.reps)
                except Q.QsimError:
                    break  # past the last set
                fac = 0.5 if ph in (-2, -3) else 1.0  # read-only / write-only move half the bytes
                print(f"n={n} set={k} phase={ph} {ms:.3f} ms  ({fac * ideal / ms * 100:.1f}% of measured HBM peak)",
                      flush=True)
