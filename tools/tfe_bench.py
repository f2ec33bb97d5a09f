"""NEXT-3 measurement: GPU full enumeration of all 2^N energies on exact-cover-shaped
instances (N x 472) vs the paper's t_FE on 4 x A100, context only.

    python tools/tfe_bench.py --qubits 30 32 34 36 38 40
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2104_03293_b200 import instances as inst  # noqa: E402
from paper_2104_03293_b200 import problems as pp  # noqa: E402
from paper_2104_03293_b200 import qsim as Q  # noqa: E402

PAPER_TFE = {30: 1.7, 32: 1.7, 34: 2.4, 36: 6.0, 38: 22.3, 40: 91.8}  # s on 4 x A100

ap = argparse.ArgumentParser()
ap.add_argument("--qubits", type=int, nargs="+", default=[30, 32, 34, 36])
a = ap.parse_args()
torch.cuda.set_device(0)
for n in a.qubits:
    ec, x_star = inst.exact_cover(n, seed=0)
    h, J, C = pp.ising_from_exact_cover(ec)
    Q.qsim_enumerate(h, J, 4)  # warm-up
    gs, emin, cnt, ms = Q.qsim_enumerate(h, J, 4)
    z_star = int(sum(int(x_star[i]) << i for i in range(n)))
    rec = {"n": n, "ms": ms, "energies_per_s": 2.0 ** n / (ms / 1e3), "emin_plus_C": emin + C,
           "count": cnt, "planted_is_ground_state": z_star in gs,
           "paper_t_FE_s_4xA100": PAPER_TFE.get(n)}
    print(json.dumps(rec), flush=True)
