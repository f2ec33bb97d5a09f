"""Single-process multi-GPU run for ncu's NVLink counters (ncu cannot follow a multi-process NCCL
job): `world` loopback ranks as threads, one GPU each (peer access enabled by the library), on the
fused split swap path (out of place: the moving passes store their peer-bound tiles straight into
the peer's second buffer over NVLink).  Kernels of the two ranks need not overlap on this path, so
ncu's kernel serialisation is harmless.

    python tools/nvlink_ncu.py --n 31 --p 2
    ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        -k regex:tma_pass --csv python tools/nvlink_ncu.py --n 31 --p 2
"""
import argparse
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=31)
ap.add_argument("--p", type=int, default=2)
ap.add_argument("--world", type=int, default=2)
a = ap.parse_args()

from paper_2104_03293_b200 import instances as inst  # noqa: E402
from paper_2104_03293_b200 import qsim as Q  # noqa: E402

h, J = inst.random_ising(a.n, 5)
rng = np.random.default_rng(1)
g, b = rng.uniform(-1, 1, a.p), rng.uniform(-1, 1, a.p)
uid = Q.qsim_loopback_id(a.world)
out, errs = [None] * a.world, []


def rank(r):
    try:
        torch.cuda.set_device(r)
        with Q.QSim(a.n, rank=r, world=a.world, nccl_unique_id=uid) as s:
            s.set_ising(h, J)
            s.init_plus()
            s.apply_qaoa(g, b)
            out[r] = (s.expect_hc(), s.norm2(), s.swap_path)
    except BaseException as e:  # noqa: BLE001
        errs.append(repr(e))


th = [threading.Thread(target=rank, args=(r,)) for r in range(a.world)]
[t.start() for t in th]
[t.join() for t in th]
print("nvlink_ncu", "errors" if errs else "ok", errs or out[0], flush=True)
sys.exit(1 if errs or abs(out[0][1] - 1.0) > 1e-10 else 0)
