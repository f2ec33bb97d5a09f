"""Per-pass timing of the multi-GPU layer (fused / split global-qubit swap).

    python -m torch.distributed.run --nproc-per-node G --master-addr 127.0.0.1 tools/mgpu_prof.py --nlocal 30

Runs one AQA evaluation (exact-cover instance, n = local + log2 G) with per-pass CUDA events and
prints, per rank, the median duration of each pass position within a layer.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nlocal", type=int, default=30)
ap.add_argument("--p", type=int, default=8)
ap.add_argument("--tag", default="")
a = ap.parse_args()

world = int(os.environ["WORLD_SIZE"])
rank = int(os.environ["RANK"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))

from paper_2104_03293_b200 import instances as inst  # noqa: E402
from paper_2104_03293_b200 import problems as pp  # noqa: E402
from paper_2104_03293_b200 import qsim as Q  # noqa: E402

g = world.bit_length() - 1
n = a.nlocal + g
obj = [Q.qsim_nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
ec, xs = inst.exact_cover(n, seed=0)
h, J, C = pp.ising_from_exact_cover(ec)
r = pp.rescale_r(h, J)
s, A, B = inst.dw_like_schedule()
stream = torch.cuda.Stream()
sim = Q.QSim(n, rank=rank, world=world, nccl_unique_id=obj[0], cuda_stream=stream.cuda_stream)
sim.set_ising(h, J)
for it in range(2):
    sim.init_plus()
    Q.qsim_profile_enable(sim.h, True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    sim.apply_aqa(0.02 * a.p, a.p, s, 2 * np.pi * A, 2 * np.pi * B / r)
    e1.record(stream)
    ms = Q.qsim_profile_passes(sim.h)
    Q.qsim_profile_enable(sim.h, False)
    e = sim.expect_hc()
    apply_ms = e0.elapsed_time(e1)
per_layer = (len(ms) - 1) // a.p
body = ms[: per_layer * a.p].reshape(a.p, per_layer)
med = np.median(body[1:], axis=0)  # skip the init layer
rec = {"tag": a.tag, "rank": rank, "world": world, "n": n, "p": a.p, "passes": len(ms),
       "per_layer_positions_ms": [round(float(x), 3) for x in med], "layer_ms_sum": round(float(med.sum()), 3),
       "trailing_ms": round(float(ms[-1]), 3), "total_ms": round(float(ms.sum()), 2),
       "apply_ms": round(apply_ms, 2), "ms_per_layer": round(apply_ms / a.p, 3), "swap_path": sim.swap_path,
       "inplace_env": os.environ.get("QSIM_SWAP_INPLACE", "0"), "weights": os.environ.get("QSIM_SPLIT_W", "default"),
       "expect_hc": e}
allrec = [None] * world
dist.all_gather_object(allrec, rec)
if rank == 0:
    for x in allrec:
        print(json.dumps(x), flush=True)
sim.close()
dist.destroy_process_group()
