"""Multi-GPU parity check over NCCL (SPMD, one process per GPU):

    python -m torch.distributed.run --nproc-per-node G --master-addr 127.0.0.1 tools/mgpu_check.py --qubits 20

Every rank drives one shard through tests/sharded_checks.run_checks (the same checks the
one-GPU loopback tests run); rank 0 compares with the CPU oracle and prints [PASS]/[FAIL].
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--qubits", type=int, nargs="+", default=[18, 20])
ap.add_argument("--p", type=int, default=3)
a = ap.parse_args()

world = int(os.environ["WORLD_SIZE"])
rank = int(os.environ["RANK"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))

from paper_2104_03293_b200 import qsim as Q  # noqa: E402
from tests.sharded_checks import run_checks  # noqa: E402


def new_sim(n, precision=Q.QSIM_FP64):
    """an ncclUniqueId is single-use: one fresh id per handle, broadcast from rank 0"""
    obj = [Q.qsim_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return Q.QSim(n, rank=rank, world=world, nccl_unique_id=obj[0], precision=precision)


fails = 0
for n in a.qubits:
    for name, ok, detail in run_checks(rank, world, new_sim, n, p=a.p, full=n <= 24, extras=n <= 24):
        print(f"[{'PASS' if ok else 'FAIL'}] {name} {detail}", flush=True)
        fails += 0 if ok else 1
dist.barrier()
dist.destroy_process_group()
sys.exit(1 if fails else 0)
