"""World-size-2 CPU tests (gloo) of the N > 1 host path: the ncclUniqueId bootstrap that
bench.py and tools/mgpu_check.py use, rank-consistent planning, and the reference arm under
torchrun (rank 0 prints one JSON line, rank 1 exits 0 without work)."""
import json
import os
import subprocess
import sys

import pytest
import torch.multiprocessing as mp

from tests.conftest import ROOT


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist

    from paper_2104_03293_b200 import build

    build.build()
    from paper_2104_03293_b200 import qsim as Q

    dist.init_process_group("gloo", rank=rank, world_size=world)
    obj = [Q.qsim_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    uid = obj[0]
    # every rank plans the same schedule for the same (n, world, p)
    plan = [Q.qsim_plan_counts(33, 8, 5), Q.qsim_plan_positions(33, 8, 1)]
    plans = [None] * world
    dist.all_gather_object(plans, plan)
    uids = [None] * world
    dist.all_gather_object(uids, uid)
    dist.destroy_process_group()
    q.put((rank, len(uid), uids[0] == uids[1], plans[0] == plans[1], plan[0]))


def test_gloo_world2_bootstrap_and_plan():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 200
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ln, same_uid, same_plan, counts in res:
        assert ln == 128 and same_uid and same_plan
        assert counts[1] == 5  # one swap per layer
        assert counts[2] * 8 == 7 * (1 << 30)  # (G-1)/G of the 2^30-amplitude shard per swap


def test_reference_arm_under_torchrun_world2():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(29800 + os.getpid() % 100), "bench.py",
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0"]
    env = dict(os.environ, OMP_NUM_THREADS="4")
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0
