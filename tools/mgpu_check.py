"""Multi-GPU parity check (SPMD, one process per GPU):

    python -m torch.distributed.run --nproc-per-node G --master-addr 127.0.0.1 tools/mgpu_check.py --qubits 20

Every rank drives one shard; rank 0 compares the gathered state, <H_C>, P_success and E(z)
against the CPU oracle (full state for n <= 24, structured pins above).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
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

from oracle import closed_forms as cf  # noqa: E402
from oracle import oracle as o  # noqa: E402
from paper_2104_03293_b200 import instances as inst  # noqa: E402
from paper_2104_03293_b200 import qsim as Q  # noqa: E402

def new_uid():
    """an ncclUniqueId is single-use: one fresh id per handle, broadcast from rank 0"""
    obj = [Q.qsim_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


fails = 0


def report(name, ok, detail=""):
    global fails
    if rank == 0:
        print(f"[{'PASS' if ok else 'FAIL'}] world={world} {name} {detail}", flush=True)
    fails += 0 if ok else 1


for n in a.qubits:
    rng = np.random.default_rng(n)
    g = rng.uniform(-2, 2, a.p)
    b = rng.uniform(-np.pi, np.pi, a.p)
    # 1) dense random instance, full-state parity
    h, J = inst.random_ising(n, 40 + n)
    sim = Q.QSim(n, rank=rank, world=world, nccl_unique_id=new_uid())
    sim.set_ising(h, J)
    sim.init_plus()
    sim.apply_qaoa(g, b)
    e = sim.expect_hc()
    nrm = sim.norm2()
    psi = sim.amplitudes() if n <= 24 else None
    en = sim.energies(0, min(1 << n, 1 << 16))
    gs = [0, 5, (1 << n) - 1]
    ps = sim.success_prob(gs)
    sim.apply_qaoa(g[:1], b[:1])  # continue from the current state (second call loads)
    psi2 = sim.amplitudes() if n <= 24 else None
    sim.close()
    if rank == 0 and n <= 24:
        ref = o.qaoa_state(h, J, g, b)
        er, sc = o.expect_hc(h, J, ref, with_abs=True)
        d = np.max(np.abs(psi - ref))
        report(f"n={n} amplitudes", d <= 1e-10 and np.linalg.norm(psi - ref) <= 1e-12, f"max|d|={d:.2e}")
        report(f"n={n} <H_C>", abs(e - er) <= 1e-9 * max(abs(er), sc), f"{e:.12f} vs {er:.12f}")
        report(f"n={n} norm", abs(nrm - 1) <= 1e-12, f"{nrm:.15f}")
        report(f"n={n} energies", np.array_equal(en, o.energies(h, J, 0, len(en))))
        pr = o.success_prob(ref, gs)
        report(f"n={n} P_success", abs(ps - pr) <= 1e-9 * pr, f"{ps:.6e} vs {pr:.6e}")
        ref2 = o.qaoa_state(h, J, np.concatenate([g, g[:1]]), np.concatenate([b, b[:1]]))
        d2 = np.max(np.abs(psi2 - ref2))
        report(f"n={n} continued apply", d2 <= 1e-10, f"max|d|={d2:.2e}")
    # 1a) spins (NEXT-2) and enumeration (NEXT-3) on the sharded handle
    sim = Q.QSim(n, rank=rank, world=world, nccl_unique_id=new_uid())
    sim.set_ising(h, J)
    sim.init_plus()
    sim.apply_qaoa(g, b)
    sz = sim.spins()
    gs, emin, cnt = sim.ground_states(max_out=8)
    sim.close()
    if rank == 0 and n <= 24:
        ref = o.qaoa_state(h, J, g, b)
        report(f"n={n} spins", np.max(np.abs(sz - o.spin_expectations(ref))) <= 1e-11)
        rgs, remin, rcnt = o.ground_states(h, J, max_out=8)
        report(f"n={n} ground states", emin == remin and cnt == rcnt and gs == rgs[: len(gs)])
    # 1c) QSDS combined stepping (NEXT-1) on the sharded handle
    s_, A, B = inst.toy_schedule()
    sim = Q.QSim(n, rank=rank, world=world, nccl_unique_id=new_uid())
    sim.set_ising(h, J)
    sim.init_plus()
    sim.apply_qsds(0.35, 3, s_, A, B)
    psi_q = sim.amplitudes() if n <= 24 else None
    sim.close()
    if rank == 0 and n <= 24:
        ref = o.qsds_state(h, J, 0.35, 3, s_, A, B)
        report(f"n={n} QSDS amplitudes", np.max(np.abs(psi_q - ref)) <= 1e-10)
    # 1d) FP32 precision mode (NEXT-4) on the sharded handle: the DESIGN §9 bound
    sim = Q.QSim(n, rank=rank, world=world, nccl_unique_id=new_uid(), precision=Q.QSIM_FP32)
    sim.set_ising(h, J)
    sim.init_plus()
    sim.apply_qaoa(g, b)
    e32 = sim.expect_hc()
    psi32 = sim.amplitudes() if n <= 24 else None
    sim.close()
    if rank == 0 and n <= 24:
        ref = o.qaoa_state(h, J, g, b)
        bound = len(g) * (2 * n + 12) * 2.0 ** -24
        d = np.linalg.norm(psi32 - ref)
        er, sc = o.expect_hc(h, J, ref, with_abs=True)
        emax = np.max(np.abs(o.energies(h, J)))
        report(f"n={n} FP32 amplitudes", d <= bound, f"l2={d:.2e} bound={bound:.2e}")
        report(f"n={n} FP32 <H_C>", abs(e32 - er) <= 2 * bound * emax + 1e-9 * sc, f"{e32:.9f} vs {er:.9f}")
    # 1b) p = 1 closed-form <H_C> (pin P4), any n
    sim = Q.QSim(n, rank=rank, world=world, nccl_unique_id=new_uid())
    sim.set_ising(h, J)
    sim.init_plus()
    sim.apply_qaoa(g[:1], b[:1])
    e1 = sim.expect_hc()
    en = sim.energies((1 << n) - 4096, 4096)
    sim.close()
    if rank == 0:
        r1 = cf.p1_expect_hc(h, J, g[0], b[0])
        report(f"n={n} p=1 closed-form <H_C>", abs(e1 - r1) <= 1e-9 * max(1.0, abs(r1)), f"{e1:.12f} vs {r1:.12f}")
        report(f"n={n} energies (top)", np.array_equal(en, o.energies(h, J, (1 << n) - 4096, 4096)))
    # 2) cluster instance mixing low, tile, top-local and global bits (pin P9)
    clusters = inst.spread_clusters(n, 5, seed=n)
    h, J = inst.cluster_ising(n, clusters, seed=n)
    sim = Q.QSim(n, rank=rank, world=world, nccl_unique_id=new_uid())
    sim.set_ising(h, J)
    sim.init_plus()
    sim.apply_qaoa(g, b)
    e = sim.expect_hc()
    zs = inst.sample_indices(n, 32, seed=1)
    amp = np.array([sim.amplitudes(int(z), 1)[0] for z in zs])
    sim.close()
    if rank == 0:
        comp = cf.ClusterComposition(h, J, clusters, g, b)
        d = np.max(np.abs(amp - comp.amplitudes(zs)))
        report(f"n={n} cluster amplitudes", d <= 1e-10, f"max|d|={d:.2e}")
        report(f"n={n} cluster <H_C>", abs(e - comp.expect) <= 1e-9 * max(1.0, abs(comp.expect)))

dist.barrier()
dist.destroy_process_group()
sys.exit(1 if fails else 0)
