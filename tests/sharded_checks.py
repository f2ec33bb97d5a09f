"""The sharded-state parity checks shared by both multi-rank transports:

* `tests/test_gpu_loopback.py`: G loopback ranks = threads of one process on one GPU
  (qsim_loopback_id), so a one-GPU box runs every global-qubit swap path;
* `tools/mgpu_check.py`: one process per GPU under torchrun, NCCL + CUDA IPC.

`run_checks(rank, world, new_sim, n, p)` is SPMD: every rank calls it with its own `new_sim`
(a factory returning a fresh sharded QSim handle on the transport) and makes the same calls;
rank 0 compares with the CPU oracle (full state at n <= 24; structured pins P4, P8, P9 at any
n) and returns [(name, ok, detail)] (other ranks return []).
"""
from __future__ import annotations

import numpy as np

from oracle import closed_forms as cf
from oracle import oracle as o
from paper_2104_03293_b200 import instances as inst


def run_checks(rank, world, new_sim, n, p=3, full=True, extras=True):
    out = []

    def report(name, ok, detail=""):
        out.append((f"world={world} n={n} {name}", bool(ok), detail))

    rng = np.random.default_rng(n)
    g = rng.uniform(-2, 2, p)
    b = rng.uniform(-np.pi, np.pi, p)
    small = n <= 24 and full
    # 1) dense random instance, full-state parity
    h, J = inst.random_ising(n, 40 + n)
    sim = new_sim(n)
    path = sim.swap_path
    sim.set_ising(h, J)
    sim.init_plus()
    sim.apply_qaoa(g, b)
    e = sim.expect_hc()
    nrm = sim.norm2()
    psi = sim.amplitudes() if small else None
    en = sim.energies(0, min(1 << n, 1 << 16))
    gs = [0, 5, (1 << n) - 1]
    ps = sim.success_prob(gs)
    sim.apply_qaoa(g[:1], b[:1])  # continue from the current state (second call loads)
    psi2 = sim.amplitudes() if small else None
    sim.close()
    if rank == 0:
        out.append((f"world={world} n={n} swap path", True, str(path)))
    if rank == 0 and small:
        ref = o.qaoa_state(h, J, g, b)
        er, sc = o.expect_hc(h, J, ref, with_abs=True)
        d = np.max(np.abs(psi - ref))
        report("amplitudes", d <= 1e-10 and np.linalg.norm(psi - ref) <= 1e-12, f"max|d|={d:.2e}")
        report("<H_C>", abs(e - er) <= 1e-9 * max(abs(er), sc), f"{e:.12f} vs {er:.12f}")
        report("norm", abs(nrm - 1) <= 1e-12, f"{nrm:.15f}")
        report("energies", np.array_equal(en, o.energies(h, J, 0, len(en))))
        pr = o.success_prob(ref, gs)
        report("P_success", abs(ps - pr) <= 1e-9 * pr, f"{ps:.6e} vs {pr:.6e}")
        ref2 = o.qaoa_state(h, J, np.concatenate([g, g[:1]]), np.concatenate([b, b[:1]]))
        d2 = np.max(np.abs(psi2 - ref2))
        report("continued apply", d2 <= 1e-10, f"max|d|={d2:.2e}")
    elif rank == 0:
        report("norm", abs(nrm - 1) <= 1e-12, f"{nrm:.15f}")
        report("energies", np.array_equal(en, o.energies(h, J, 0, len(en))))
    if extras and small:
        # spins (NEXT-2) and enumeration (NEXT-3) on the sharded handle
        sim = new_sim(n)
        sim.set_ising(h, J)
        sim.init_plus()
        sim.apply_qaoa(g, b)
        sz = sim.spins()
        gsl, emin, cnt = sim.ground_states(max_out=8)
        sim.close()
        if rank == 0:
            ref = o.qaoa_state(h, J, g, b)
            report("spins", np.max(np.abs(sz - o.spin_expectations(ref))) <= 1e-11)
            rgs, remin, rcnt = o.ground_states(h, J, max_out=8)
            report("ground states", emin == remin and cnt == rcnt and gsl == rgs[: len(gsl)])
        # QSDS combined stepping (NEXT-1)
        s_, A, B = inst.toy_schedule()
        sim = new_sim(n)
        sim.set_ising(h, J)
        sim.init_plus()
        sim.apply_qsds(0.35, 3, s_, A, B)
        psi_q = sim.amplitudes()
        sim.close()
        if rank == 0:
            ref = o.qsds_state(h, J, 0.35, 3, s_, A, B)
            report("QSDS amplitudes", np.max(np.abs(psi_q - ref)) <= 1e-10)
        # FP32 precision mode (NEXT-4): the DESIGN §9 bound
        from paper_2104_03293_b200 import qsim as Q

        sim = new_sim(n, precision=Q.QSIM_FP32)
        sim.set_ising(h, J)
        sim.init_plus()
        sim.apply_qaoa(g, b)
        e32 = sim.expect_hc()
        psi32 = sim.amplitudes()
        sim.close()
        if rank == 0:
            ref = o.qaoa_state(h, J, g, b)
            bound = len(g) * (2 * n + 12) * 2.0 ** -24
            d = np.linalg.norm(psi32 - ref)
            er, sc = o.expect_hc(h, J, ref, with_abs=True)
            emax = np.max(np.abs(o.energies(h, J)))
            report("FP32 amplitudes", d <= bound, f"l2={d:.2e} bound={bound:.2e}")
            report("FP32 <H_C>", abs(e32 - er) <= 2 * bound * emax + 1e-9 * sc, f"{e32:.9f} vs {er:.9f}")
    # p = 1 closed-form <H_C> (pin P4), any n
    sim = new_sim(n)
    sim.set_ising(h, J)
    sim.init_plus()
    sim.apply_qaoa(g[:1], b[:1])
    e1 = sim.expect_hc()
    en = sim.energies((1 << n) - 4096, 4096)
    sim.close()
    if rank == 0:
        r1 = cf.p1_expect_hc(h, J, g[0], b[0])
        report("p=1 closed-form <H_C>", abs(e1 - r1) <= 1e-9 * max(1.0, abs(r1)), f"{e1:.12f} vs {r1:.12f}")
        report("energies (top)", np.array_equal(en, o.energies(h, J, (1 << n) - 4096, 4096)))
    # cluster instance mixing low, tile, top-local and global bits (pin P9)
    clusters = inst.spread_clusters(n, 5, seed=n)
    h, J = inst.cluster_ising(n, clusters, seed=n)
    sim = new_sim(n)
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
        report("cluster amplitudes", d <= 1e-10, f"max|d|={d:.2e}")
        report("cluster <H_C>", abs(e - comp.expect) <= 1e-9 * max(1.0, abs(comp.expect)))
    # product instance J = 0 (pin P8): every amplitude factorises over the qubits
    h, J = inst.product_ising(n, seed=n)
    sim = new_sim(n)
    sim.set_ising(h, J)
    sim.init_plus()
    sim.apply_qaoa(g, b)
    amp = np.array([sim.amplitudes(int(z), 1)[0] for z in zs])
    sim.close()
    if rank == 0:
        d = np.max(np.abs(amp - cf.product_amplitudes(h, g, b, zs)))
        report("product amplitudes", d <= 1e-12, f"max|d|={d:.2e}")
    return out if rank == 0 else []
