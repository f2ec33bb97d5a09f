#!/usr/bin/env python
"""Benchmark of the QAOA/AQA hot path (BASELINE.json metric: seconds per QAOA/AQA layer and
amplitude-updates/s at n qubits, % HBM roofline, on 1/2/4/8 B200).

One "step" = one full AQA evaluation: |+>^n, p layers of e^{-i gamma_k H_C} then
e^{-i beta_k H_D} (eq:QAOA_state, angles eq:beta_k / eq:gamma_k), <H_C> and P_success.
Workload (weak scaling): n = 30 + log2(N) qubits on N GPUs (2^30 amplitudes = 17.2 GB per
GPU), exact-cover-shaped instance (N x 472, seed 0, paper's 30(0)-like, r ~ 37), synthetic
DW-like schedule, tau = 0.4 ns, p = 32 (BASELINE configs[2] at N=1, configs[3] at N=8).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--p P]

Under torchrun (N > 1) every rank drives its GPU; rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sec per QAOA/AQA layer & amplitude-updates/s at n qubits, % HBM roofline, 1/2/4/8 B200"
UNIT = "layer-amplitude-updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--p", type=int, default=32)
    ap.add_argument("--nlocal", type=int, default=30, help="qubits per GPU shard (n = nlocal + log2 N)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--precision", default="fp64", choices=["fp64", "fp32"],
                    help="amplitude precision (fp64 = the north-star path; fp32 = the NEXT-4 mode)")
    return ap.parse_args()


def workload(n: int, p: int):
    from paper_2104_03293_b200 import instances as inst
    from paper_2104_03293_b200 import problems as pp

    a, x_star = inst.exact_cover(n, seed=0)
    h, J, C = pp.ising_from_exact_cover(a)
    r = pp.rescale_r(h, J)
    s, A, B = inst.dw_like_schedule()
    tau = 0.4  # ns
    # angular units: 2 pi GHz; the rescale 1/r is folded into B (gamma/r, reading R6)
    A_ang = 2 * np.pi * A
    B_ang = 2 * np.pi * B / r
    T = tau * p
    z_star = int(sum(int(x_star[i]) << i for i in range(n)))
    return dict(h=h, J=J, C=C, r=r, s=s, A=A_ang, B=B_ang, T=T, z_star=z_star)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for k, nm in enumerate(names):
                if r[5 + k].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows)}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy R+W)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def cpu_baseline(nlocal_sample: int = 26, p_sample: int = 2):
    """The oracle as it stands, on a bounded sample of the same workload (same generator and
    schedule, n = nlocal_sample, p_sample layers), timed on the host cores."""
    from oracle import oracle as o

    w = workload(nlocal_sample, p_sample)
    o.lib()
    t0 = time.perf_counter()
    psi = o.aqa_state(w["h"], w["J"], w["T"], p_sample, w["s"], w["A"], w["B"])
    e = o.expect_hc(w["h"], w["J"], psi)
    ps = o.success_prob(psi, [w["z_star"]])
    dt = time.perf_counter() - t0
    value = (1 << nlocal_sample) * p_sample / dt
    return {"value": value, "unit": UNIT, "cores": o.num_threads(), "kind": "oracle",
            "sample": f"oracle.aqa_state + expect_hc + success_prob at n={nlocal_sample}, p={p_sample} "
                      f"(same generator/schedule), {dt:.2f} s", "seconds": dt, "expect_hc": e, "p_success": ps}


def run_reference(args):
    """--impl reference: the CPU oracle as it stands, each step a bounded sample."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle as o

    n_s, p_s = 24, 2
    w = workload(n_s, p_s)
    o.lib()
    for _ in range(args.warmup):
        psi = o.aqa_state(w["h"], w["J"], w["T"], p_s, w["s"], w["A"], w["B"])
    t0 = time.perf_counter()
    for _ in range(args.steps):
        psi = o.aqa_state(w["h"], w["J"], w["T"], p_s, w["s"], w["A"], w["B"])
        o.expect_hc(w["h"], w["J"], psi)
        o.success_prob(psi, [w["z_star"]])
    dt = (time.perf_counter() - t0) / args.steps
    value = (1 << n_s) * p_s / dt
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"AQA exact-cover-shaped, bounded CPU sample n={n_s} p={p_s} of the "
                                   f"n={args.nlocal}+log2(N) p={args.p} workload", "n": n_s, "p": p_s},
            "cpu_baseline": {"value": value, "unit": UNIT, "kind": "oracle", "cores": o.num_threads(),
                             "sample": f"n={n_s}, p={p_s} per step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    from paper_2104_03293_b200 import qsim as Q

    g = int(math.log2(world))
    assert 1 << g == world
    n = args.nlocal + g
    p = args.p
    w = workload(n, p)
    uid = None
    if world > 1:
        obj = [Q.qsim_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    # a dedicated stream: the library enqueues every kernel on it and the timing events are
    # recorded on it (torch's default stream is the legacy null stream, handle 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    f32 = args.precision == "fp32"
    es = 8 if f32 else 16
    sim = Q.QSim(n, rank=rank, world=world, nccl_unique_id=uid, cuda_stream=stream.cuda_stream,
                 precision=Q.QSIM_FP32 if f32 else Q.QSIM_FP64)
    sim.set_ising(w["h"], w["J"])

    def step():
        sim.init_plus()
        sim.apply_aqa(w["T"], p, w["s"], w["A"], w["B"])
        e = sim.expect_hc()
        ps = sim.success_prob([w["z_star"]])
        return e, ps

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        step()
    barrier()
    clk = ClockSampler(local)
    clk.start()
    launches0 = sim.launches
    Q.qsim_profile_enable(sim.h, True)
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        e, ps = step()
    ev1.record(stream)
    barrier()
    ms = ev0.elapsed_time(ev1)
    pass_ms, pass_cnt, pass_bytes = Q.qsim_profile_read(sim.h)
    Q.qsim_profile_enable(sim.h, False)
    launches = sim.launches - launches0
    clocks = clk.stop()
    t = torch.tensor([ms, pass_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, pass_ms_max = float(t[0]), float(t[1])
    ms_step = ms_max / args.steps
    value = (1 << n) * p / (ms_step / 1e3)

    # end to end through the public API with host buffers: H2D of (h, J, schedule) and D2H of
    # (<H_C>, P_success) inside the timed region, every step
    h_host = np.ascontiguousarray(w["h"])
    J_host = np.ascontiguousarray(w["J"])
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        sim.set_ising(h_host, J_host)
        step()
    barrier()
    e2e_s = (time.perf_counter() - t0) / args.steps
    if world > 1:
        tt = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt[0])
    h2d = h_host.nbytes + J_host.nbytes + 3 * w["s"].nbytes + 8
    d2h = 16 + 16

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline()
    if rank == 0:
        peak, peak_src = peaks()
        avg_pass_ms = pass_ms_max / max(pass_cnt, 1)
        avg_bytes = pass_bytes / max(pass_cnt, 1)
        achieved = avg_bytes / (avg_pass_ms / 1e3) / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "pass_kernel_traffic.json")
        if os.path.exists(tp) and not f32 and world == 1:
            try:
                traffic = json.load(open(tp)).get("dram_bytes_per_launch")
            except Exception:
                traffic = None
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32" if f32 else "f64", "data": "synthetic",
            "config": {"workload": f"AQA exact-cover-shaped n={n} (N x 472, seed 0), p={p}, tau=0.4 ns, "
                                   f"DW-like schedule; step = |+> + {p} layers + <H_C> + P_success",
                       "n": n, "p": p, "n_local": args.nlocal, "parallelism": f"state sharded over {world} GPU"
                       + ("s (global-qubit swaps)" if world > 1 else ""),
                       "precision": args.precision,
                       "l2": f"state {es * (1 << args.nlocal) / 1e9:.1f} GB per GPU >> 126 MB L2 (no flush needed)"},
            "sec_per_layer": ms_step / 1e3 / p,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "kernel": "qk::tma_pass_kernel", "avg_launch_ms": avg_pass_ms,
                         "launches": pass_cnt, "alg_bytes_per_launch": avg_bytes,
                         "pass_share_of_step": pass_ms_max / ms_max},
            "cpu_baseline": ({k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")} if cpu else None),
            "e2e": {"value": (1 << n) * p / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "sec_per_step": e2e_s},
            "gpu_launches": int(launches),
            "nvlink": ({"swap_bytes_per_layer_per_dir": (world - 1) / world * es * (1 << args.nlocal),
                        "layer_ms": ms_step / p,
                        "implied_GBps_per_dir": (world - 1) / world * es * (1 << args.nlocal) / (ms_step / p / 1e3) / 1e9,
                        "peak_GBps_per_dir": 770.0,
                        "peak_source": "B200_PROFILING.md measured peer copy (nominal 900)",
                        "note": "one global-qubit swap per layer, its stores spread over the layer's passes "
                                "(split swap); implied rate = swap bytes / whole layer time"}
                       if world > 1 else None),
            "clocks": clocks,
            "results": {"expect_hc": e, "p_success": ps, "r": w["r"]},
        }
        print(json.dumps(line), flush=True)
    sim.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
