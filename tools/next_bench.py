"""Measurements of the SURVEY §8(f) NEXT rows on one B200 (JSON lines):
  NEXT-1 QSDS combined step: ms per step operator at n qubits (eq. AQA4), vs the split form
  NEXT-2 <sigma^z_i>: ms per read-only sweep
  NEXT-3 full enumeration: see tools/tfe_bench.py
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2104_03293_b200 import instances as inst  # noqa: E402
from paper_2104_03293_b200 import problems as pp  # noqa: E402
from paper_2104_03293_b200 import qsim as Q  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--qubits", type=int, default=30)
ap.add_argument("--steps", type=int, default=16)
a = ap.parse_args()
torch.cuda.set_device(0)
n = a.qubits
ec, x_star = inst.exact_cover(n, seed=0)
h, J, C = pp.ising_from_exact_cover(ec)
r = pp.rescale_r(h, J)
s_, A, B = inst.dw_like_schedule()
A, B = 2 * np.pi * A, 2 * np.pi * B / r
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
sim = Q.QSim(n, cuda_stream=st.cuda_stream)
sim.set_ising(h, J)
z_star = int(sum(int(x_star[i]) << i for i in range(n)))


def timed(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def qsds():
    sim.init_plus()
    sim.apply_qsds(0.4, a.steps - 1, s_, A, B)


def aqa():
    sim.init_plus()
    sim.apply_aqa(0.4 * a.steps, a.steps, s_, A, B)


ms_q = timed(qsds)
ps_q = sim.success_prob([z_star])
ms_a = timed(aqa)
ps_a = sim.success_prob([z_star])
ms_s = timed(lambda: sim.spins(), reps=3)


def hadamard():
    sim.init_plus()
    sim.apply_hadamard(11)


ms_h = timed(hadamard, reps=2)
amp0 = sim.amplitudes(0, 1)[0]
print(json.dumps({"row": "NEXT-1 QSDS combined step", "n": n, "step_operators": a.steps,
                  "ms_total": ms_q, "ms_per_step": ms_q / a.steps, "p_success": ps_q,
                  "split_form_ms_per_layer": ms_a / a.steps, "split_form_p_success": ps_a}))
print(json.dumps({"row": "NEXT-2 <sigma^z_i> sweep", "n": n, "ms": ms_s,
                  "GB_per_s": 16 * 2.0 ** n / (ms_s / 1e3) / 1e9}))
gates = 11 * n
print(json.dumps({"row": "NEXT-4 Hadamard (H^N)^11 (P:177)", "n": n, "ms": ms_h, "gates": gates,
                  "gate_amplitude_updates_per_s": gates * 2.0 ** n / (ms_h / 1e3),
                  "normalized_time_s_to_32_gates": 352.0 / gates * ms_h / 1e3,
                  "amp0_of_final_state": [amp0.real, amp0.imag],
                  "paper_context": "JUQCS-G A100 compute-only ~5.5e10 gate-amplitude updates/s per GPU "
                                   "(derived from P:197, P:177; precision not stated, likely FP32)"}))
sim.close()
