"""Workload for the debug build (tests/test_gpu_debug_build.py; run with
QSIM_LIBRARY=paper_2104_03293_b200/libqsim_debug.so): every pass program and swap path at small
n, with the device-side bound checks armed (a failed check traps: cudaErrorAssert -> ECUDA).
Checks the results against the CPU oracle and prints "debug_case OK"."""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import oracle as o  # noqa: E402
from paper_2104_03293_b200 import instances as inst  # noqa: E402
from paper_2104_03293_b200 import qsim as Q  # noqa: E402

assert Q.LIB_PATH.endswith("libqsim_debug.so"), Q.LIB_PATH
bad = []
g, b = np.array([0.4, -0.7, 0.2]), np.array([0.9, 1.3, -0.4])  # beta = 1.3: the flip form
for n in (13, 17, 21, 24):
    h, J = inst.random_ising(n, n)
    with Q.QSim(n) as s:
        s.set_ising(h, J)
        s.init_plus()
        s.apply_qaoa(g, b)
        e = s.expect_hc()
        psi = s.amplitudes()
        en = s.energies(0, min(1 << n, 1 << 14))
        sa, A, B = inst.toy_schedule()
        s.init_plus()
        s.apply_qsds(0.3, 2, sa, A, B)
        s.apply_hadamard(1)
        s.spins()
        s.ground_states(4)
    ref = o.qaoa_state(h, J, g, b)
    if np.max(np.abs(psi - ref)) > 1e-10:
        bad.append(f"n={n} amplitudes")
    if not np.array_equal(en, o.energies(h, J, 0, len(en))):
        bad.append(f"n={n} energies")


def sharded(n, world, env):
    for k, v in env.items():
        os.environ[k] = v
    h, J = inst.random_ising(n, 99 + n)
    uid = Q.qsim_loopback_id(world)
    out, errs = [None] * world, []

    def rank(r):
        try:
            with Q.QSim(n, rank=r, world=world, nccl_unique_id=uid) as s:
                s.set_ising(h, J)
                s.init_plus()
                s.apply_qaoa(g, b)
                out[r] = (s.amplitudes(), s.swap_path)
        except BaseException as ex:  # noqa: BLE001
            errs.append(repr(ex))

    th = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
    [t.start() for t in th]
    [t.join() for t in th]
    for k in env:
        del os.environ[k]
    if errs:
        bad.append(f"sharded n={n} G={world} {env}: {errs}")
    elif np.max(np.abs(out[0][0] - o.qaoa_state(h, J, g, b))) > 1e-10:
        bad.append(f"sharded n={n} G={world} {env}: amplitudes")


sharded(20, 2, {})
sharded(21, 4, {})
sharded(20, 2, {"QSIM_SWAP_INPLACE": "1"})
sharded(22, 4, {"QSIM_SWAP_INPLACE": "1"})
sharded(20, 8, {"QSIM_SWAP_INPLACE": "1"})
sharded(23, 2, {"QSIM_LOWSWAP": "1"})
sharded(20, 2, {"QSIM_FUSED_SWAP": "0"})
print("debug_case", "OK" if not bad else f"FAIL {bad}", flush=True)
sys.exit(1 if bad else 0)
