"""Multi-GPU parity inside the pytest suite, on boxes with 2 or more GPUs (skipped
below that; the one-GPU loopback tests cover the same swap paths on one device):

* NCCL, one process per GPU: `tools/mgpu_check.py` under torchrun on 2 and (when present) 4 GPUs,
  on the default fused split path and on the fused in-place path (QSIM_SWAP_INPLACE=1); rank 0
  compares the gathered sharded state, <H_C>, P_success and E(z) with the CPU oracle (full state
  at n <= 24, structured pins P4/P8/P9 above) and exits non-zero on any FAIL;
* loopback across devices: the ranks as threads of this process, one GPU each (peer access),
  through the same checks (tests/sharded_checks.py)."""
import os
import subprocess
import sys
import threading

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    import torch

    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("world,qubits,inplace", [(2, ["18", "24"], 0), (2, ["20", "24"], 1), (4, ["20", "24"], 0),
                                                  (4, ["21", "24"], 1)])
def test_sharded_parity_torchrun(world, qubits, inplace):
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    from paper_2104_03293_b200 import build

    build.build()
    env = dict(os.environ)
    if inplace:
        env["QSIM_SWAP_INPLACE"] = "1"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", f"--master-port={29610 + world + 10 * inplace}",
           os.path.join(ROOT, "tools", "mgpu_check.py"), "--qubits", *qubits, "--p", "3"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "[PASS]" in out and "[FAIL]" not in out, out[-4000:]
    assert f"swap path {6 if inplace else 1}" in out, out[-4000:]


@pytest.mark.parametrize("world,n,inplace", [(2, 22, 0), (2, 23, 1)])
def test_loopback_across_devices(world, n, inplace, monkeypatch):
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    import torch

    from paper_2104_03293_b200 import qsim as Q
    from tests.sharded_checks import run_checks

    if inplace:
        monkeypatch.setenv("QSIM_SWAP_INPLACE", "1")
    ids = [Q.qsim_loopback_id(world) for _ in range(8)]
    res, errs = [None] * world, []

    def worker(rank):
        try:
            torch.cuda.set_device(rank)
            k = [0]

            def new_sim(nq, precision=Q.QSIM_FP64):
                k[0] += 1
                return Q.QSim(nq, rank=rank, world=world, nccl_unique_id=ids[k[0] - 1], precision=precision)

            res[rank] = run_checks(rank, world, new_sim, n, p=3, full=True, extras=False)
        except BaseException as e:  # noqa: BLE001
            errs.append(repr(e))

    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(world)]
    [t.start() for t in th]
    [t.join(900) for t in th]
    assert not errs, errs
    bad = [x for x in res[0] if not x[1]]
    assert not bad, bad
    assert any(x[0].endswith("swap path") and x[2] == str(6 if inplace else 1) for x in res[0])
