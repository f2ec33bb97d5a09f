"""Multi-GPU parity inside the pytest suite: runs `tools/mgpu_check.py` under
torchrun (one process per GPU, NCCL) on 2 and, when present, 4 GPUs of this box.  Rank 0
compares the gathered sharded state, <H_C>, P_success and E(z) with the CPU oracle (full state
at n <= 24, structured pins P4/P8/P9 above) and exits non-zero on any FAIL.  Skipped when
fewer than 2 GPUs are visible (the round-end `pytest -m gpu` box may have one)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    import torch

    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("world,qubits", [(2, ["18", "24"]), (4, ["20", "24"])])
def test_sharded_parity_torchrun(world, qubits):
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    from paper_2104_03293_b200 import build

    build.build()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", f"--master-port={29610 + world}",
           os.path.join(ROOT, "tools", "mgpu_check.py"), "--qubits", *qubits, "--p", "3"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "[PASS]" in out and "[FAIL]" not in out, out[-4000:]
