"""The debug build (libqsim_debug.so: the same sources with -DQSIM_DEBUG) arms device-side bound
checks on every tile id, tile base, swapped-store address, tensor-map destination and handshake
slot, and on the stage-issue invariant of the TMA ring (a stage is never refilled before its tile
was consumed); a failed check traps.  compute-sanitizer is closed on this GPU pool (runs under it
left GPUs needing a reset), so this and tests/test_gpu_determinism.py are the race / bounds
evidence: tools/debug_case.py runs every pass program and swap path at small n under the checks
and compares with the oracle."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_debug_build_bound_checks():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2104_03293_b200 import build

    lib = build.build(debug=True)
    env = dict(os.environ, QSIM_LIBRARY=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "debug_case.py")], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "debug_case OK" in out, out[-4000:]
