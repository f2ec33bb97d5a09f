"""Build libqsim.so (sm_100a) in-tree with nvcc.  No JIT cache: the .so sits next to
this file so it travels with the repo snapshot to the GPU box."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libqsim.so")
SOURCES = [os.path.join(CSRC, f) for f in ("qsim_device.cu", "qsim_tma.cu", "qsim_extra.cu", "qsim_comm.cu", "qsim_engine.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("qsim_device.h", "qsim_kernels.cuh", "qsim_comm.h")] + [
    os.path.join(ROOT, "include", "qsim.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dir() -> str:
    """Use the NCCL that torch itself loads (same SONAME libnccl.so.2), so the two never
    mix in one process whichever is imported first."""
    import importlib.util

    spec = importlib.util.find_spec("nvidia.nccl")
    if spec and spec.submodule_search_locations:
        d = list(spec.submodule_search_locations)[0]
        if os.path.exists(os.path.join(d, "lib", "libnccl.so.2")):
            return d
    return ""


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    nd = _nccl_dir()
    nccl = (["-I", os.path.join(nd, "include"), "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2",
             "-Xlinker", "-rpath=" + os.path.join(nd, "lib")] if nd else ["-lnccl"])
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "-I", os.path.join(ROOT, "include"), *nccl[:2], "-o", LIB, *SOURCES, *nccl[2:]]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
    print(LIB)
