"""Build libqsim.so (sm_100a) in-tree with nvcc.  No JIT cache: the .so sits next to this file
so it travels with the repo snapshot to the GPU box.

The translation units compile in parallel (one nvcc per .cu; device code never crosses a unit,
so no relocatable device code is needed) and link into one shared library.  `build(debug=True)`
makes libqsim_debug.so: the same sources with -DQSIM_DEBUG, whose device-side bound checks
(`QSIM_DCHECK` in qsim_kernels.cuh) trap on an out-of-range tile, store address, tensor-map
coordinate or handshake slot -- the race / bounds evidence on this pool, where compute-sanitizer
is closed (tests/test_gpu_debug_build.py)."""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libqsim.so")
LIB_DEBUG = os.path.join(HERE, "libqsim_debug.so")
SOURCES = [os.path.join(CSRC, f) for f in ("qsim_tma_f32.cu", "qsim_tma_f64mv.cu", "qsim_tma_f64.cu", "qsim_tma_pw.cu",
                                            "qsim_tma.cu", "qsim_device.cu", "qsim_extra.cu", "qsim_comm.cu",
                                            "qsim_engine.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("qsim_device.h", "qsim_kernels.cuh", "qsim_comm.h",
                                                  "qsim_tma_impl.cuh")] + [
    os.path.join(ROOT, "include", "qsim.h"), os.path.abspath(__file__)]
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


def _stale(lib: str) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False, debug: bool = False) -> str:
    lib = LIB_DEBUG if debug else LIB
    if not force and not _stale(lib):
        return lib
    nd = _nccl_dir()
    inc = ["-I", os.path.join(ROOT, "include")] + (["-I", os.path.join(nd, "include")] if nd else [])
    link = (["-L", os.path.join(nd, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(nd, "lib")]
            if nd else ["-lnccl"])
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC"] + (["-DQSIM_DEBUG"] if debug else [])
    if verbose:
        flags.append("-Xptxas=-v")
    objdir = os.path.join(HERE, "build", "debug" if debug else "release")
    os.makedirs(objdir, exist_ok=True)
    objs = [os.path.join(objdir, os.path.basename(s).replace(".cu", ".o")) for s in SOURCES]

    def compile_one(args):
        src, obj = args
        subprocess.check_call([NVCC, *flags, *inc, "-c", src, "-o", obj])

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        list(ex.map(compile_one, zip(SOURCES, objs)))
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", lib, *objs, *link])
    return lib


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv, debug="--debug" in sys.argv)
    print(LIB_DEBUG if "--debug" in sys.argv else LIB)
