"""B200-native (sm_100a) FP64 state-vector engine for the QAOA / AQA hot path of
arXiv:2104.03293 (JUQCS-G paper).

    csrc/            CUDA kernels + C++ engine + C-ABI implementation (libqsim.so)
    qsim.py          thin ctypes binding with the C names (import fails if libqsim.so is missing)
    instances.py     seeded synthetic input generators (shared with the tests; no method arithmetic)
    problems.py      host-side problem reductions (exact cover / 2-SAT -> Ising, rescale r)
    build.py         nvcc build of libqsim.so in-tree
"""
