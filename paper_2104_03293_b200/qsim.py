"""Thin ctypes binding of libqsim.so (include/qsim.h).

Argument marshalling only: every step of the hot path runs in the CUDA kernels of
libqsim.so.  There is no CPU fallback -- importing this module fails loudly if the
library is missing, and every non-OK return code raises QsimError.

The functions keep the C names (qsim_create, qsim_set_ising, ...); `QSim` is a small
convenience wrapper owning one handle.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# QSIM_LIBRARY selects another build of the same library (the debug build libqsim_debug.so of
# tests/test_gpu_debug_build.py); there is no fallback: the file must exist
LIB_PATH = os.environ.get("QSIM_LIBRARY") or os.path.join(_HERE, "libqsim.so")

QSIM_OK = 0
QSIM_EINVAL = -1
QSIM_ENOMEM = -2
QSIM_ERANGE = -3
QSIM_ESTATE = -4
QSIM_EUNSUPPORTED = -5
QSIM_ECUDA = -6
QSIM_ENCCL = -7
QSIM_FP64 = 0
QSIM_FP32 = 1
QSIM_SWAP_NONE, QSIM_SWAP_FUSED_SPLIT, QSIM_SWAP_FUSED, QSIM_SWAP_LOWBIT = 0, 1, 2, 3
QSIM_SWAP_COLLECTIVE, QSIM_SWAP_INPLACE_STAGED, QSIM_SWAP_FUSED_INPLACE = 4, 5, 6

_ERRNAMES = {QSIM_EINVAL: "EINVAL", QSIM_ENOMEM: "ENOMEM", QSIM_ERANGE: "ERANGE",
             QSIM_ESTATE: "ESTATE", QSIM_EUNSUPPORTED: "EUNSUPPORTED", QSIM_ECUDA: "ECUDA",
             QSIM_ENCCL: "ENCCL"}

# every symbol include/qsim.h declares (tests check the library exports all of them)
EXPORTS = ["qsim_create", "qsim_create_ex", "qsim_destroy", "qsim_set_ising", "qsim_init_plus",
           "qsim_apply_qaoa", "qsim_qaoa_batch", "qsim_apply_aqa", "qsim_apply_qsds", "qsim_apply_hadamard", "qsim_aqa_angles", "qsim_expect_hc", "qsim_norm2",
           "qsim_success_prob", "qsim_get_amplitudes", "qsim_energies", "qsim_spin_expectations",
           "qsim_apply_aqa_traced", "qsim_ground_states", "qsim_enumerate", "qsim_sync",
           "qsim_plan_counts", "qsim_plan_positions", "qsim_nccl_unique_id", "qsim_loopback_id",
           "qsim_swap_path", "qsim_num_qubits",
           "qsim_bench_pass", "qsim_profile_enable", "qsim_profile_read", "qsim_profile_passes", "qsim_kernel_launches", "qsim_last_error",
           "qsim_version"]


class QsimError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_ERRNAMES.get(code, code)}: {msg}")
        self.code = code


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                      "g.build()'` (no CPU fallback exists)")

_D = ctypes.POINTER(ctypes.c_double)
_U64 = ctypes.POINTER(ctypes.c_uint64)
_H = ctypes.c_void_p

lib = ctypes.CDLL(LIB_PATH)
lib.qsim_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(_H)]
lib.qsim_create_ex.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                               ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.POINTER(_H)]
lib.qsim_destroy.argtypes = [_H]
lib.qsim_set_ising.argtypes = [_H, _D, _D]
lib.qsim_init_plus.argtypes = [_H]
lib.qsim_apply_qaoa.argtypes = [_H, _D, _D, ctypes.c_int]
lib.qsim_apply_aqa.argtypes = [_H, ctypes.c_double, ctypes.c_int, _D, _D, _D, ctypes.c_int]
lib.qsim_qaoa_batch.argtypes = [_H, _D, _D, ctypes.c_int, ctypes.c_int, _D]
lib.qsim_apply_qsds.argtypes = [_H, ctypes.c_double, ctypes.c_int, _D, _D, _D, ctypes.c_int]
lib.qsim_apply_hadamard.argtypes = [_H, ctypes.c_int]
lib.qsim_aqa_angles.argtypes = [ctypes.c_double, ctypes.c_int, _D, _D, _D, ctypes.c_int, _D, _D]
lib.qsim_expect_hc.argtypes = [_H, _D]
lib.qsim_norm2.argtypes = [_H, _D]
lib.qsim_success_prob.argtypes = [_H, _U64, ctypes.c_int, _D]
lib.qsim_get_amplitudes.argtypes = [_H, ctypes.c_uint64, ctypes.c_uint64, _D]
lib.qsim_energies.argtypes = [_H, ctypes.c_uint64, ctypes.c_uint64, _D]
lib.qsim_sync.argtypes = [_H]
lib.qsim_spin_expectations.argtypes = [_H, _D]
lib.qsim_apply_aqa_traced.argtypes = [_H, ctypes.c_double, ctypes.c_int, _D, _D, _D, ctypes.c_int, _D]
lib.qsim_ground_states.argtypes = [_H, _U64, ctypes.c_int, _D, _U64]
lib.qsim_enumerate.argtypes = [ctypes.c_int, _D, _D, _U64, ctypes.c_int, _D, _U64, _D]
lib.qsim_plan_counts.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                 ctypes.POINTER(ctypes.c_int), _U64]
lib.qsim_plan_positions.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
lib.qsim_nccl_unique_id.argtypes = [ctypes.c_void_p]
lib.qsim_loopback_id.argtypes = [ctypes.c_int, ctypes.c_void_p]
lib.qsim_swap_path.argtypes = [_H]
lib.qsim_num_qubits.argtypes = [_H]
lib.qsim_bench_pass.argtypes = [_H, ctypes.c_int, ctypes.c_int, ctypes.c_int, _D]
lib.qsim_profile_enable.argtypes = [_H, ctypes.c_int]
lib.qsim_profile_read.argtypes = [_H, _D, _U64, _D]
lib.qsim_profile_passes.argtypes = [_H, _D, ctypes.POINTER(ctypes.c_int), ctypes.c_int]
lib.qsim_kernel_launches.argtypes = [_H]
lib.qsim_kernel_launches.restype = ctypes.c_uint64
lib.qsim_last_error.argtypes = [_H]
lib.qsim_last_error.restype = ctypes.c_char_p
lib.qsim_version.restype = ctypes.c_char_p
for _name in EXPORTS:
    if _name not in ("qsim_kernel_launches", "qsim_last_error", "qsim_version"):
        getattr(lib, _name).restype = ctypes.c_int


def _f64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_D)


def _check(rc: int, h=None):
    if rc != QSIM_OK:
        raise QsimError(rc, (lib.qsim_last_error(h) or b"").decode())


# ------------------------------------------------------------------ C-named functions
def qsim_create(n: int, precision: int = QSIM_FP64):
    h = _H()
    _check(lib.qsim_create(int(n), int(precision), ctypes.byref(h)))
    return h


def qsim_create_ex(n: int, precision: int, rank: int, world: int, nccl_unique_id: bytes | None = None,
                   state_buf: int | None = None, buf_bytes: int = 0, cuda_stream: int | None = None):
    h = _H()
    uid = ctypes.create_string_buffer(bytes(nccl_unique_id), 128) if nccl_unique_id is not None else None
    _check(lib.qsim_create_ex(int(n), int(precision), int(rank), int(world), uid, state_buf, int(buf_bytes),
                              cuda_stream, ctypes.byref(h)))
    return h


def qsim_destroy(h) -> None:
    _check(lib.qsim_destroy(h))


def qsim_set_ising(h, hfield, J) -> None:
    hf = _f64(hfield)
    n = hf.shape[0]
    JJ = _f64(J).reshape(n, n)
    _check(lib.qsim_set_ising(h, _dp(hf), _dp(JJ)), h)


def qsim_init_plus(h) -> None:
    _check(lib.qsim_init_plus(h), h)


def qsim_apply_qaoa(h, gamma, beta) -> None:
    g, b = _f64(gamma), _f64(beta)
    if g.shape != b.shape or g.ndim != 1:
        raise ValueError("gamma and beta must be 1-D arrays of equal length")
    _check(lib.qsim_apply_qaoa(h, _dp(g), _dp(b), int(g.shape[0])), h)


def qsim_qaoa_batch(h, gamma, beta) -> np.ndarray:
    """<H_C> for each row of gamma, beta ([count, p]) -- n <= 12, one launch"""
    g, b = _f64(gamma), _f64(beta)
    if g.ndim == 1:
        g, b = g[:, None], b[:, None]
    if g.shape != b.shape or g.ndim != 2:
        raise ValueError("gamma and beta must be [count, p] arrays of equal shape")
    g, b = np.ascontiguousarray(g), np.ascontiguousarray(b)
    out = np.empty(g.shape[0])
    _check(lib.qsim_qaoa_batch(h, _dp(g), _dp(b), int(g.shape[1]), int(g.shape[0]), _dp(out)), h)
    return out


def qsim_apply_aqa(h, T: float, p: int, s, A, B) -> None:
    s, A, B = _f64(s), _f64(A), _f64(B)
    _check(lib.qsim_apply_aqa(h, float(T), int(p), _dp(s), _dp(A), _dp(B), int(s.shape[0])), h)


def qsim_apply_qsds(h, tau: float, n_steps: int, s, A, B) -> None:
    s, A, B = _f64(s), _f64(A), _f64(B)
    _check(lib.qsim_apply_qsds(h, float(tau), int(n_steps), _dp(s), _dp(A), _dp(B), int(s.shape[0])), h)


def qsim_apply_hadamard(h, reps: int) -> None:
    _check(lib.qsim_apply_hadamard(h, int(reps)), h)


def qsim_aqa_angles(T: float, p: int, s, A, B):
    s, A, B = _f64(s), _f64(A), _f64(B)
    g = np.empty(p)
    b = np.empty(p)
    _check(lib.qsim_aqa_angles(float(T), int(p), _dp(s), _dp(A), _dp(B), int(s.shape[0]), _dp(g), _dp(b)))
    return g, b


def qsim_expect_hc(h) -> float:
    out = ctypes.c_double()
    _check(lib.qsim_expect_hc(h, ctypes.byref(out)), h)
    return out.value


def qsim_norm2(h) -> float:
    out = ctypes.c_double()
    _check(lib.qsim_norm2(h, ctypes.byref(out)), h)
    return out.value


def qsim_success_prob(h, ground_states) -> float:
    gs = np.ascontiguousarray(np.asarray(ground_states, dtype=np.uint64))
    out = ctypes.c_double()
    _check(lib.qsim_success_prob(h, gs.ctypes.data_as(_U64), int(gs.shape[0]), ctypes.byref(out)), h)
    return out.value


def qsim_get_amplitudes(h, first: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.complex128)
    _check(lib.qsim_get_amplitudes(h, int(first), int(count), _dp(out.view(np.float64))), h)
    return out


def qsim_energies(h, first: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.float64)
    _check(lib.qsim_energies(h, int(first), int(count), _dp(out)), h)
    return out


def qsim_spin_expectations(h) -> np.ndarray:
    out = np.empty(qsim_num_qubits(h))
    _check(lib.qsim_spin_expectations(h, _dp(out)), h)
    return out


def qsim_apply_aqa_traced(h, T: float, p: int, s, A, B) -> np.ndarray:
    s, A, B = _f64(s), _f64(A), _f64(B)
    tr = np.empty((p, qsim_num_qubits(h)))
    _check(lib.qsim_apply_aqa_traced(h, float(T), int(p), _dp(s), _dp(A), _dp(B), int(s.shape[0]), _dp(tr)), h)
    return tr


def qsim_ground_states(h, max_out: int = 64):
    """-> (list of minimisers (ascending), minimum energy, number of minimisers)"""
    out = np.zeros(max(max_out, 1), dtype=np.uint64)
    emin = ctypes.c_double()
    cnt = ctypes.c_uint64()
    _check(lib.qsim_ground_states(h, out.ctypes.data_as(_U64), int(max_out), ctypes.byref(emin),
                                  ctypes.byref(cnt)), h)
    return [int(x) for x in out[: min(cnt.value, max_out)]], emin.value, cnt.value


def qsim_enumerate(hfield, J, max_out: int = 64):
    """-> (minimisers ascending, minimum energy, number of minimisers, device ms); no state."""
    hf = _f64(hfield)
    n = hf.shape[0]
    JJ = _f64(J).reshape(n, n)
    out = np.zeros(max(max_out, 1), dtype=np.uint64)
    emin, ms = ctypes.c_double(), ctypes.c_double()
    cnt = ctypes.c_uint64()
    _check(lib.qsim_enumerate(n, _dp(hf), _dp(JJ), out.ctypes.data_as(_U64), int(max_out), ctypes.byref(emin),
                              ctypes.byref(cnt), ctypes.byref(ms)))
    return [int(x) for x in out[: min(cnt.value, max_out)]], emin.value, cnt.value, ms.value


def qsim_sync(h) -> None:
    _check(lib.qsim_sync(h), h)


def qsim_plan_counts(n: int, world: int, p: int):
    pa, sw = ctypes.c_int(), ctypes.c_int()
    amps = ctypes.c_uint64()
    _check(lib.qsim_plan_counts(int(n), int(world), int(p), ctypes.byref(pa), ctypes.byref(sw),
                                ctypes.byref(amps)))
    return pa.value, sw.value, amps.value


def qsim_plan_positions(n: int, world: int, layers: int):
    pos = (ctypes.c_int * n)()
    _check(lib.qsim_plan_positions(int(n), int(world), int(layers), pos))
    return list(pos)


def qsim_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib.qsim_nccl_unique_id(buf))
    return buf.raw


def qsim_loopback_id(world: int) -> bytes:
    """128-byte group id of the in-process loopback transport (world ranks = threads of this
    process on the current device, each passing the id to qsim_create_ex)."""
    buf = ctypes.create_string_buffer(128)
    _check(lib.qsim_loopback_id(int(world), buf))
    return buf.raw


def qsim_swap_path(h) -> int:
    rc = lib.qsim_swap_path(h)
    _check(min(rc, 0), h)
    return rc


def qsim_num_qubits(h) -> int:
    rc = lib.qsim_num_qubits(h)
    _check(min(rc, 0), h)
    return rc


def qsim_bench_pass(h, set_index: int, phase: int, reps: int = 5) -> float:
    out = ctypes.c_double()
    _check(lib.qsim_bench_pass(h, int(set_index), int(phase), int(reps), ctypes.byref(out)), h)
    return out.value


def qsim_profile_enable(h, on: bool = True) -> None:
    _check(lib.qsim_profile_enable(h, int(bool(on))), h)


def qsim_profile_read(h):
    """-> (pass-kernel ms summed, number of pass launches, algorithmic bytes summed)"""
    ms, by = ctypes.c_double(), ctypes.c_double()
    cnt = ctypes.c_uint64()
    _check(lib.qsim_profile_read(h, ctypes.byref(ms), ctypes.byref(cnt), ctypes.byref(by)), h)
    return ms.value, cnt.value, by.value


QSIM_PASS_PLAIN12, QSIM_PASS_PLAIN_RUN, QSIM_PASS_TURN12, QSIM_PASS_TURN_RUN = 0, 1, 2, 3
QSIM_PASS_MOVING, QSIM_PASS_INIT, QSIM_PASS_REDUCE = 4, 8, 16


def qsim_profile_passes(h, cap: int = 4096, kinds: bool = False):
    """-> per-pass durations (ms) of the recorded passes, in launch order (and, with kinds=True,
    their pass programs: QSIM_PASS_* codes)"""
    out = np.zeros(cap)
    kd = np.zeros(cap, dtype=np.int32)
    rc = lib.qsim_profile_passes(h, out.ctypes.data_as(_D), kd.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), cap)
    _check(min(rc, 0), h)
    k = min(rc, cap)
    return (out[:k].copy(), kd[:k].copy()) if kinds else out[:k].copy()


def qsim_kernel_launches(h) -> int:
    return int(lib.qsim_kernel_launches(h))


def qsim_last_error(h=None) -> str:
    return (lib.qsim_last_error(h) or b"").decode()


def qsim_version() -> str:
    return lib.qsim_version().decode()


# ------------------------------------------------------------------ convenience wrapper
class QSim:
    """One state-vector handle.  Single GPU: QSim(n).  Multi-GPU (SPMD, one process
    per GPU): QSim(n, rank=r, world=G, nccl_unique_id=uid).  Loopback test transport (G
    threads of one process on one device): nccl_unique_id=qsim_loopback_id(G), one thread per
    rank."""

    def __init__(self, n: int, rank: int = 0, world: int = 1, nccl_unique_id: bytes | None = None,
                 state_buf: int | None = None, buf_bytes: int = 0, cuda_stream: int | None = None,
                 precision: int = QSIM_FP64):
        self.n = n
        self.rank = rank
        self.world = world
        self.precision = precision
        if world == 1 and state_buf is None and cuda_stream is None:
            self.h = qsim_create(n, precision)
        else:
            self.h = qsim_create_ex(n, precision, rank, world, nccl_unique_id, state_buf, buf_bytes,
                                    cuda_stream)

    def close(self):
        if self.h is not None:
            qsim_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_ising(self, hfield, J):
        qsim_set_ising(self.h, hfield, J)

    def init_plus(self):
        qsim_init_plus(self.h)

    def apply_qaoa(self, gamma, beta):
        qsim_apply_qaoa(self.h, gamma, beta)

    def qaoa_batch(self, gamma, beta):
        return qsim_qaoa_batch(self.h, gamma, beta)

    def apply_aqa(self, T, p, s, A, B):
        qsim_apply_aqa(self.h, T, p, s, A, B)

    def apply_qsds(self, tau, n_steps, s, A, B):
        qsim_apply_qsds(self.h, tau, n_steps, s, A, B)

    def apply_hadamard(self, reps):
        qsim_apply_hadamard(self.h, reps)

    def expect_hc(self):
        return qsim_expect_hc(self.h)

    def norm2(self):
        return qsim_norm2(self.h)

    def success_prob(self, gs):
        return qsim_success_prob(self.h, gs)

    def amplitudes(self, first=0, count=None):
        if count is None:
            count = (1 << self.n) - first
        return qsim_get_amplitudes(self.h, first, count)

    def energies(self, first=0, count=None):
        if count is None:
            count = (1 << self.n) - first
        return qsim_energies(self.h, first, count)

    def spins(self):
        return qsim_spin_expectations(self.h)

    def apply_aqa_traced(self, T, p, s, A, B):
        return qsim_apply_aqa_traced(self.h, T, p, s, A, B)

    def ground_states(self, max_out=64):
        return qsim_ground_states(self.h, max_out)

    def sync(self):
        qsim_sync(self.h)

    @property
    def swap_path(self):
        return qsim_swap_path(self.h)

    @property
    def launches(self):
        return qsim_kernel_launches(self.h)
