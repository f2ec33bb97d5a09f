"""ctypes binding for the plain-C CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of bench.py -- never by the product
package ``paper_2104_03293_b200``.  Shares no code with the CUDA path.

Conventions: see the header of oracle.c (qubit j <-> bit j, s = 2 z - 1,
E(z) = sum h_i s_i + sum_{i<j} J_ij s_i s_j, eq:HC P:252-255).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_D = ctypes.POINTER(ctypes.c_double)
_U64 = ctypes.POINTER(ctypes.c_uint64)


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (-O2, no FMA contraction, no fast-math, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared",
               "-fPIC", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.oracle_energy.restype = ctypes.c_double
        L.oracle_energy.argtypes = [ctypes.c_int, _D, _D, ctypes.c_uint64]
        L.oracle_energies.argtypes = [ctypes.c_int, _D, _D, ctypes.c_uint64, ctypes.c_uint64, _D]
        L.oracle_init_plus.argtypes = [ctypes.c_int, _D]
        L.oracle_apply_phase.argtypes = [ctypes.c_int, _D, _D, _D, ctypes.c_double, _D]
        L.oracle_apply_rx.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, _D]
        L.oracle_apply_mixer.argtypes = [ctypes.c_int, ctypes.c_double, _D]
        L.oracle_apply_qaoa.argtypes = [ctypes.c_int, _D, _D, _D, _D, ctypes.c_int, _D]
        L.oracle_apply_layers.argtypes = [ctypes.c_int, _D, _D, _D, _D, ctypes.c_int, _D]
        L.oracle_aqa_angles.restype = ctypes.c_int
        L.oracle_aqa_angles.argtypes = [ctypes.c_double, ctypes.c_int, _D, _D, _D, ctypes.c_int,
                                        _D, _D]
        L.oracle_expect_hc.restype = ctypes.c_double
        L.oracle_expect_hc.argtypes = [ctypes.c_int, _D, _D, _D, _D]
        L.oracle_norm2.restype = ctypes.c_double
        L.oracle_norm2.argtypes = [ctypes.c_int, _D]
        L.oracle_success_prob.restype = ctypes.c_double
        L.oracle_success_prob.argtypes = [ctypes.c_int, _D, _U64, ctypes.c_int]
        L.oracle_ground_states.restype = ctypes.c_int
        L.oracle_ground_states.argtypes = [ctypes.c_int, _D, _D, _U64, ctypes.c_int, _D]
        L.oracle_num_threads.restype = ctypes.c_int
        L.oracle_spin_expectations.argtypes = [ctypes.c_int, _D, _D]
        L.oracle_apply_qsds.argtypes = [ctypes.c_int, _D, _D, ctypes.c_double, ctypes.c_int, _D, _D, _D,
                                        ctypes.c_int, _D]
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_D)


def _f64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def _hJ(h, J):
    h = _f64(h)
    n = h.shape[0]
    J = _f64(J).reshape(n, n)
    return n, h, J


def energy(h, J, z: int) -> float:
    n, h, J = _hJ(h, J)
    return lib().oracle_energy(n, _dp(h), _dp(J), int(z))


def energies(h, J, first: int = 0, count: int | None = None) -> np.ndarray:
    n, h, J = _hJ(h, J)
    if count is None:
        count = (1 << n) - first
    out = np.empty(count, dtype=np.float64)
    lib().oracle_energies(n, _dp(h), _dp(J), int(first), int(count), _dp(out))
    return out


def _psi_view(psi: np.ndarray) -> np.ndarray:
    assert psi.dtype == np.complex128 and psi.flags.c_contiguous
    return psi.view(np.float64)


def init_plus(n: int) -> np.ndarray:
    psi = np.empty(1 << n, dtype=np.complex128)
    lib().oracle_init_plus(n, _dp(_psi_view(psi)))
    return psi


def apply_phase(h, J, gamma: float, psi: np.ndarray) -> None:
    n, h, J = _hJ(h, J)
    lib().oracle_apply_phase(n, _dp(h), _dp(J), None, float(gamma), _dp(_psi_view(psi)))


def apply_rx(n: int, q: int, beta: float, psi: np.ndarray) -> None:
    lib().oracle_apply_rx(n, q, float(beta), _dp(_psi_view(psi)))


def apply_mixer(n: int, beta: float, psi: np.ndarray) -> None:
    lib().oracle_apply_mixer(n, float(beta), _dp(_psi_view(psi)))


def qaoa_state(h, J, gamma, beta) -> np.ndarray:
    """|beta,gamma> of eq:QAOA_state, layer 1 first, phase then mixer."""
    n, h, J = _hJ(h, J)
    g = _f64(gamma)
    b = _f64(beta)
    assert g.shape == b.shape and g.ndim == 1 and g.shape[0] >= 1
    psi = np.empty(1 << n, dtype=np.complex128)
    lib().oracle_apply_qaoa(n, _dp(h), _dp(J), _dp(g), _dp(b), g.shape[0], _dp(_psi_view(psi)))
    return psi


def apply_layers(h, J, gamma, beta, psi: np.ndarray) -> None:
    n, h, J = _hJ(h, J)
    g = _f64(gamma)
    b = _f64(beta)
    lib().oracle_apply_layers(n, _dp(h), _dp(J), _dp(g), _dp(b), g.shape[0], _dp(_psi_view(psi)))


def aqa_angles(T: float, p: int, s, A, B):
    """eq:beta_k / eq:gamma_k with s_k=(k-1)/(p-1) and tau=T/p."""
    s, A, B = _f64(s), _f64(A), _f64(B)
    g = np.empty(p, dtype=np.float64)
    b = np.empty(p, dtype=np.float64)
    rc = lib().oracle_aqa_angles(float(T), int(p), _dp(s), _dp(A), _dp(B), s.shape[0], _dp(g), _dp(b))
    if rc != 0:
        raise ValueError("oracle_aqa_angles: invalid arguments")
    return g, b


def aqa_state(h, J, T: float, p: int, s, A, B) -> np.ndarray:
    g, b = aqa_angles(T, p, s, A, B)
    return qaoa_state(h, J, g, b)


def expect_hc(h, J, psi: np.ndarray, with_abs: bool = False):
    """<H_C> = sum |psi_z|^2 E(z); optionally also sum |psi_z|^2 |E(z)| (reading R12)."""
    n, h, J = _hJ(h, J)
    a = ctypes.c_double(0.0)
    v = lib().oracle_expect_hc(n, _dp(h), _dp(J), _dp(_psi_view(psi)), ctypes.byref(a))
    return (v, a.value) if with_abs else v


def norm2(psi: np.ndarray) -> float:
    n = int(psi.shape[0]).bit_length() - 1
    return lib().oracle_norm2(n, _dp(_psi_view(psi)))


def success_prob(psi: np.ndarray, ground_states) -> float:
    n = int(psi.shape[0]).bit_length() - 1
    gs = np.ascontiguousarray(np.asarray(ground_states, dtype=np.uint64))
    return lib().oracle_success_prob(n, _dp(_psi_view(psi)), gs.ctypes.data_as(_U64), gs.shape[0])


def ground_states(h, J, max_out: int = 64):
    """Brute-force minimisers of E(z) over all 2^n z (ascending), and the minimum energy."""
    n, h, J = _hJ(h, J)
    out = np.zeros(max_out, dtype=np.uint64)
    emin = ctypes.c_double(0.0)
    cnt = lib().oracle_ground_states(n, _dp(h), _dp(J), out.ctypes.data_as(_U64), max_out,
                                     ctypes.byref(emin))
    return [int(x) for x in out[: min(cnt, max_out)]], emin.value, cnt


def spin_expectations(psi: np.ndarray) -> np.ndarray:
    """<sigma^z_i> = sum_z |psi_z|^2 s_i(z), i = 0..n-1."""
    n = int(psi.shape[0]).bit_length() - 1
    out = np.empty(n)
    lib().oracle_spin_expectations(n, _dp(_psi_view(psi)), _dp(out))
    return out


def qsds_state(h, J, tau: float, nsteps: int, s, A, B) -> np.ndarray:
    """QSDS combined second-order stepping (eq. AQA4) from |+>^n, l = 0..nsteps."""
    n, h, J = _hJ(h, J)
    s, A, B = _f64(s), _f64(A), _f64(B)
    psi = init_plus(n)
    lib().oracle_apply_qsds(n, _dp(h), _dp(J), float(tau), int(nsteps), _dp(s), _dp(A), _dp(B), s.shape[0],
                            _dp(_psi_view(psi)))
    return psi


def num_threads() -> int:
    return lib().oracle_num_threads()
