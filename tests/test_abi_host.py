"""CPU-only checks of the C-ABI library: it loads, exports every symbol include/qsim.h
declares, and its host-only logic (AQA angles, pass planner, permutation bookkeeping)
is right.  No compute calls need a GPU here."""
import ctypes
import json
import os
import re

import numpy as np
import pytest

from tests.conftest import ROOT

HEADER = os.path.join(ROOT, "include", "qsim.h")


@pytest.fixture(scope="module")
def Q():
    from paper_2104_03293_b200 import build

    build.build()
    from paper_2104_03293_b200 import qsim

    return qsim


def header_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(qsim_[a-z0-9_]+)\s*\(", txt)))


def test_header_symbols_exported(Q):
    syms = header_symbols()
    assert len(syms) >= 18
    lib = ctypes.CDLL(Q.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(Q.EXPORTS) == syms


def test_library_is_sm100a(Q):
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", Q.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_version(Q):
    assert "sm_100a" in Q.qsim_version()


def test_aqa_angles_golden(Q, golden_dir):
    g = json.load(open(os.path.join(golden_dir, "aqa_angles_toy.json")))
    sch = g["schedule"]
    for case in g["cases"]:
        gam, bet = Q.qsim_aqa_angles(case["T"], case["p"], sch["s"], sch["A"], sch["B"])
        assert list(bet) == case["beta"] and list(gam) == case["gamma"]


def test_aqa_angles_match_oracle(Q):
    from oracle import oracle as o
    from paper_2104_03293_b200 import instances as inst

    s, A, B = inst.dw_like_schedule()
    for p in (2, 5, 16, 51):
        T = 0.4 * p
        g1, b1 = Q.qsim_aqa_angles(T, p, s, 2 * np.pi * A, 2 * np.pi * B)
        g2, b2 = o.aqa_angles(T, p, s, 2 * np.pi * A, 2 * np.pi * B)
        assert np.max(np.abs(g1 - g2)) <= 1e-15 * max(1, np.max(np.abs(g2)))
        assert np.max(np.abs(b1 - b2)) <= 1e-15 * max(1, np.max(np.abs(b2)))


def test_aqa_angles_errors(Q):
    with pytest.raises(Q.QsimError):
        Q.qsim_aqa_angles(1.0, 1, [0, 1], [1, 0], [0, 1])  # p < 2 (reading R8)
    with pytest.raises(Q.QsimError):
        Q.qsim_aqa_angles(1.0, 3, [0, 0.5, 0.4, 1], [1, 1, 1, 0], [0, 0, 0, 1])  # non-monotone knots
    with pytest.raises(Q.QsimError):
        Q.qsim_aqa_angles(float("nan"), 3, [0, 1], [1, 0], [0, 1])


@pytest.mark.parametrize("n", [13, 20, 24, 30, 33])
def test_plan_single_gpu_boustrophedon(Q, n):
    # sets: 12 bits, then runs of <= 9 -> P sets; (P-1) p + 1 passes
    P = 1 + -(-(n - 12) // 9)
    for p in (1, 2, 7):
        passes, swaps, amps = Q.qsim_plan_counts(n, 1, p)
        assert passes == (P - 1) * p + 1 and swaps == 0 and amps == 0


def test_plan_small_state_single_launch(Q):
    assert Q.qsim_plan_counts(12, 1, 5)[0] == 1


@pytest.mark.parametrize("n,world", [(18, 2), (31, 2), (33, 2), (34, 2), (33, 4), (33, 8), (36, 8)])
def test_plan_multi_gpu_transfer_law(Q, n, world):
    """One swap per layer; each rank sends (G-1)/G of its shard per swap (SURVEY §4 ledger law)."""
    g = world.bit_length() - 1
    m = n - g
    P = 1 + -(-(m - 12) // 9)
    # top-bit swap schedule: P passes per layer + a trailing pass.  Opt-in low-bit swap schedule
    # (QSIM_LOWSWAP=1; G = 2 with 22 <= m <= 32): the single-GPU boustrophedon, (P-1) p + 1 passes
    low = os.environ.get("QSIM_LOWSWAP") == "1" and world == 2 and 22 <= m <= 32
    for p in (1, 3):
        passes, swaps, amps = Q.qsim_plan_counts(n, world, p)
        assert swaps == p
        assert passes == ((P - 1) * p + 1 if low else P * p + 1)
        assert amps * world == (world - 1) * (1 << m)


def test_plan_rejects_bad_layouts(Q):
    with pytest.raises(Q.QsimError):
        Q.qsim_plan_counts(33, 3, 1)
    with pytest.raises(Q.QsimError):
        Q.qsim_plan_counts(14, 8, 1)  # n - g < 15


def test_plan_positions_swap_involution(Q):
    n, world = 20, 4
    p0 = Q.qsim_plan_positions(n, world, 0)
    p1 = Q.qsim_plan_positions(n, world, 1)
    p2 = Q.qsim_plan_positions(n, world, 2)
    assert p0 == list(range(n)) and p2 == p0
    assert sorted(p1) == list(range(n))
    # top 2 local qubits <-> 2 global qubits
    assert p1[16:18] == [18, 19] and p1[18:20] == [16, 17] and p1[:16] == list(range(16))


def test_create_without_gpu_fails_loudly(Q):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(Q.QsimError) as ei:
        Q.qsim_create(10)
    assert ei.value.code == Q.QSIM_ECUDA


def test_create_rejects_bad_arguments(Q):
    with pytest.raises(Q.QsimError) as ei:
        Q.qsim_create(10, 7)  # neither QSIM_FP64 nor QSIM_FP32
    assert ei.value.code == Q.QSIM_EINVAL
    with pytest.raises(Q.QsimError) as ei:
        Q.qsim_create(0)
    assert ei.value.code == Q.QSIM_EINVAL


def test_plan_low_bit_swap(Q, monkeypatch):
    """Opt-in low-bit swap schedule (G = 2, m >= 22): the global qubit is exchanged with passenger
    position 2 once per layer, 2 passes per layer as on one GPU."""
    monkeypatch.setenv("QSIM_LOWSWAP", "1")
    n = 31
    p1 = Q.qsim_plan_positions(n, 2, 1)
    assert p1[2] == 30 and p1[30] == 2
    assert [p1[i] for i in range(n) if i not in (2, 30)] == [i for i in range(n) if i not in (2, 30)]
    assert Q.qsim_plan_positions(n, 2, 2) == list(range(n))
    for p in (1, 4):
        passes, swaps, amps = Q.qsim_plan_counts(n, 2, p)
        assert passes == 2 * p + 1 and swaps == p and amps * 2 == 1 << 30
    monkeypatch.delenv("QSIM_LOWSWAP")
    assert Q.qsim_plan_positions(n, 2, 1)[29] == 30  # default: top local bit <-> global


def test_loopback_ids(Q):
    """qsim_loopback_id: host-only group ids (magic prefix + key + world), fresh per call; worlds
    other than 1, 2, 4, 8 are EINVAL.  A loopback id is not mistaken for an ncclUniqueId."""
    a, b = Q.qsim_loopback_id(2), Q.qsim_loopback_id(2)
    assert len(a) == 128 and a != b and a[:15] == b"QSIM-LOOPBACK-1" == b[:15]
    assert int.from_bytes(a[24:28], "little") == 2
    for w in (0, 3, 16):
        with pytest.raises(Q.QsimError) as ei:
            Q.qsim_loopback_id(w)
        assert ei.value.code == Q.QSIM_EINVAL


def test_profile_pass_codes_match_header(Q):
    txt = open(HEADER).read()
    for name in ("QSIM_PASS_PLAIN12", "QSIM_PASS_PLAIN_RUN", "QSIM_PASS_TURN12", "QSIM_PASS_TURN_RUN",
                 "QSIM_PASS_MOVING", "QSIM_PASS_INIT", "QSIM_PASS_REDUCE", "QSIM_SWAP_FUSED_INPLACE",
                 "QSIM_SWAP_INPLACE_STAGED", "QSIM_SWAP_COLLECTIVE", "QSIM_SWAP_LOWBIT", "QSIM_SWAP_FUSED_SPLIT"):
        m = re.search(name + r"\s*=\s*(\d+)", txt)
        assert m and int(m.group(1)) == getattr(Q, name), name


def _build_c_example(tmpdir):
    import subprocess

    exe = os.path.join(str(tmpdir), "qaoa_c")
    libdir = os.path.join(ROOT, "paper_2104_03293_b200")
    subprocess.check_call(["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "qaoa_c.c"), "-L", libdir, "-l:libqsim.so",
                           f"-Wl,-rpath,{libdir}", "-o", exe])
    return exe


def test_c_example_compiles_and_links(Q, tmp_path):
    """examples/qaoa_c.c uses the C-ABI from plain C (no Python, no torch): it compiles against
    include/qsim.h and links against libqsim.so (running it needs a GPU: test_gpu_parity)."""
    assert os.path.exists(_build_c_example(tmp_path))


def c_example_instance(n, p):
    """the LCG instance and angles of examples/qaoa_c.c, reproduced for the oracle"""
    seed = 12345
    M = (1 << 64) - 1
    h = np.zeros(n)
    J = np.zeros((n, n))
    for i in range(n):
        seed = (seed * 6364136223846793005 + 1442695040888963407) & M
        h[i] = (int((seed >> 33) % 9) - 4) / 2.0
        for j in range(i + 1, n):
            seed = (seed * 6364136223846793005 + 1442695040888963407) & M
            J[i, j] = (int((seed >> 33) % 5) - 2) / 2.0
    k = np.arange(1, p + 1)
    return h, J, 0.8 * k / (p + 1), -0.6 * (1.0 - k / (p + 1))
