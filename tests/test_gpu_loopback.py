"""Multi-GPU swap paths on ONE GPU: the G ranks
of a sharded handle are threads of this process (the loopback transport of qsim_loopback_id),
each with its own shard buffers and stream.  The engine, the pass kernels with their peer
stores, the split-swap group ranges, the in-place handshake and the permutation / flip
bookkeeping are the NCCL path's; only the transport differs.  Every swap path runs here: fused
split (default), fused in place (QSIM_SWAP_INPLACE=1: no second buffer, the n = 36 path),
collective (QSIM_FUSED_SWAP=0), staged in place (both), low-bit (QSIM_LOWSWAP=1) and
non-default split weights (QSIM_SPLIT_W) and spatial-split shares (QSIM_SP), against the oracle (full state at n <= 24, structured
pins P4/P8/P9 at n = 31-33, up to 8 ranks)."""
from __future__ import annotations

import threading

import pytest

from tests.sharded_checks import run_checks

pytestmark = pytest.mark.gpu


def _q():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2104_03293_b200 import qsim as Q

    return Q


class _Ids:
    """fresh loopback group id per handle, shared by the world rank threads (k-th handle of
    every rank gets the k-th id)"""

    def __init__(self, Q, world):
        self.Q, self.world, self.lock, self.ids, self.count = Q, world, threading.Lock(), {}, [0] * world

    def get(self, rank):
        k = self.count[rank]
        self.count[rank] += 1
        with self.lock:
            if k not in self.ids:
                self.ids[k] = self.Q.qsim_loopback_id(self.world)
            return self.ids[k]


def run_loopback(world, body, timeout=1500):
    """run body(rank, new_sim) on `world` threads; returns rank 0's result, re-raises errors"""
    Q = _q()
    ids = _Ids(Q, world)
    res, errs = [None] * world, []

    def worker(rank):
        try:
            def new_sim(n, precision=Q.QSIM_FP64):
                return Q.QSim(n, rank=rank, world=world, nccl_unique_id=ids.get(rank), precision=precision)

            res[rank] = body(rank, new_sim)
        except BaseException as e:  # noqa: BLE001
            errs.append((rank, repr(e)))

    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout)
    assert not any(t.is_alive() for t in th), "loopback ranks hung"
    assert not errs, errs
    return res[0]


def _check(world, n, expect_path, p=3, full=True, extras=True):
    out = run_loopback(world, lambda r, ns: run_checks(r, world, ns, n, p=p, full=full, extras=extras))
    paths = [d for (nm, ok, d) in out if nm.endswith("swap path")]
    assert paths and int(paths[0]) == expect_path, (paths, expect_path)
    bad = [(nm, d) for (nm, ok, d) in out if not ok]
    assert not bad, bad
    assert len(out) >= 5


@pytest.mark.parametrize("world,n", [(2, 18), (2, 24), (4, 20), (4, 24), (8, 22)])
def test_loopback_fused_split(world, n):
    Q = _q()
    _check(world, n, Q.QSIM_SWAP_FUSED_SPLIT)


@pytest.mark.parametrize("world,n", [(2, 20), (4, 21)])
def test_loopback_collective_swap(world, n, monkeypatch):
    Q = _q()
    monkeypatch.setenv("QSIM_FUSED_SWAP", "0")
    _check(world, n, Q.QSIM_SWAP_COLLECTIVE, extras=False)


@pytest.mark.parametrize("world,n", [(2, 20), (4, 22), (2, 24)])
def test_loopback_inplace_staged_swap(world, n, monkeypatch):
    Q = _q()
    monkeypatch.setenv("QSIM_SWAP_INPLACE", "1")
    monkeypatch.setenv("QSIM_FUSED_SWAP", "0")
    _check(world, n, Q.QSIM_SWAP_INPLACE_STAGED, extras=(n == 24))


@pytest.mark.parametrize("world,n", [(2, 18), (2, 24), (4, 20), (4, 24), (8, 22)])
def test_loopback_fused_inplace_swap(world, n, monkeypatch):
    """the n = 36 path (no second buffer): peer stores in place after the per-tile handshake"""
    Q = _q()
    monkeypatch.setenv("QSIM_SWAP_INPLACE", "1")
    _check(world, n, Q.QSIM_SWAP_FUSED_INPLACE, extras=(n == 24))


@pytest.mark.parametrize("n", [23, 24])
def test_loopback_lowbit_swap(n, monkeypatch):
    Q = _q()
    monkeypatch.setenv("QSIM_LOWSWAP", "1")
    _check(2, n, Q.QSIM_SWAP_LOWBIT, p=4, extras=False)


@pytest.mark.parametrize("world,n,sp", [(2, 22, "0"), (4, 24, "0"), (2, 24, "0.5"), (8, 23, "0.05")])
def test_loopback_spatial_split_shares(world, n, sp, monkeypatch):
    """QSIM_SP: the whole-tile moving run passes with the group-bits-first order (0) and with
    non-default CTA shares for the moving tiles (the default share is covered above)."""
    Q = _q()
    monkeypatch.setenv("QSIM_SP", sp)
    _check(world, n, Q.QSIM_SWAP_FUSED_SPLIT, extras=False)


def test_loopback_split_weights(monkeypatch):
    Q = _q()
    monkeypatch.setenv("QSIM_SPLIT_W", "0,1,2")  # n = 24, G = 2: 3 passes per layer
    _check(2, 24, Q.QSIM_SWAP_FUSED_SPLIT, extras=False)


@pytest.mark.parametrize("world,n,inplace", [(2, 31, 0), (4, 32, 0), (8, 32, 0), (2, 32, 1), (4, 33, 1),
                                              (8, 33, 1), (2, 33, 1)])
def test_loopback_full_size_structured(world, n, inplace, monkeypatch):
    """the bench's per-GPU shard (2^30 amplitudes per rank) on the fused split path: p = 1
    closed-form <H_C>, energies, cluster (P9) and product (P8) amplitudes spanning global bits"""
    import torch

    need = world * (1 if inplace else 2) * 16 * (1 << (n - (world.bit_length() - 1))) + (8 << 30)
    if torch.cuda.mem_get_info()[0] < need:
        pytest.skip("not enough device memory for the loopback shards")
    Q = _q()
    if inplace:
        monkeypatch.setenv("QSIM_SWAP_INPLACE", "1")
    _check(world, n, Q.QSIM_SWAP_FUSED_INPLACE if inplace else Q.QSIM_SWAP_FUSED_SPLIT, p=3, full=False,
           extras=False)


@pytest.mark.parametrize("world,n,inplace", [(2, 20, 0), (4, 22, 1)])
def test_loopback_stg_moves(world, n, inplace, monkeypatch):
    """QSIM_TMA_MOVES=0: the whole-tile moves of the split swap as 16-byte stores from registers
    instead of TMA tensor stores through the destination ranks' tensor maps"""
    Q = _q()
    monkeypatch.setenv("QSIM_TMA_MOVES", "0")
    if inplace:
        monkeypatch.setenv("QSIM_SWAP_INPLACE", "1")
    _check(world, n, Q.QSIM_SWAP_FUSED_INPLACE if inplace else Q.QSIM_SWAP_FUSED_SPLIT, extras=False)


def test_loopback_caller_owned_buffers():
    """state_buf on a sharded handle: no fused swap (its peer mappings need library-owned
    buffers), so the ranks take the collective swap; parity against the oracle."""
    import numpy as np
    import torch

    from oracle import oracle as o
    from paper_2104_03293_b200 import instances as inst

    Q = _q()
    n, world = 20, 2
    h, J = inst.random_ising(n, 62)
    g, b = np.array([0.4, -0.3, 0.7]), np.array([0.5, -0.6, 1.2])
    bufs = [torch.zeros(1 << (n - 1), dtype=torch.complex128, device="cuda") for _ in range(world)]

    def body(rank, _new_sim):
        s = Q.QSim(n, rank=rank, world=world, nccl_unique_id=ids, state_buf=bufs[rank].data_ptr(),
                   buf_bytes=bufs[rank].numel() * 16)
        try:
            s.set_ising(h, J)
            s.init_plus()
            s.apply_qaoa(g, b)
            return s.amplitudes(), s.swap_path
        finally:
            s.close()

    ids = Q.qsim_loopback_id(world)
    psi, path = run_loopback(world, body)
    assert path == Q.QSIM_SWAP_COLLECTIVE
    assert np.max(np.abs(psi - o.qaoa_state(h, J, g, b))) <= 1e-10


def test_loopback_create_errors():
    """create-time validation of sharded handles: world must be a power of two <= 8 (EINVAL), the
    shard must keep >= 15 local qubits (EUNSUPPORTED), and a group id serves exactly its world
    (a loopback id made for 4 ranks is refused by a world-2 handle: ENCCL)."""
    Q = _q()
    uid4 = Q.qsim_loopback_id(4)
    for args, code in [((20, 0, 3, uid4), Q.QSIM_EINVAL), ((15, 0, 2, Q.qsim_loopback_id(2)), Q.QSIM_EUNSUPPORTED),
                       ((20, 0, 2, uid4), Q.QSIM_ENCCL), ((20, 2, 2, Q.qsim_loopback_id(2)), Q.QSIM_EINVAL)]:
        n, rank, world, uid = args
        with pytest.raises(Q.QsimError) as ei:
            Q.QSim(n, rank=rank, world=world, nccl_unique_id=uid)
        assert ei.value.code == code, (args, ei.value)
