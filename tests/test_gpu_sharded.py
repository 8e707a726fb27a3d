"""GPU parity of the sharded mode: amplitudes split over R = 2, 4, 8 shards by the
high qubits, global<->local qubit exchanges, shard-conditional gates and rank relabels.  The local
communicator drives all shards from one process on one device -- the same host logic and kernels
as the one-process-per-GPU NCCL path, whose exchanges are send/recv of the same half-shards.

Bars as for replica mode: amplitudes <= 1e-10 (c128) / 1e-4 (c64) against the oracle's replay;
shot slots equal the oracle's except oracle-flagged edge draws (the sampler walks the shards in
logical order after restoring the canonical layout, so draws are comparable slot for slot).
"""
import numpy as np
import pytest

from conftest import edge_budget
from workloads import circuits as W

pytestmark = pytest.mark.gpu

TOL = {128: 1e-10, 64: 1e-4}


@pytest.fixture(scope="module")
def T():
    import paper_2508_04880_b200 as T
    return T


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available()
    return torch


def _tree(T, cfg):
    nz = cfg.noise
    return T.build_error_tree(cfg.n, cfg.ops, nz.p1, nz.p2, nz.p_meas, cfg.shots, cfg.seed)


def _random_cfg(seed, n, n_gates, shots=512):
    rng = np.random.default_rng(seed)
    ops = W.random_circuit(rng, n, n_gates)
    return W.Config(f"rand{n}", n, ops, W.Noise(0.01, 0.02, 0.01), shots, seed)


@pytest.mark.parametrize("name,nshards", [("C2a", 2), ("C2a", 8), ("C2b", 2), ("C2b", 4), ("C2b", 8)])
def test_sharded_slots_match_oracle(T, torch, oracle_runs, name, nshards):
    cfg = W.config(name)
    t = _tree(T, cfg)
    comm = T.Comm.local(nshards)
    slots, stats = T.run_tree(t, 128, comm=comm)
    ref, edge = oracle_runs.run(name)
    assert int(edge.sum()) <= edge_budget(cfg.shots)
    bad = (slots != ref) & ~edge
    assert bad.sum() == 0, (int(bad.sum()), int(edge.sum()), stats)
    assert stats["draws"] == cfg.shots and stats["leaves"] == t.n_leaves
    if name == "C2b":
        assert stats["exchanges"] > 0


@pytest.mark.parametrize("name,nshards,prec", [("C2b", 4, 128), ("C2b", 8, 64), ("C3", 2, 128), ("C1", 2, 128)])
def test_sharded_leaf_amplitudes(T, torch, oracle_runs, name, nshards, prec):
    # after a DFS range (uncompute + re-anchor + exchanges), the canonical shards = the oracle replay
    # of the leaf's core (its readout flips relabel draws, reading #7)
    cfg = W.config(name)
    t = _tree(T, cfg)
    ot = oracle_runs.tree(name)
    comm = T.Comm.local(nshards)
    nl = t.n_leaves
    rng = np.random.default_rng(5)
    dt = torch.complex128 if prec == 128 else torch.complex64
    for l in sorted({0, nl - 1, *[int(x) for x in rng.integers(0, nl, size=2)]}):
        d = torch.zeros(1 << cfg.n, dtype=dt, device="cuda")
        T.run_tree(t, prec, d_state=d, leaf_begin=max(0, l - 30), leaf_end=l + 1, flags=T.EXEC_NO_SAMPLE, comm=comm)
        torch.cuda.synchronize()
        err = np.abs(d.cpu().numpy() - ot.replay_leaf_core(l)).max()
        assert err < TOL[prec], (l, err)


@pytest.mark.parametrize("n,nshards", [(13, 2), (14, 4), (15, 8), (6, 4)])
def test_sharded_random_circuits(T, torch, oracle, n, nshards):
    # the full gate set with dense gates, CX / CZ / CP across global and local qubits, Y / X on
    # global qubits: slots and final amplitudes vs the oracle
    cfg = _random_cfg(40 + n, n, 60)
    nz = cfg.noise
    t = T.build_error_tree(n, cfg.ops, nz.p1, nz.p2, nz.p_meas, cfg.shots, cfg.seed)
    ot = oracle.Tree(n, cfg.ops, nz.p1, nz.p2, nz.p_meas, cfg.shots, cfg.seed)
    comm = T.Comm.local(nshards)
    d = torch.zeros(1 << n, dtype=torch.complex128, device="cuda")
    slots, stats = T.run_tree(t, 128, d_state=d, comm=comm)
    torch.cuda.synchronize()
    ref, edge = ot.run()
    assert int(edge.sum()) <= edge_budget(cfg.shots)
    assert ((slots != ref) & ~edge).sum() == 0, stats
    assert np.abs(d.cpu().numpy() - ot.replay_leaf_core(t.n_leaves - 1)).max() < 1e-10
    # the same tree in replica mode gives the same slots
    slots_r, _ = T.run_tree(t, 128)
    assert ((slots != slots_r) & ~edge).sum() == 0


def test_sharded_errors(T, torch):
    n, ops = W.ghz(6)
    t = T.build_error_tree(n, ops, 0.01, 0.01, 0.0, 16, 1)
    with pytest.raises(T.TusqError):
        T.Comm.local(3)
    comm = T.Comm.local(8)
    d = torch.zeros(4, dtype=torch.complex128, device="cuda")
    with pytest.raises(T.TusqError) as e:
        T.run_tree(t, 128, d_state=d, comm=comm)
    assert e.value.status == 6   # TUSQ_ERR_CAPACITY
