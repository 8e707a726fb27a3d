"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star), used exactly: amplitudes max |err| <= 1e-10 (complex128)
and <= 1e-4 (complex64); shot slots exact except draws within the edge window of a CDF edge
(oracle-flagged), which are counted, reported and bounded (conftest.edge_budget: a broken edge
flag cannot make a slot test vacuous); ECM trees bit-exact (tests/test_lib_host.py).

Oracle references: the dense C oracle (oracle/tusq_oracle.c) up to 24 qubits, and for the Adder
leaves at 24 and 30 qubits its sparse replay (oracle/sparse.py, pinned to the dense oracle), which
makes every amplitude of a 2^30 leaf checkable: the GPU vector is compared on the oracle's
support, then the rest of it must be zero to the same tolerance.
"""
import math

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


def dstate(torch, n, prec, host=None):
    dt = torch.complex128 if prec == 128 else torch.complex64
    if host is None:
        return torch.zeros(1 << n, dtype=dt, device="cuda")
    return torch.from_numpy(host.astype(np.complex128 if prec == 128 else np.complex64)).cuda()


def rand_state(rng, n):
    st = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return st / np.linalg.norm(st)


def oracle_apply(oracle, st, n, ops, inverse=False):
    st = st.astype(np.complex128).copy()
    seq = list(reversed(ops)) if inverse else ops
    for g in seq:
        oracle.apply_gate(st, n, g, inverse=inverse)
    return st


def _tree(T, cfg):
    nz = cfg.noise
    return T.build_error_tree(cfg.n, cfg.ops, nz.p1, nz.p2, nz.p_meas, cfg.shots, cfg.seed)


def _check_slots(slots, ref, edge, draws):
    ne = int(edge.sum())
    assert ne <= edge_budget(draws), f"{ne} edge draws of {draws}"
    bad = int(((slots != ref) & ~edge).sum())
    assert bad == 0, f"{bad} slot mismatches ({ne} edge draws excluded)"
    return ne


# ------------------------------------------------------------------ kernels (K1-K5) vs the oracle
@pytest.mark.parametrize("prec", [128, 64])
@pytest.mark.parametrize("kind", list(range(16)))
def test_single_gate_kernels(T, torch, oracle, prec, kind):
    # K1-K4 per gate kind, every qubit position incl. 0 and n-1, both operand orders
    n = 13
    rng = np.random.default_rng(kind)
    st = rand_state(rng, n)
    for q in range(n):
        q1 = (q + 1 + int(rng.integers(n - 1))) % n
        g = W.op(kind, q, q1, float(rng.uniform(-3, 3)))
        for flags in (T.APPLY_UNFUSED, 0):
            d = dstate(torch, n, prec, st)
            T.apply_ops(d, n, prec, [g], flags=flags)
            torch.cuda.synchronize()
            ref = oracle_apply(oracle, st, n, [g])
            assert np.abs(d.cpu().numpy() - ref).max() < TOL[prec], (kind, q, q1, flags)


@pytest.mark.parametrize("prec", [128, 64])
@pytest.mark.parametrize("n", [3, 7, 12, 13, 15, 17])
def test_random_circuits_fused_and_unfused(T, torch, oracle, prec, n):
    rng = np.random.default_rng(100 + n)
    for trial in range(4):
        ops = W.random_circuit(rng, n, int(rng.integers(20, 160)))
        st = rand_state(rng, n)
        ref = oracle_apply(oracle, st, n, ops)
        for flags in (T.APPLY_UNFUSED, 0):
            d = dstate(torch, n, prec, st)
            T.apply_ops(d, n, prec, ops, flags=flags)
            torch.cuda.synchronize()
            err = np.abs(d.cpu().numpy() - ref).max()
            assert err < TOL[prec], (trial, flags, err)
        # uncompute restores the state: forward then inverse
        d = dstate(torch, n, prec, st)
        T.apply_ops(d, n, prec, ops)
        T.apply_ops(d, n, prec, ops, flags=T.APPLY_INVERSE)
        torch.cuda.synchronize()
        err = np.abs(d.cpu().numpy() - st).max()
        assert err < TOL[prec], (trial, err)


def test_adder_circuit_fused(T, torch, oracle):
    # a full noiseless Cuccaro adder (k = 7, n = 16) through the fused path: closed form
    n, ops = W.adder(7)
    d = dstate(torch, n, 128)
    T.init_basis(d, n, 128, 0)
    T.apply_ops(d, n, 128, ops)
    torch.cuda.synchronize()
    st = d.cpu().numpy()
    idx = W.adder_expected_output(7)
    assert abs(st[idx] - 1) < 1e-12 and np.abs(np.delete(st, idx)).max() < 1e-12


def _qft_closed_form_check(torch, d, n, n_idx, seed):
    # amplitude(y) = e^{2 pi i x rev_n(y) / 2^n} / sqrt(2^n) (reading #14; pinned in test_oracle_pins)
    rng = np.random.default_rng(seed)
    y = np.unique(np.concatenate([rng.integers(0, 1 << n, size=n_idx, dtype=np.int64),
                                  np.array([0, 1, (1 << n) - 1], dtype=np.int64)]))
    rev = np.zeros_like(y)
    for b in range(n):
        rev |= ((y >> b) & 1) << (n - 1 - b)
    x = W.qft_input(n)
    ph = (np.uint64(x) * rev.astype(np.uint64)) & np.uint64((1 << n) - 1)
    ref = np.exp(2j * np.pi * ph.astype(np.float64) / float(1 << n)) / math.sqrt(float(1 << n))
    got = d[torch.from_numpy(y).cuda()].cpu().numpy().astype(np.complex128)
    return float(np.abs(got - ref).max()), len(y)


def test_qft30_noiseless_closed_form(T, torch):
    # the full 30-qubit QFT (CX basis, 2 160 gates) through K5 in c128: 10^6 seeded indices
    n, ops = W.qft(30)
    d = dstate(torch, n, 128)
    T.init_basis(d, n, 128, 0)
    T.apply_ops(d, n, 128, ops)
    torch.cuda.synchronize()
    err, m = _qft_closed_form_check(torch, d, n, 1_000_000, 30)
    assert err < TOL[128], (err, m)
    del d
    torch.cuda.empty_cache()


def test_qft34_c64_closed_form(T, torch):
    # C5's circuit (34-qubit QFT, native CP) on ONE B200 in c64 (128 GiB): the noiseless (all-I)
    # path, 10^6 seeded indices against the closed form at the c64 tolerance
    free, _ = torch.cuda.mem_get_info()
    if free < (8 << 34) + (4 << 30):
        pytest.skip(f"needs 132 GiB free device memory, have {free / 2**30:.0f} GiB")
    n, ops = W.qft(34, native_cp=True)
    d = torch.empty(1 << n, dtype=torch.complex64, device="cuda")
    T.init_basis(d, n, 64, 0)
    T.apply_ops(d, n, 64, ops)
    torch.cuda.synchronize()
    err, m = _qft_closed_form_check(torch, d, n, 1_000_000, 34)
    del d
    torch.cuda.empty_cache()
    assert err < TOL[64], (err, m)


# ------------------------------------------------------------------ K6 sampler vs the oracle
def test_init_and_sample_examples(T, torch):
    n = 14
    d = dstate(torch, n, 128)
    T.init_basis(d, n, 128, 0x1234, 0.6, 0.8)
    out = torch.zeros(1000, dtype=torch.int64, device="cuda")
    T.sample(d, n, 128, 1000, 5, 0, out)
    torch.cuda.synchronize()
    assert (out.cpu().numpy() == 0x1234).all()


@pytest.mark.parametrize("prec", [128, 64])
def test_sampler_matches_oracle(T, torch, oracle, prec):
    # shot parity on dense random states, both precisions on the SAME amplitudes (the c64 state is
    # given to the oracle rounded to c64): the two CDFs differ only by fp64 summation order, so
    # the 1e-9 window applies to both and excludes almost nothing (bounded below)
    rng = np.random.default_rng(7)
    for n in (5, 12, 16, 18):
        st = rand_state(rng, n)
        if prec == 64:
            st = st.astype(np.complex64).astype(np.complex128)
        d = dstate(torch, n, prec, st)
        nd = 3000
        out = torch.zeros(nd, dtype=torch.int64, device="cuda")
        T.sample(d, n, prec, nd, 11, 3, out)
        torch.cuda.synchronize()
        ref, edge = oracle.sample_state(st, n, 11, 3, nd, 1e-9)
        got = out.cpu().numpy().astype(np.uint64)
        _check_slots(got, ref, edge, nd)


def test_sampler_peaked_state_c64(T, torch, oracle):
    # c64 leaf parity uses the wider 1e-5 window (reading #17); on a peaked state (16 dominant
    # outcomes over 2^16) its CDF steps are >> 1e-5, so the window still excludes < 1 % of draws
    rng = np.random.default_rng(70)
    n = 16
    st = 1e-6 * (rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n))
    big = rng.choice(1 << n, size=16, replace=False)
    st[big] = rng.normal(size=16) + 1j * rng.normal(size=16)
    st = (st / np.linalg.norm(st)).astype(np.complex64).astype(np.complex128)
    d = dstate(torch, n, 64, st)
    nd = 4000
    out = torch.zeros(nd, dtype=torch.int64, device="cuda")
    T.sample(d, n, 64, nd, 5, 9, out)
    torch.cuda.synchronize()
    ref, edge = oracle.sample_state(st, n, 5, 9, nd, 1e-5)
    assert int(edge.sum()) < nd // 100
    assert ((out.cpu().numpy().astype(np.uint64) != ref) & ~edge).sum() == 0


# ------------------------------------------------------------------ end to end (ECM -> DFTT -> K6)
@pytest.mark.parametrize("name", ["C1", "C2a", "C2b"])
@pytest.mark.parametrize("flags", [0, 0x1, 0x2, 0x3])
def test_run_tree_slots_match_oracle(T, torch, oracle_runs, name, flags):
    # ECM -> DFTT with uncompute -> leaf sampling, slot for slot vs the oracle (cached full run)
    cfg = W.config(name)
    t = _tree(T, cfg)
    slots, stats = T.run_tree(t, 128, flags=flags)
    ref, edge = oracle_runs.run(name)
    ne = _check_slots(slots, ref, edge, cfg.shots)
    assert stats["draws"] == cfg.shots and stats["leaves"] == t.n_leaves
    print(f"{name} flags {flags}: {ne} edge draws of {cfg.shots}, {stats['sampled_vectors']} vectors "
          f"for {stats['leaves']} leaves")
    if name == "C2a":   # GHZ: every error reaches the readout frame -> ONE vector
        assert stats["sampled_vectors"] == 1


def test_replica_leaf_ranges_compose(T, torch, oracle_runs):
    # the slot arrays of 4 partition ranges (as 4 replicas would run them) sum to the full run
    cfg = W.config("C2b")
    t = _tree(T, cfg)
    b = t.partition(4)
    acc = np.zeros(cfg.shots, dtype=np.uint64)
    for r in range(4):
        part = np.zeros(cfg.shots, dtype=np.uint64)
        T.run_tree(t, 128, leaf_begin=int(b[r]), leaf_end=int(b[r + 1]), out_slots=part)
        acc += part
    ref, edge = oracle_runs.run("C2b")
    _check_slots(acc, ref, edge, cfg.shots)


@pytest.mark.parametrize("name", ["C1", "C2b", "C3"])
def test_leaf_amplitudes_after_rollback(T, torch, oracle_runs, name):
    # the state after a DFS prefix of leaves (uncompute + re-anchor) equals the oracle replay of
    # the last leaf's core from |0..0>
    cfg = W.config(name)
    t = _tree(T, cfg)
    ot = oracle_runs.tree(name)
    nl = t.n_leaves
    rng = np.random.default_rng(3)
    picks = sorted({0, 1, nl - 1, *[int(x) for x in rng.integers(0, nl, size=3)]})
    refs = {l: ot.replay_leaf_core(l) for l in picks}
    for prec in (128, 64):
        for flags in (0, T.EXEC_NO_RESET, T.EXEC_NO_FUSE):
            for l in picks:
                d = dstate(torch, cfg.n, prec)
                lo = max(0, l - 40)
                T.run_tree(t, prec, d_state=d, leaf_begin=lo, leaf_end=l + 1, flags=flags | T.EXEC_NO_SAMPLE)
                torch.cuda.synchronize()
                err = np.abs(d.cpu().numpy() - refs[l]).max()
                assert err < TOL[prec], (prec, flags, l, err)


# ------------------------------------------------------------------ Adder leaves via the sparse oracle
def _sparse_leaf(ot, cfg, l):
    from oracle import sparse as SP
    tr, cnt, off = ot.leaf(l)
    psi = SP.replay(cfg.ops, SP.core_triples(tr, len(cfg.ops)), drop_below=1e-14)
    return psi, cnt, off, ot.terminal_mask(l)


def _sparse_slots(ot, cfg, l, psi, cnt, mask):
    from oracle import sparse as SP
    k, e = SP.sample(psi, cfg.seed, l, cnt, 1e-9, mask)
    return np.array(k, dtype=np.uint64), np.array(e, dtype=bool)


def _check_full_vector(torch, d, psi, tol):
    """max |gpu - oracle| over ALL 2^n entries: on the oracle's support, then zero elsewhere."""
    idx = torch.tensor(sorted(psi), dtype=torch.int64, device="cuda")
    ref = torch.tensor([psi[i] for i in sorted(psi)], dtype=torch.complex128, device="cuda")
    got = d[idx].to(torch.complex128)
    e1 = float((got - ref).abs().max().item())
    d.index_fill_(0, idx, 0)
    e2 = float(d.abs().max().item())
    assert max(e1, e2) < tol, (e1, e2)
    return max(e1, e2)


def test_c3_all_slots(T, torch, oracle_runs):
    # C3 (24q Adder, 190 leaves) in bench's launch configuration: EVERY draw vs the oracle (sparse
    # replay of each leaf's core + the oracle's sampler), edge draws bounded
    cfg = W.config("C3")
    t = _tree(T, cfg)
    slots, stats = T.run_tree(t, 128)
    ref, edge = oracle_runs.sparse_run("C3")
    _check_slots(slots, ref, edge, cfg.shots)
    assert stats["draws"] == cfg.shots


def test_c3_continued_batches(T, torch, oracle_runs):
    # bench.py's launch configuration at N = 1: the range split into contiguous batches, each call
    # continuing the DFS state the previous one left (TUSQ_EXEC_CONTINUE) -- the valid-set /
    # sums-only bookkeeping must hand over a whole, stored state at every call boundary
    cfg = W.config("C3")
    t = _tree(T, cfg)
    b = t.partition(5)
    d = dstate(torch, cfg.n, 128)
    slots = np.zeros(cfg.shots, dtype=np.uint64)
    for s_ in range(5):
        T.run_tree(t, 128, d_state=d, leaf_begin=int(b[s_]), leaf_end=int(b[s_ + 1]),
                   flags=T.EXEC_CONTINUE if s_ else 0, out_slots=slots)
    ref, edge = oracle_runs.sparse_run("C3")
    _check_slots(slots, ref, edge, cfg.shots)
    torch.cuda.synchronize()
    last = t.n_leaves - 1
    assert float(np.abs(d.cpu().numpy() - oracle_runs.tree("C3").replay_leaf_core(last)).max()) <= 1e-10


def test_c3_all_slots_c64(T, torch, oracle_runs):
    # the same at complex64 (fp64 CDF sums; edge window 1e-5, reading #17): exercises the c64 K5
    # path with live tiles, valid sets and sums-only sampling (replayed tiles) at 24 qubits
    cfg = W.config("C3")
    t = _tree(T, cfg)
    slots, stats = T.run_tree(t, 64)
    ref, edge = oracle_runs.sparse_run("C3", 1e-5)
    _check_slots(slots, ref, edge, cfg.shots)
    assert stats["draws"] == cfg.shots


def test_c3_all_slots_no_live(T, torch, oracle_runs):
    # the plain dense path (TUSQ_EXEC_NO_LIVE: every sweep visits the whole state, every sampled
    # state stored) gives the same slots as the oracle -- and so as the default path
    cfg = W.config("C3")
    t = _tree(T, cfg)
    slots, stats = T.run_tree(t, 128, flags=T.EXEC_NO_LIVE)
    ref, edge = oracle_runs.sparse_run("C3")
    _check_slots(slots, ref, edge, cfg.shots)
    d = dstate(torch, cfg.n, 128)
    T.run_tree(t, 128, d_state=d, leaf_begin=100, leaf_end=140, flags=T.EXEC_NO_LIVE | T.EXEC_NO_SAMPLE)
    torch.cuda.synchronize()
    assert float(np.abs(d.cpu().numpy() - oracle_runs.tree("C3").replay_leaf_core(139)).max()) <= 1e-10


def test_c4_spot_leaves(T, torch, oracle_runs):
    # C4 (30 qubits, 16 GiB c128) in bench's launch configuration (fused, hybrid re-anchor):
    # SURVEY 8(d)'s 9 spot-check leaves (all-I, first 2, last 2, 4 seeded) plus the 2 leaves of
    # largest support in a seeded sample.  For each: every amplitude after a fresh descent AND
    # after rollback from 5 DFS predecessors <= 1e-10, and the leaf's shot slots.
    from oracle import sparse as SP
    cfg = W.config("C4")
    t = _tree(T, cfg)
    ot = oracle_runs.tree("C4")
    nl = t.n_leaves
    assert nl == ot.n_leaves and t.leaf(0)[0] == []
    rng = np.random.default_rng(4)
    picks = {0, 1, 2, nl - 2, nl - 1, *[int(x) for x in rng.integers(3, nl - 2, size=4)]}
    sample = [int(x) for x in rng.integers(0, nl, size=300)]
    L = len(cfg.ops)
    support = sorted(sample, key=lambda l: -len(SP.replay(cfg.ops, SP.core_triples(ot.leaf(l)[0], L),
                                                           drop_below=1e-14)))
    picks |= set(support[:2])
    n = cfg.n
    d = dstate(torch, n, 128)
    slots = np.zeros(cfg.shots, dtype=np.uint64)
    for l in sorted(picks):
        psi, cnt, off, mask = _sparse_leaf(ot, cfg, l)
        if l == 0:
            assert list(psi) == [W.adder_expected_output(14)]   # the noiseless leaf: closed form
        for lo in (l, max(0, l - 5)):
            flags = 0 if lo == l else T.EXEC_NO_RESET
            T.run_tree(t, 128, d_state=d, leaf_begin=lo, leaf_end=l + 1, out_slots=slots, flags=flags)
            torch.cuda.synchronize()
            _check_full_vector(torch, d, psi, TOL[128])
        ref, edge = _sparse_slots(ot, cfg, l, psi, cnt, mask)
        assert ((slots[off:off + cnt] != ref) & ~edge).sum() == 0, l
        assert edge.sum() <= edge_budget(cnt)
    del d
    torch.cuda.empty_cache()


def test_run_tree_errors(T, torch):
    cfg = W.config("C1")
    t = _tree(T, cfg)
    d = dstate(torch, 2, 128)   # too small
    with pytest.raises(T.TusqError) as e:
        T.run_tree(t, 128, d_state=d)
    assert e.value.status == 6
    with pytest.raises(T.TusqError):
        T.run_tree(t, 32)
    with pytest.raises(T.TusqError):
        T.run_tree(t, 128, leaf_begin=5, leaf_end=3)
    with pytest.raises(T.TusqError) as e:
        T.run_tree(t, 128, fuse_qubits=10)
    assert e.value.status == 2
    with pytest.raises(ValueError):
        T.run_tree(t, 128, out_slots=np.zeros(10, dtype=np.uint64))


# ------------------------------------------------------------------ general Pauli channels (Eq. 2)
def test_qaoa_twirled_decoherence_slots(T, torch, oracle_runs):
    # Q13: the paper's QAOA at 13 qubits under Pauli-twirled decoherence on
    # every gate and a readout channel -- ECM -> DFTT -> sampling, slot for slot vs the oracle
    cfg = W.config("Q13")
    t = T.build_error_tree(cfg.n, cfg.ops, 0, 0, 0, cfg.shots, cfg.seed, pauli=cfg.noise.pauli)
    ref, edge = oracle_runs.run("Q13")
    for flags in (0, T.EXEC_NO_FUSE):
        slots, stats = T.run_tree(t, 128, flags=flags)
        _check_slots(slots, ref, edge, cfg.shots)
        assert stats["draws"] == cfg.shots


def test_random_asymmetric_channels_slots(T, torch, oracle):
    rng = np.random.default_rng(91)
    for trial in range(6):
        n = int(rng.integers(3, 15))
        ops = W.random_circuit(rng, n, int(rng.integers(20, 80)))
        chan = [tuple(float(x) for x in rng.dirichlet([1, 1, 1, 1])[:3] * 0.05) for _ in range(3)]
        t = T.build_error_tree(n, ops, 0, 0, 0, 2048, 100 + trial, pauli=chan)
        ot = oracle.Tree(n, ops, 0, 0, 0, 2048, 100 + trial, chan=chan)
        ref, edge = ot.run()
        slots, _ = T.run_tree(t, 128)
        _check_slots(slots, ref, edge, 2048)


def test_delta_study_matches_oracle(T, torch, oracle):
    # the fidelity-deviation study (scripts/delta_study.py) at small sizes:
    # the library's pruned / unpruned fidelities equal the oracle's (same slots up to edge draws)
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "delta_study", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts",
                                    "delta_study.py"))
    D = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(D)
    assert abs(D.delta(0.9, 0.8) - 0.1 / 1.7) < 1e-15          # SPEC S:503's worked example
    for family, n in (("bv", 6), ("adder", 6), ("bv", 10)):
        row = D.run(family, n, 4096, 3, 0.01)
        if family == "bv":
            _, ops = W.bv(n)
            ideal = W.bv_expected_output(n)
        else:
            _, ops = W.adder((n - 2) // 2)
            ideal = W.adder_expected_output((n - 2) // 2)
        for tag, prune in (("pruned", True), ("unpruned", False)):
            slots, edge = oracle.Tree(n, ops, 0.01, 0.01, 0.01, 4096, 3, prune=prune).run()
            f = float(np.mean(slots == np.uint64(ideal)))
            assert abs(row[f"f_{tag}"] - f) <= edge.sum() / 4096 + 1e-15, (family, n, tag)
