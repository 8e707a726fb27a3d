"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star): amplitudes max |err| <= 1e-10 (complex128) and <= 1e-4
(complex64); shot slots exact except draws within 1e-9 of a CDF edge (oracle-flagged), which are
counted and reported; ECM trees bit-exact (tests/test_lib_host.py).
"""
import numpy as np
import pytest

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
            assert np.abs(d.cpu().numpy() - ref).max() < TOL[prec] * 10, (trial, flags)
        # uncompute restores the state: forward then inverse
        d = dstate(torch, n, prec, st)
        T.apply_ops(d, n, prec, ops)
        T.apply_ops(d, n, prec, ops, flags=T.APPLY_INVERSE)
        torch.cuda.synchronize()
        assert np.abs(d.cpu().numpy() - st).max() < TOL[prec] * 10


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
    # shot parity on a dense random state: exact except oracle-flagged edge draws
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
        ref, edge = oracle.sample_state(st, n, 11, 3, nd, 1e-9 if prec == 128 else 1e-5)
        got = out.cpu().numpy().astype(np.uint64)
        bad = (got != ref) & ~edge
        assert bad.sum() == 0, (n, int(bad.sum()), int(edge.sum()))


def _cfg_tree(T, cfg):
    nz = cfg.noise
    return T.build_error_tree(cfg.n, cfg.ops, nz.p1, nz.p2, nz.p_meas, cfg.shots, cfg.seed)


@pytest.mark.parametrize("name", ["C1", "C2a", "C2b"])
@pytest.mark.parametrize("flags", [0, 0x1, 0x2, 0x3])
def test_run_tree_slots_match_oracle(T, torch, oracle, name, flags):
    # end to end: ECM -> DFTT with uncompute -> leaf sampling, slot for slot vs the oracle
    cfg = W.config(name)
    t = _cfg_tree(T, cfg)
    slots, stats = T.run_tree(t, 128, flags=flags)
    ot = oracle.Tree.from_config(cfg)
    ref, edge = ot.run()
    bad = (slots != ref) & ~edge
    assert bad.sum() == 0, (int(bad.sum()), int(edge.sum()), stats)
    assert stats["draws"] == cfg.shots and stats["leaves"] == t.n_leaves


@pytest.mark.parametrize("name", ["C1", "C2b", "C3"])
def test_leaf_amplitudes_after_rollback(T, torch, oracle, name):
    # the state after a DFS prefix of leaves (uncompute + re-anchor) equals the oracle replay of
    # the last leaf from |0..0>
    cfg = W.config(name)
    t = _cfg_tree(T, cfg)
    ot = oracle.Tree.from_config(cfg)
    nl = t.n_leaves
    rng = np.random.default_rng(3)
    picks = sorted({0, 1, nl - 1, *[int(x) for x in rng.integers(0, nl, size=3)]})
    for prec in (128, 64):
        for flags in (0, T.EXEC_NO_RESET, T.EXEC_NO_FUSE):
            for l in picks:
                d = dstate(torch, cfg.n, prec)
                lo = max(0, l - 40)
                T.run_tree(t, prec, d_state=d, leaf_begin=lo, leaf_end=l + 1, flags=flags | T.EXEC_NO_SAMPLE)
                torch.cuda.synchronize()
                ref = ot.replay_leaf(l)
                err = np.abs(d.cpu().numpy() - ref).max()
                assert err < TOL[prec], (prec, flags, l, err)


def test_c3_sampled_leaf_slots(T, torch, oracle):
    # C3 (24q) in the launch configuration bench uses: slots of sampled leaves vs the oracle
    cfg = W.config("C3")
    t = _cfg_tree(T, cfg)
    slots, _ = T.run_tree(t, 128)
    ot = oracle.Tree.from_config(cfg)
    rng = np.random.default_rng(1)
    for l in sorted({0, t.n_leaves - 1, *[int(x) for x in rng.integers(0, t.n_leaves, size=4)]}):
        _, cnt, off = ot.leaf(l)
        ref, edge = ot.sample_leaf(ot.replay_leaf(l), l)
        got = slots[off:off + cnt]
        assert ((got != ref) & ~edge).sum() == 0


def test_c4_full_size(T, torch, oracle):
    # C4 (30 qubits, 16 GiB c128) in bench's launch configuration (fused, hybrid re-anchor):
    # leaf 0 is the noiseless leaf -> closed form |0x26666664>; rollback over a DFS range equals
    # a fresh descent; one noisy leaf vs the oracle's full replay (amplitudes and its shot slots).
    cfg = W.config("C4")
    t = _cfg_tree(T, cfg)
    assert t.leaf(0)[0] == []
    n = cfg.n
    d = dstate(torch, n, 128)
    slots, _ = T.run_tree(t, 128, d_state=d, leaf_begin=0, leaf_end=1)
    idx = W.adder_expected_output(14)
    assert abs(complex(d[idx].item()) - 1) < 1e-12
    d[idx] = 0
    assert float(d.abs().max().item()) < 1e-12
    assert (slots[:t.leaf(0)[1]] == idx).all()
    # rollback over the last DFS leaves (errors from gate 25 on, Y/X frozen before T gates)
    # vs a fresh descent to the last leaf
    nl = t.n_leaves
    T.run_tree(t, 128, d_state=d, leaf_begin=nl - 6, leaf_end=nl, flags=T.EXEC_NO_SAMPLE | T.EXEC_NO_RESET)
    d2 = dstate(torch, n, 128)
    T.run_tree(t, 128, d_state=d2, leaf_begin=nl - 1, leaf_end=nl, flags=T.EXEC_NO_SAMPLE)
    torch.cuda.synchronize()
    assert float((d - d2).abs().max().item()) < 1e-10
    del d2
    # that noisy leaf against the oracle (full 2^30 replay on the host)
    ot = oracle.Tree.from_config(cfg)
    ref = ot.replay_leaf(nl - 1)
    got = d.cpu().numpy()
    assert np.abs(got - ref).max() < 1e-10
    out = torch.zeros(max(t.leaf(nl - 1)[1], 64), dtype=torch.int64, device="cuda")
    T.sample(d, n, 128, out.numel(), cfg.seed, nl - 1, out)
    r, edge = oracle.sample_state(ref, n, cfg.seed, nl - 1, out.numel())
    assert ((out.cpu().numpy().astype(np.uint64) != r) & ~edge).sum() == 0


def test_run_tree_errors(T, torch):
    cfg = W.config("C1")
    t = _cfg_tree(T, cfg)
    d = dstate(torch, 2, 128)   # too small
    with pytest.raises(T.TusqError) as e:
        T.run_tree(t, 128, d_state=d)
    assert e.value.status == 6
    with pytest.raises(T.TusqError):
        T.run_tree(t, 32)
    with pytest.raises(T.TusqError):
        T.run_tree(t, 128, leaf_begin=5, leaf_end=3)
