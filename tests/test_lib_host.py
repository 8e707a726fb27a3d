"""CPU tests of the C-ABI library: it loads, exports every declared symbol, and its host-side
ECM / tree / scheduler logic is bit-exact with the independent oracle (no device calls)."""
import hashlib
import os
import re

import numpy as np
import pytest

from workloads import circuits as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="session")
def lib():
    # build.py by path: the package import raises until libtusq.so exists
    import importlib.util
    spec = importlib.util.spec_from_file_location("_tusq_build", os.path.join(ROOT, "paper_2508_04880_b200", "build.py"))
    build = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(build)
    build.build()
    import paper_2508_04880_b200 as T
    return T


def test_library_exports_header_symbols(lib):
    hdr = open(os.path.join(ROOT, "include", "tusq.h")).read()
    declared = set(re.findall(r"\b(tusq_[a-z_]+)\s*\(", hdr))
    assert {"tusq_build_error_tree", "tusq_run_tree", "tusq_sample"} <= declared
    import ctypes
    so = ctypes.CDLL(lib.LIB_PATH)
    for name in declared:
        assert hasattr(so, name), name
    assert set(lib.EXPORTED) == declared
    assert "sm_100a" in lib.version()


def test_build_errors(lib):
    n, ops = W.ghz(3)
    with pytest.raises(lib.TusqError) as e:
        lib.build_error_tree(n, ops + [W.op(W.CX, 1, 1)], 0.01, 0.01, 0, 10, 1)
    assert e.value.status == 1 and "target" in str(e.value)
    with pytest.raises(lib.TusqError):
        lib.build_error_tree(n, ops + [W.op(W.H, 5)], 0.01, 0.01, 0, 10, 1)
    with pytest.raises(lib.TusqError):
        lib.build_error_tree(n, ops, 1.5, 0.01, 0, 10, 1)
    with pytest.raises(lib.TusqError):
        lib.build_error_tree(n, ops, 0.01, 0.01, 0, 0, 1)
    with pytest.raises(lib.TusqError):
        lib.build_error_tree(63, [], 0.01, 0.01, 0, 10, 1)
    with pytest.raises(lib.TusqError):
        lib.build_error_tree(n, ops, 0.01, 0.01, 0, 10, 1, beta=0)
    with pytest.raises(lib.TusqError):
        lib.build_error_tree(n, [(99, 0, 0, 0.0)], 0.01, 0.01, 0, 10, 1)


def _both(lib, oracle, n, ops, p1, p2, pm, shots, seed, beta=100, prune=True):
    a = lib.build_error_tree(n, ops, p1, p2, pm, shots, seed, beta=beta, prune=prune)
    b = oracle.Tree(n, ops, p1, p2, pm, shots, seed, beta=beta, prune=prune)
    return a, b


@pytest.mark.parametrize("name", ["C1", "C2a", "C2b", "C3", "C4"])
@pytest.mark.parametrize("seed", [1, 2])
def test_ecm_tree_bit_exact_configs(lib, oracle, name, seed):
    # ECM trees and tallies: bit-exact between the library's frame-based ECM and the oracle's
    # literal-stack ECM (north star), including pruning selection, DFS order and offsets.
    cfg = W.config(name, seed)
    a, b = _both(lib, oracle, cfg.n, cfg.ops, cfg.noise.p1, cfg.noise.p2, cfg.noise.p_meas, cfg.shots, seed)
    sa, sb = a.serialize(), b.serialize()
    assert len(sa) == len(sb)
    assert hashlib.sha256(sa).hexdigest() == hashlib.sha256(sb).hexdigest()


def test_ecm_bit_exact_random(lib, oracle):
    rng = np.random.default_rng(21)
    for trial in range(60):
        n = int(rng.integers(1, 7))
        ops = W.random_circuit(rng, n, int(rng.integers(1, 40)))
        p1, p2, pm = [float(x) for x in rng.choice([0.0, 0.01, 0.1, 0.4], size=3)]
        shots = int(rng.integers(1, 3000))
        seed = int(rng.integers(0, 1 << 62))
        beta = int(rng.integers(1, 30))
        prune = bool(rng.integers(0, 2))
        a, b = _both(lib, oracle, n, ops, p1, p2, pm, shots, seed, beta, prune)
        assert a.serialize() == b.serialize(), (trial, n, ops, p1, p2, pm, shots, seed, beta, prune)


def _events(ops, tr):
    L = len(ops)
    ev = []
    k = 0
    for pos in range(L + 1):
        while k < len(tr) and tr[k][0] == pos:
            ev.append(("P", tr[k][1], tr[k][2]))
            k += 1
        if pos < L:
            ev.append(("G", pos))
    return ev


def test_tree_info_matches_explicit_trie(lib):
    # |E| = number of ops on the edges of the prefix trie of leaf event streams;
    # DFTT fwd + inv = 2|E| - depth(last leaf) (P:329 counts every edge twice; the path to the
    # last leaf is never uncomputed); naive = sum of leaf lengths (P:333 T_naive).
    for name in ["C1", "C2a", "C3"]:
        cfg = W.config(name)
        t = lib.build_error_tree(cfg.n, cfg.ops, cfg.noise.p1, cfg.noise.p2, cfg.noise.p_meas, cfg.shots, cfg.seed)
        info = t.info()
        streams = [_events(cfg.ops, t.leaf(l)[0]) for l in range(info["n_leaves"])]
        trie = set()
        for s in streams:
            for d in range(1, len(s) + 1):
                trie.add(tuple(s[:d]))
        assert info["edges"] == len(trie)
        assert info["dftt_ops"] == 2 * info["edges"] - len(streams[-1])
        assert info["naive_ops"] == sum(len(s) for s in streams)
        assert info["S1"] >= info["S2"] >= info["S3"] >= info["n_leaves"]


def test_dftt_closed_forms_full_tree():
    # full b-ary tree of height h: |E| = b(b^h - 1)/(b - 1), N_l = b^h = (1 - 1/b)|E| + 1,
    # h = log_b((b-1)|E| + b) - 1, T_dftt = 2|E|, T_naive = N_l h.
    import math
    for b, h, E, Nl in [(4, 2, 20, 16), (2, 5, 62, 32)]:
        assert b * (b ** h - 1) // (b - 1) == E
        assert (1 - 1 / b) * E + 1 == Nl
        assert abs(math.log((b - 1) * E + b, b) - 1 - h) < 1e-12
        # explicit DFS over the full tree: every edge traversed twice
        leaves = [tuple((i // b ** j) % b for j in range(h)) for i in range(b ** h)]
        trie = {lf[:d] for lf in leaves for d in range(1, h + 1)}
        assert len(trie) == E and len(leaves) == Nl


def test_partition_contiguous_and_balanced(lib):
    cfg = W.config("C3")
    t = lib.build_error_tree(cfg.n, cfg.ops, cfg.noise.p1, cfg.noise.p2, cfg.noise.p_meas, cfg.shots, cfg.seed)
    nl = t.n_leaves
    for nr in (1, 2, 4, 8):
        b = t.partition(nr)
        assert b[0] == 0 and b[-1] == nl and np.all(np.diff(b.astype(np.int64)) >= 0)


def test_sharded_plan_only(lib):
    # sharded mode's host logic (no device): same scheduler as replica mode (gate applications,
    # leaves), global<->local exchanges only where a dense gate meets a global qubit.  Sharded mode
    # has no live tiles, so it keeps the gate-count reset rule of the plain dense path (NO_LIVE)
    for name in ("C2a", "C2b", "C3"):
        cfg = W.config(name)
        nz = cfg.noise
        t = lib.build_error_tree(cfg.n, cfg.ops, nz.p1, nz.p2, nz.p_meas, cfg.shots, cfg.seed)
        _, rep = lib.run_tree(t, 128, flags=lib.EXEC_PLAN_ONLY | lib.EXEC_NO_LIVE)
        for R in (2, 4, 8):
            _, s = lib.run_tree(t, 128, flags=lib.EXEC_PLAN_ONLY, comm=lib.Comm.local(R))
            assert s["gate_apps"] == rep["gate_apps"] and s["leaves"] == rep["leaves"]
            assert s["draws"] == cfg.shots
            assert s["exchanges"] > 0
    # a circuit of diagonal / CX-from-global / X gates never exchanges
    n = 8
    ops = [W.op(W.H, 0), W.op(W.CX, 7, 0), W.op(W.X, 7), W.op(W.T, 6), W.op(W.CZ, 6, 1), W.op(W.CP, 7, 6, 0.3)]
    t = lib.build_error_tree(n, ops, 0.0, 0.0, 0.0, 8, 1)
    _, s = lib.run_tree(t, 128, flags=lib.EXEC_PLAN_ONLY, comm=lib.Comm.local(4))
    assert s["exchanges"] == 0
    with pytest.raises(lib.TusqError):
        lib.Comm.local(3)


def test_general_pauli_channels_bit_exact(lib, oracle):
    # TUSQ_NOISE_PAULI (Eq. 2): library trees == oracle trees, bit for bit, for random
    # asymmetric channels on the 1q / 2q / readout site classes (incl. all-zero classes: no sites)
    rng = np.random.default_rng(44)
    for trial in range(40):
        n = int(rng.integers(1, 7))
        ops = W.random_circuit(rng, n, int(rng.integers(1, 40)))
        chan = []
        for c in range(3):
            if rng.integers(0, 4) == 0:
                chan.append((0.0, 0.0, 0.0))
            else:
                w = rng.dirichlet([1, 1, 1, 1]) * float(rng.choice([0.02, 0.3, 1.0]))
                chan.append(tuple(float(x) for x in w[:3]))
        shots, seed = int(rng.integers(1, 3000)), int(rng.integers(0, 1 << 62))
        prune = bool(rng.integers(0, 2))
        a = lib.build_error_tree(n, ops, 0, 0, 0, shots, seed, prune=prune, pauli=chan)
        b = oracle.Tree(n, ops, 0, 0, 0, shots, seed, prune=prune, chan=chan)
        assert a.serialize() == b.serialize(), (trial, chan)
    cfg = W.config("Q13")
    a = lib.build_error_tree(cfg.n, cfg.ops, 0, 0, 0, cfg.shots, cfg.seed, pauli=cfg.noise.pauli)
    b = oracle.Tree.from_config(cfg)
    assert a.serialize() == b.serialize()
    # depolarizing through the general interface is the same tree
    n, ops = W.qft(5)
    a = lib.build_error_tree(n, ops, 0.01, 0.02, 0.03, 2048, 3)
    b = lib.build_error_tree(n, ops, 0, 0, 0, 2048, 3, pauli=((0.01 / 3,) * 3, (0.02 / 3,) * 3, (0.03, 0, 0)))
    assert a.serialize() == b.serialize()
    with pytest.raises(lib.TusqError):
        lib.build_error_tree(n, ops, 0, 0, 0, 10, 1, pauli=((0.5, 0.4, 0.2), (0, 0, 0), (0, 0, 0)))


def test_twirl_decoherence_matches_oracle(lib, oracle):
    for (t, T1, T2) in [(1.0, 1.0, 1.0), (0.3, 2.0, 3.5), (0.0, 1.0, 1.0), (5.0, 1.0, 2.0), (0.02, 1.0, 1.0)]:
        assert lib.twirl_decoherence(t, T1, T2) == oracle.twirl(t, T1, T2)
    with pytest.raises(lib.TusqError):
        lib.twirl_decoherence(1.0, 1.0, 3.0)   # T2 > 2 T1
    with pytest.raises(lib.TusqError):
        lib.twirl_decoherence(-1.0, 1.0, 1.0)


def test_live_tile_plan(lib):
    # live tiles: after a reset the planner's support analysis bounds the
    # tiles a sweep visits -- the same sweeps and gate applications, far fewer bytes; a reset group
    # moves one tile (64 KiB); a noiseless circuit of diagonal gates after an X-load folds entirely
    cfg = W.config("C3")
    nz = cfg.noise
    t = lib.build_error_tree(cfg.n, cfg.ops, nz.p1, nz.p2, nz.p_meas, cfg.shots, cfg.seed)
    _, s = lib.run_tree(t, 128, flags=lib.EXEC_PLAN_ONLY)
    full = 2.0 * (1 << cfg.n) * 16
    assert s["sweeps"] > 0 and s["hbm_bytes"] < 0.7 * s["sweeps"] * full
    # the plain dense path (TUSQ_EXEC_NO_LIVE): every sweep over the whole state (and the gate-count
    # reset rule, so a slightly different schedule: live tiles make resets cheaper than uncomputes)
    _, d = lib.run_tree(t, 128, flags=lib.EXEC_PLAN_ONLY | lib.EXEC_NO_LIVE)
    assert d["leaves"] == s["leaves"] and d["resets"] <= s["resets"]
    assert d["hbm_bytes"] >= 0.5 * d["sweeps"] * full > s["hbm_bytes"]
    # one H on a low qubit after a reset: the reset group is one tile, written as one tile
    n = 20
    ops = [W.op(W.X, 15), W.op(W.H, 3)]
    t = lib.build_error_tree(n, ops, 0.0, 0.0, 0.0, 8, 1, prune=False)
    _, s = lib.run_tree(t, 128, flags=lib.EXEC_PLAN_ONLY)
    assert s["fused_launches"] == 1
    # the launch moves one 64 KiB tile; finish() writes the zeros outside it once (2^n x 16 B)
    assert s["hbm_bytes"] <= 4096 * 16 + (1 << n) * 16
