"""Pins of the C oracle against things other than itself (CPU only).

Each test names what fixes the expected value: Random123/curand Philox KATs,
the paper's worked examples (PAPER.md P:<line>), closed forms, an independent
numpy density-matrix / matrix-chain simulator (oracle/dms.py), invariants and
brute force on tiny inputs.
"""
import itertools
import math

import numpy as np
import pytest

from oracle import dms
from workloads import circuits as W

PI, PX, PY, PZ = 0, 1, 2, 3


# ------------------------------------------------------------------ Philox (reading #9)
def test_philox_known_answers(oracle):
    # Random123 philox4x32-10 known-answer vectors (kat_vectors), the generator curand implements.
    assert oracle.philox([0, 0, 0, 0], [0, 0]) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert oracle.philox([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2) == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert oracle.philox([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0]) == \
        [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


# ------------------------------------------------------------------ channels / sites
def test_depolarizing_thresholds(oracle):
    # p = 0.1 -> I 90 %, X/Y/Z 10/3 % each
    n, ops = 1, [W.op(W.X, 0)]
    st = oracle.site_table(n, ops, 0.1, 0.0, 0.0)
    assert len(st) == 1
    s = st[0]
    assert int(s["tX"]) == int(s["tY"]) == int(s["tZ"]) == round(2 ** 32 / 30)
    assert int(s["tI"]) + 3 * int(s["tX"]) == 2 ** 32
    assert abs(int(s["tI"]) / 2 ** 32 - 0.9) < 1e-9
    # bit flip (1-p, p, 0, 0), p = 1 -> deterministic flip
    st = oracle.site_table(1, [], 0, 0, 1.0)
    assert int(st[0]["tX"]) == 2 ** 32 and int(st[0]["tI"]) == 0


def test_site_counts(oracle):
    # one site per (gate, acted qubit) (reading #1), measurement sites only when p_meas > 0
    for name, m in [("C1", 54), ("C2a", 47), ("C3", 569), ("C4", 723)]:
        cfg = W.config(name)
        assert len(oracle.site_table(cfg.n, cfg.ops, cfg.noise.p1, cfg.noise.p2, cfg.noise.p_meas)) == m
    # GHZ(2) with measurement -> 1 + 2 + 2 sites
    n, ops = W.ghz(2)
    assert len(oracle.site_table(n, ops, 0.01, 0.01, 0.01)) == 5


def test_er_sampler_marginals(oracle):
    # site marginals converge to (1-p, p/3, p/3, p/3); 4-sigma binomial band
    n, ops = 1, [W.op(W.H, 0)]
    p, shots = 0.3, 60000
    cnt = np.zeros(4)
    for s in range(shots):
        er = oracle.sample_er(n, ops, p, 0.0, 0.0, 7, s)
        cnt[er[0][1] if er else 0] += 1
    exp = np.array([1 - p, p / 3, p / 3, p / 3]) * shots
    sig = np.sqrt(exp * (1 - exp / shots))
    assert np.all(np.abs(cnt - exp) < 4 * sig), (cnt, exp)


def test_er_all_identity_frequency(oracle):
    # all-I frequency ~ (1-p)^M, via the tally of the tree builder
    n, ops = W.ghz(3)
    M = 1 + 2 * 2
    p = 0.05
    shots = 20000
    hw0 = sum(1 for s in range(shots) if not oracle.sample_er(n, ops, p, p, 0.0, 3, s))
    e = (1 - p) ** M * shots
    assert abs(hw0 - e) < 4 * math.sqrt(e * (1 - e / shots))


# ------------------------------------------------------------------ ECM worked examples
def test_fig_p186_commutation(oracle):
    # Fig. P:186: on H + CNOT, ER (X after H, II after CX) == (I after H, XX after CX)
    n, ops = 2, [W.op(W.H, 0), W.op(W.CX, 0, 1)]
    a = oracle.canonicalize(n, ops, [(0, 0, PX)])
    b = oracle.canonicalize(n, ops, [(1, 0, PX), (1, 1, PX)])
    assert a == b == [(2, 0, PX), (2, 1, PX)]


def test_fig_p193_rz_blocks_x(oracle):
    # Fig. P:193: a noisy X is not pushed through RZ(theta)
    n, ops = 1, [W.op(W.X, 0), W.op(W.RZ, 0, 0, 0.7)]
    assert oracle.canonicalize(n, ops, [(0, 0, PX)]) == [(1, 0, PX)]
    # ... but Z passes through RZ (rule 3) and is dropped before measurement (reading #7)
    assert oracle.canonicalize(n, ops, [(0, 0, PZ)]) == []


def test_rule6_y_on_target(oracle):
    # P:219 rule 6: Y on the CNOT target -> Z on control, Y on target.  Pin it through
    # blocking gates: H turns Z_c into X_c, then T blocks X_c and Y_t in place.
    n = 2
    ops = [W.op(W.I, 1), W.op(W.CX, 0, 1), W.op(W.H, 0), W.op(W.T, 0), W.op(W.T, 1)]
    assert oracle.canonicalize(n, ops, [(0, 1, PY)]) == [(3, 0, PX), (4, 1, PY)]
    # rule 4: X on the control -> X on both (both blocked by T)
    ops = [W.op(W.I, 0), W.op(W.CX, 0, 1), W.op(W.T, 0), W.op(W.T, 1)]
    assert oracle.canonicalize(n, ops, [(0, 0, PX)]) == [(2, 0, PX), (3, 1, PX)]
    # rule 1: two noisy X back to back cancel
    assert oracle.canonicalize(n, ops, [(0, 0, PX), (1, 0, PX), (1, 1, PX)]) == []


def test_commutation_soundness_random(oracle):
    # canonical placement == original placement in |amp|^2, checked with
    # the independent numpy matrix-chain simulator.
    rng = np.random.default_rng(11)
    for trial in range(300):
        n = int(rng.integers(1, 5))
        ops = W.random_circuit(rng, n, int(rng.integers(1, 24)))
        if not ops:
            continue
        L = len(ops)
        ins = []
        for pos in range(L + 1):
            qs = range(n) if pos == L else ([ops[pos][1], ops[pos][2]] if ops[pos][0] in W.TWO_QUBIT else [ops[pos][1]])
            for q in qs:
                if rng.random() < 0.35:
                    ins.append((pos, q, int(rng.integers(1, 4))))
        can = oracle.canonicalize(n, ops, ins)
        a = np.abs(dms.statevector(n, ops, insert_after=ins)) ** 2
        b = np.abs(dms.statevector(n, ops, insert_before=can)) ** 2
        assert np.abs(a - b).max() < 1e-12, (trial, ops, ins, can)


def test_monotonicity_S1_S2_S3(oracle):
    # Fig. P:40: S1 >= S2 >= S3 and shots conserved
    for name in ["C1", "C2a", "C3"]:
        cfg = W.config(name)
        t = oracle.Tree.from_config(cfg)
        st = t.stats()
        assert st["S1"] >= st["S2"] >= st["S3"] >= st["n_leaves"] > 0
        assert sum(t.leaf(l)[1] for l in range(st["n_leaves"])) == cfg.shots


def test_ghz_errors_reach_terminal_frame(oracle):
    # GHZ is H + CNOTs: every noisy Pauli either passes every gate or is dropped
    # (Z before readout) -- canonical leaves carry only terminal X.
    cfg = W.config("C2a")
    t = oracle.Tree.from_config(cfg, prune=False)
    for l in range(t.n_leaves):
        tr, _, _ = t.leaf(l)
        assert all(pos == len(cfg.ops) and p == PX for (pos, q, p) in tr)


# ------------------------------------------------------------------ pruning
def test_pruning_worked_example(oracle):
    # counts {800,100,50,42,5,3}, alpha = 0.01 -> threshold 8; 5 and 3 insignificant
    counts = [800, 100, 50, 42, 5, 3]
    oc, cl, st = oracle.prune(counts, 1, 100, beta=100)
    assert st["p0"] == 800 and st["n_sig"] == 4 and st["n_insig"] == 2
    assert list(cl) == [1, 1, 1, 1, 2, 2]
    assert list(oc) == counts      # |I| <= beta: gamma = 1, exact no-op
    # beta = 1: one of the two is kept and carries p_insig = 8 shots (P:340 scaling)
    oc, cl, st = oracle.prune(counts, 1, 100, beta=1)
    assert st["n_selected"] == 1 and sorted(cl[4:]) == [0, 2]
    assert oc[4:].sum() == 8 and oc.sum() == sum(counts)
    # P:415 bound with K = {5}: gamma = 8/5, p0 alpha (|I| + gamma |K|) / S = 0.0288
    gamma = 8 / 5
    assert abs(800 * 0.01 * (2 + gamma * 1) / 1000 - 0.0288) < 1e-15


def test_pruning_scaling_conserves_shots(oracle):
    rng = np.random.default_rng(5)
    for _ in range(50):
        counts = list(rng.integers(1, 40, size=int(rng.integers(1, 400))))
        counts[int(rng.integers(len(counts)))] = 3000
        oc, cl, st = oracle.prune(counts, 1, 100, beta=int(rng.integers(1, 120)), seed=int(rng.integers(1 << 30)))
        assert oc.sum() == sum(counts)
        for c, o, k in zip(counts, oc, cl):
            if k == 1:
                assert o == c and c * 100 >= 3000
            if k == 2:
                assert c * 100 < 3000 and o >= c


def _exact_mixture(oracle, t, n):
    P = np.zeros(1 << n)
    S = 0
    for l in range(t.n_leaves):
        tr, c, _ = t.leaf(l)
        P += c * np.abs(t.replay_leaf(l)) ** 2
        S += c
    return P / S


def test_pruning_bound_holds(oracle):
    # max_k |P(k) - P'(k)| <= p0 alpha (|I| + gamma |K|), counts normalized by S
    rng = np.random.default_rng(8)
    checked = 0
    for trial in range(12):
        n = 4
        ops = W.random_circuit(rng, n, 14)
        shots, seed = 3000, int(rng.integers(1, 1 << 30))
        full = oracle.Tree(n, ops, 0.08, 0.12, 0.05, shots, seed, beta=5, prune=False)
        pr = oracle.Tree(n, ops, 0.08, 0.12, 0.05, shots, seed, beta=5, prune=True)
        st = pr.stats()
        if st["n_insig"] <= 5:
            continue
        # gamma = p_insig / sum_K p (original counts of the kept insignificant leaves)
        full_counts = {tuple(full.leaf(l)[0]): full.leaf(l)[1] for l in range(full.n_leaves)}
        p0 = st["p0"]
        insig = [c for c in full_counts.values() if c * 100 < p0]
        kept = [full_counts[tuple(pr.leaf(l)[0])] for l in range(pr.n_leaves) if full_counts[tuple(pr.leaf(l)[0])] * 100 < p0]
        gamma = sum(insig) / sum(kept)
        bound = p0 * 0.01 * (len(insig) + gamma * len(kept)) / shots
        d = np.abs(_exact_mixture(oracle, full, n) - _exact_mixture(oracle, pr, n)).max()
        assert d <= bound + 1e-12, (d, bound)
        checked += 1
    assert checked >= 3


# ------------------------------------------------------------------ DFS order (reading #12)
def _slot_vector(tr, slots):
    d = {(p, q): P for (p, q, P) in tr}
    return tuple(d.get(s, 0) for s in slots)


def test_dfs_order_matches_trie_preorder(oracle):
    # DFS of the trie over slots (pos, q), children I < X < Y < Z, equals lexicographic
    # order of the per-slot Pauli vectors (brute force over the explicit slot list).
    cfg = W.config("C1")
    t = oracle.Tree.from_config(cfg)
    leaves = [t.leaf(l)[0] for l in range(t.n_leaves)]
    slots = sorted({(p, q) for tr in leaves for (p, q, _) in tr})
    vecs = [_slot_vector(tr, slots) for tr in leaves]
    assert vecs == sorted(vecs)
    assert len(set(vecs)) == len(vecs)
    # offsets are the exclusive prefix sum of counts
    offs = [t.leaf(l)[2] for l in range(t.n_leaves)]
    cnts = [t.leaf(l)[1] for l in range(t.n_leaves)]
    assert offs == list(np.concatenate([[0], np.cumsum(cnts)[:-1]]))


# ------------------------------------------------------------------ gate application (Eq. 1)
def test_gates_match_dense_matrix_chain(oracle):
    # per-gate loops == dense matrix-chain product, n <= 4
    rng = np.random.default_rng(3)
    for _ in range(200):
        n = int(rng.integers(1, 5))
        ops = W.random_circuit(rng, n, int(rng.integers(1, 20)))
        a = oracle.replay(n, ops, [])
        b = dms.statevector(n, ops)
        assert np.abs(a - b).max() < 1e-13


def test_gate_examples(oracle):
    # RZ(pi/2) = diag(e^{-i pi/4}, e^{i pi/4})
    for b, ph in [(0, -1), (1, 1)]:
        st = np.zeros(2, dtype=complex)
        st[b] = 1
        oracle.apply_gate(st, 1, W.op(W.RZ, 0, 0, math.pi / 2))
        assert abs(st[b] - np.exp(1j * ph * math.pi / 4)) < 1e-15
    # CNOT(0,1) (|00> + |01>)/sqrt2 -> (|00> + |11>)/sqrt2
    st = np.array([1, 1, 0, 0], dtype=complex) / math.sqrt(2)
    oracle.apply_gate(st, 2, W.op(W.CX, 0, 1))
    assert np.allclose(st, np.array([1, 0, 0, 1]) / math.sqrt(2), atol=1e-16)
    # X on qubit 0 of |00> -> |01> (index 1)
    st = np.array([1, 0, 0, 0], dtype=complex)
    oracle.apply_gate(st, 2, W.op(W.X, 0))
    assert st[1] == 1


def test_round_trip_inverse(oracle):
    # G then G^-1 restores the state up to rounding
    rng = np.random.default_rng(4)
    n = 5
    for _ in range(50):
        ops = W.random_circuit(rng, n, 30)
        st = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
        st /= np.linalg.norm(st)
        ref = st.copy()
        for g in ops:
            oracle.apply_gate(st, n, g)
        for g in reversed(ops):
            oracle.apply_gate(st, n, g, inverse=True)
        assert np.abs(st - ref).max() < 1e-13
    # X, CX, Z, Y, S round trips are bit-exact (pure moves, sign and re/im swaps)
    ops = [W.op(k, 0) for k in (W.X, W.Y, W.Z, W.S)] + [W.op(W.CX, 1, 2)]
    st = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    ref = st.copy()
    for g in ops:
        oracle.apply_gate(st, n, g)
    for g in reversed(ops):
        oracle.apply_gate(st, n, g, inverse=True)
    assert np.array_equal(st, ref)


# ------------------------------------------------------------------ closed forms
def test_ghz_closed_form(oracle):
    for n in (2, 5, 12):
        st = oracle.replay(*W.ghz(n), [])
        ref = np.zeros(1 << n, dtype=complex)
        ref[0] = ref[-1] = 1 / math.sqrt(2)
        assert np.abs(st - ref).max() < 1e-15


def test_adder_closed_form(oracle):
    # Noiseless Cuccaro adder is a classical permutation: output |a, a+b> with amplitude 1.
    for k in (1, 2, 3, 4, 6):
        n, ops = W.adder(k)
        st = oracle.replay(n, ops, [])
        idx = W.adder_expected_output(k)
        assert abs(st[idx] - 1) < 1e-13
        assert abs(np.linalg.norm(st) - 1) < 1e-13
    assert W.adder_expected_output(1) == 0xC
    assert W.adder_expected_output(11) == 0xE66664
    assert W.adder_expected_output(14) == 0x26666664
    # exhaustive operand pairs at k <= 3: replace the X-load prefix
    for k in (1, 2, 3):
        n, ops = W.adder(k)
        a0, b0 = W.adder_operands(k)
        body = ops[bin(a0).count("1") + bin(b0).count("1"):]
        for a in range(1 << k):
            for b in range(1 << k):
                load = []
                for i in range(k):
                    if (a >> i) & 1:
                        load.append(W.op(W.X, 2 * i + 2))
                    if (b >> i) & 1:
                        load.append(W.op(W.X, 2 * i + 1))
                st = oracle.replay(n, load + body, [])
                s = a + b
                idx = sum(((a >> i) & 1) << (2 * i + 2) | ((s >> i) & 1) << (2 * i + 1) for i in range(k))
                idx |= ((s >> k) & 1) << (2 * k + 1)
                assert abs(st[idx] - 1) < 1e-13


def test_qft_closed_form(oracle):
    # amplitude(y) = e^{2 pi i x rev_n(y) / 2^n} / sqrt(2^n) (reading #14)
    for native in (False, True):
        for n in (3, 6, 9):
            _, ops = W.qft(n, native)
            st = oracle.replay(n, ops, [])
            x = W.qft_input(n)
            y = np.arange(1 << n)
            rev = np.array([int(format(v, f"0{n}b")[::-1], 2) for v in y])
            ref = np.exp(2j * np.pi * ((x * rev) % (1 << n)) / (1 << n)) / math.sqrt(1 << n)
            assert np.abs(st - ref).max() < 1e-13


# ------------------------------------------------------------------ DMS equivalence
def _enumerate_exact(oracle, n, ops, p1, p2, pm, canonical):
    sites = oracle.site_table(n, ops, p1, p2, pm)
    choices = []
    for s in sites:
        if int(s["pos"]) == len(ops):
            choices.append([(PI, 1 - pm), (PX, pm)])
        else:
            p = p2 if ops[int(s["pos"])][0] in W.TWO_QUBIT else p1
            choices.append([(PI, 1 - p), (PX, p / 3), (PY, p / 3), (PZ, p / 3)])
    P = np.zeros(1 << n)
    for combo in itertools.product(*choices):
        w = np.prod([c[1] for c in combo])
        ins = [(int(s["pos"]), int(s["q"]), c[0]) for s, c in zip(sites, combo) if c[0] != PI]
        if canonical:
            st = oracle.replay(n, ops, oracle.canonicalize(n, ops, ins), before_gate=True)
        else:
            st = oracle.replay(n, ops, ins, before_gate=False)
        P += w * np.abs(st) ** 2
    return P


def test_brute_force_matches_dms(oracle):
    # sum over all ERs of Pr(ER) |psi_ER|^2 == diag(rho) of the DMS.
    n = 2
    ops = [W.op(W.H, 0), W.op(W.T, 0), W.op(W.H, 0), W.op(W.CX, 0, 1), W.op(W.T, 1), W.op(W.H, 1)]
    p1, p2, pm = 0.05, 0.1, 0.07
    ref = dms.dms_run(n, ops, p1, p2, pm)
    assert np.abs(ref - [0.35712378, 0.14287622, 0.35712378, 0.14287622]).max() < 1e-8
    for canonical in (False, True):
        P = _enumerate_exact(oracle, n, ops, p1, p2, pm, canonical)
        assert np.abs(P - ref).max() < 1e-12


def test_noisy_ghz2_closed_form():
    # GHZ-2 under p2 on both CX qubits and p_meas: f = 2 p2 / 3, f <- f(1-pm) + (1-f) pm,
    # P(01) = P(10) = f (1-f) (independent of p1).
    p1, p2, pm = 1e-3, 1e-2, 0.0
    n, ops = W.ghz(2)
    P = dms.dms_run(n, ops, p1, p2, pm)
    f = 2 * p2 / 3
    assert abs(P[1] - f * (1 - f)) < 1e-15 and abs(P[1] - 0.00662222) < 1e-8
    pm = 0.02
    P = dms.dms_run(n, ops, p1, p2, pm)
    f = f * (1 - pm) + (1 - f) * pm
    assert abs(P[2] - f * (1 - f)) < 1e-15


@pytest.mark.parametrize("family", ["adder", "ghz", "qft"])
def test_pipeline_tvd_to_dms(oracle, family):
    # P:112 (trajectory average -> DMS as S grows): seed-fixed tally + commutation + DFS
    # pipeline vs DMS, TVD <= 0.01.  Pruning is off here: with beta = 100 its
    # resampling error (~p_insig/sqrt(beta), reading #10) exceeds 0.01 at p = 1 %;
    # pruning is pinned by its own bound in test_pruning_bound_holds.
    if family == "adder":
        n, ops = W.adder(1)
    elif family == "ghz":
        n, ops = W.ghz(4)
    else:
        n, ops = W.qft(4)
    p1, p2, pm = 0.01, 0.01, 0.01
    ref = dms.dms_run(n, ops, p1, p2, pm)
    t = oracle.Tree(n, ops, p1, p2, pm, 200000, 2024, prune=False)
    slots, edge = t.run()
    hist = np.bincount(slots.astype(np.int64), minlength=1 << n) / len(slots)
    assert 0.5 * np.abs(hist - ref).sum() <= 0.01


# ------------------------------------------------------------------ sampling
def test_sampling_examples(oracle):
    # |01> -> every draw is index 1
    st = np.zeros(4, dtype=complex)
    st[1] = 1
    out, edge = oracle.sample_state(st, 2, 1, 0, 100)
    assert np.all(out == 1) and not edge.any()
    # (|0> + |1>)/sqrt2, 10^5 draws within 4 sigma of 1/2
    st = np.array([1, 1], dtype=complex) / math.sqrt(2)
    out, _ = oracle.sample_state(st, 1, 9, 3, 100000)
    assert abs(int(out.sum()) - 50000) < 4 * math.sqrt(25000)
    # zero-probability outcomes are never drawn (strict C(k) > t)
    st = np.array([0, 0.6, 0, 0.8], dtype=complex)
    out, _ = oracle.sample_state(st, 2, 2, 0, 20000)
    assert set(np.unique(out)) <= {1, 3}
    assert abs((out == 3).mean() - 0.64) < 0.02


# ------------------------------------------------------------------ readout relabel (reading #7)
def test_terminal_flips_are_readout_relabels(oracle):
    # measurement noise = an X right before readout.  The oracle samples a leaf from
    # its core state (triples before the readout) and XORs the drawn bitstrings with the leaf's
    # terminal X mask.  Pin: |core|^2 permuted by the mask equals |full replay|^2 EXACTLY (X is a
    # pure permutation), and every slot of or_run is the core draw XOR the mask.
    cfg = W.config("C2a")
    nz = cfg.noise
    n, ops = W.ghz(6)
    t = oracle.Tree(n, ops, nz.p1, nz.p2, 0.05, 4096, 7)
    idx = np.arange(1 << n)
    seen = 0
    for l in range(t.n_leaves):
        tr, cnt, off = t.leaf(l)
        mask = t.terminal_mask(l)
        expect = 0
        for (pos, q, p) in tr:
            if pos == len(ops):
                assert p == 1          # terminal triples are X flips only (Z dropped)
                expect ^= 1 << q
        assert mask == expect
        seen += mask != 0
        full = np.abs(t.replay_leaf(l)) ** 2
        core = np.abs(t.replay_leaf_core(l)) ** 2
        assert np.array_equal(full, core[idx ^ mask])
    assert seen > 0
    slots, edge = t.run()
    for l in range(t.n_leaves):
        _, cnt, off = t.leaf(l)
        k, e = oracle.sample_state(t.replay_leaf_core(l), n, 7, l, cnt)
        assert np.array_equal(slots[off:off + cnt], k ^ np.uint64(t.terminal_mask(l)))


# ------------------------------------------------------------------ sparse replay (oracle/sparse.py)
def test_sparse_replay_matches_dense_oracle(oracle):
    # the dict-based replay equals the dense oracle's replay (same definition, Eq. 1) on
    # random circuits over the full gate set with random frozen Paulis, forward and inverse gates
    from oracle import sparse as SP
    rng = np.random.default_rng(31)
    for trial in range(30):
        n = int(rng.integers(2, 8))
        ops = W.random_circuit(rng, n, int(rng.integers(5, 60)))
        L = len(ops)
        triples = sorted({(int(rng.integers(0, L + 1)), int(rng.integers(n)), int(rng.integers(1, 4)))
                          for _ in range(int(rng.integers(0, 6)))})
        dense = oracle.replay(n, ops, triples)
        sp = SP.replay(ops, triples)
        got = np.zeros(1 << n, dtype=complex)
        for i, a in sp.items():
            got[i] = a
        assert np.abs(got - dense).max() < 1e-13, trial
        # inverse gates: G^-1 G = I on a random basis state
        i0 = int(rng.integers(1 << n))
        st = {i0: 1.0 + 0j}
        for g in ops:
            st = SP.apply_gate(st, g)
        for g in reversed(ops):
            st = SP.apply_gate(st, g, inverse=True)
        back = np.zeros(1 << n, dtype=complex)
        for i, a in st.items():
            back[i] = a
        ref = np.zeros(1 << n, dtype=complex)
        ref[i0] = 1
        assert np.abs(back - ref).max() < 1e-12


def test_sparse_replay_adder_closed_form():
    # noiseless Cuccaro adder (reading #13): a single basis state with amplitude 1; with the
    # 1e-14 rounding-residue cut the support stays one entry through all 498 gates at 30 qubits
    from oracle import sparse as SP
    for k in (1, 3, 11, 14):
        n, ops = W.adder(k)
        st = SP.replay(ops, [], drop_below=1e-14)
        assert list(st) == [W.adder_expected_output(k)]
        assert abs(st[W.adder_expected_output(k)] - 1) < 1e-13


def test_sparse_sampler_matches_dense_sampler(oracle):
    # oracle/sparse.sample over the nonzero entries == or_sample_state over the dense vector
    # (zeros leave the compensated CDF unchanged), draw for draw incl. edge flags
    from oracle import sparse as SP
    rng = np.random.default_rng(12)
    for trial in range(20):
        n = int(rng.integers(1, 11))
        N = 1 << n
        st = np.zeros(N, dtype=complex)
        nz = rng.choice(N, size=int(rng.integers(1, min(N, 40) + 1)), replace=False)
        st[nz] = rng.normal(size=len(nz)) + 1j * rng.normal(size=len(nz))
        st /= np.linalg.norm(st)
        seed, leaf, nd = int(rng.integers(1 << 40)), int(rng.integers(1 << 33)), int(rng.integers(1, 300))
        ref, redge = oracle.sample_state(st, n, seed, leaf, nd, 1e-3)
        sp = {int(i): complex(st[i]) for i in nz}
        got, gedge = SP.sample(sp, seed, leaf, nd, 1e-3)
        assert np.array_equal(np.array(got, dtype=np.uint64), ref), trial
        assert np.array_equal(np.array(gedge), redge), trial


# ------------------------------------------------------------------ general Pauli channels (Eq. 2)
def test_twirl_closed_forms(oracle):
    # pX = pY = (1 - e^{-t/T1})/4, pZ = (1 - e^{-t/T2})/2 - (1 - e^{-t/T1})/4
    c = (1 - math.exp(-1)) / 4                      # t = T1 = T2: all three equal, ~0.158
    assert np.allclose(oracle.twirl(1.0, 1.0, 1.0), (c, c, c), atol=1e-15, rtol=0) and abs(c - 0.158) < 1e-3
    px, py, pz = oracle.twirl(3.0, 3.0, 6.0)        # T2 = 2 T1, t = T1
    assert px == py and abs(pz - ((1 - math.exp(-0.5)) / 2 - (1 - math.exp(-1)) / 4)) < 1e-15
    assert oracle.twirl(0.0, 1.0, 1.0) == (0.0, 0.0, 0.0)
    assert oracle.twirl(1.0, 1.0, 3.0) is None      # T2 > 2 T1: p_Z < 0, unphysical
    assert W.TWIRL_NOISE.pauli[0] == oracle.twirl(0.02, 1.0, 1.0)   # the Q13 config's numbers


def _enumerate_exact_chan(oracle, n, ops, chan, canonical):
    sites = oracle.site_table_chan(n, ops, chan)
    choices = []
    for s in sites:
        pos = int(s["pos"])
        c = chan[2] if pos == len(ops) else (chan[1] if ops[pos][0] in W.TWO_QUBIT else chan[0])
        choices.append([(p, w) for p, w in ((PI, 1 - sum(c)), (PX, c[0]), (PY, c[1]), (PZ, c[2])) if w > 0])
    P = np.zeros(1 << n)
    for combo in itertools.product(*choices):
        w = np.prod([c[1] for c in combo])
        ins = [(int(s["pos"]), int(s["q"]), c[0]) for s, c in zip(sites, combo) if c[0] != PI]
        if canonical:
            st = oracle.replay(n, ops, oracle.canonicalize(n, ops, ins), before_gate=True)
        else:
            st = oracle.replay(n, ops, ins, before_gate=False)
        P += w * np.abs(st) ** 2
    return P


def test_brute_force_general_channel_matches_dms(oracle):
    # P:139-147 + SPEC S:405 with NON-depolarizing channels (asymmetric pX/pY/pZ, a readout channel
    # with Y and Z parts): sum over all ERs of Pr(ER)|psi_ER|^2 == diag(rho), for the raw and the
    # canonical (commuted) Pauli placement; then the sampling pipeline converges to it
    n = 2
    ops = [W.op(W.H, 0), W.op(W.T, 0), W.op(W.H, 0), W.op(W.CX, 0, 1), W.op(W.RZ, 1, 0, 0.7), W.op(W.H, 1)]
    chan = ((0.05, 0.01, 0.08), (0.02, 0.09, 0.03), (0.06, 0.02, 0.04))
    ref = dms.dms_run_chan(n, ops, *chan)
    assert abs(ref.sum() - 1) < 1e-12
    for canonical in (False, True):
        P = _enumerate_exact_chan(oracle, n, ops, chan, canonical)
        assert np.abs(P - ref).max() < 1e-12
    t = oracle.Tree(n, ops, 0, 0, 0, 200000, 77, prune=False, chan=chan)
    slots, _ = t.run()
    hist = np.bincount(slots.astype(np.int64), minlength=1 << n) / len(slots)
    assert 0.5 * np.abs(hist - ref).sum() <= 0.01


def test_depolarizing_is_the_symmetric_pauli_channel(oracle):
    # the depolarizing site table (p/3, p/3, p/3) and bit flip (p, 0, 0) equal the general form
    n, ops = W.qft(4)
    a = oracle.site_table(n, ops, 0.01, 0.02, 0.03)
    b = oracle.site_table_chan(n, ops, ((0.01 / 3,) * 3, (0.02 / 3,) * 3, (0.03, 0.0, 0.0)))
    assert np.array_equal(a, b)
    t1 = oracle.Tree(n, ops, 0.01, 0.02, 0.03, 4096, 5)
    t2 = oracle.Tree(n, ops, 0, 0, 0, 4096, 5, chan=((0.01 / 3,) * 3, (0.02 / 3,) * 3, (0.03, 0.0, 0.0)))
    assert t1.serialize() == t2.serialize()
