"""ctypes wrapper of the C oracle (oracle/tusq_oracle.c) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module.  The product path (paper_2508_04880_b200/) never
does.  See tusq_oracle.c for the paper citations of every step.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import List, Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "tusq_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

OP_DTYPE = np.dtype([("kind", "<u4"), ("q0", "<u4"), ("q1", "<u4"), ("pad", "<u4"), ("theta", "<f8")])


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no FMA contraction)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-shared", "-fPIC",
                               "-o", tmp, SRC, "-lm"])
        os.replace(tmp, LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        u32p, u64p, dp = C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), C.POINTER(C.c_double)
        L.or_philox.argtypes = [u32p, u32p, u32p]
        L.or_site_table.restype = C.c_uint64
        L.or_site_table.argtypes = [C.c_uint32, C.c_void_p, C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_void_p]
        L.or_sample_er.restype = C.c_uint64
        L.or_sample_er.argtypes = [C.c_uint32, C.c_void_p, C.c_uint64, C.c_double, C.c_double, C.c_double,
                                   C.c_uint64, C.c_uint64, u32p, C.c_uint64]
        L.or_canonicalize.restype = C.c_uint32
        L.or_canonicalize.argtypes = [C.c_uint32, C.c_void_p, C.c_uint64, u32p, C.c_uint32, u32p, C.c_uint32]
        L.or_dfs_cmp.restype = C.c_int
        L.or_dfs_cmp.argtypes = [u32p, C.c_uint32, u32p, C.c_uint32]
        L.or_prune.argtypes = [u64p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, C.c_uint64,
                               u64p, C.POINTER(C.c_uint8), u64p]
        L.or_build.argtypes = [C.c_uint32, C.c_void_p, C.c_uint64, C.c_double, C.c_double, C.c_double,
                               C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int,
                               C.POINTER(C.c_void_p)]
        L.or_build_chan.argtypes = [C.c_uint32, C.c_void_p, C.c_uint64, dp, C.c_uint64, C.c_uint64, C.c_uint32,
                                    C.c_uint32, C.c_uint32, C.c_int, C.POINTER(C.c_void_p)]
        L.or_site_table_chan.restype = C.c_uint64
        L.or_site_table_chan.argtypes = [C.c_uint32, C.c_void_p, C.c_uint64, dp, C.c_void_p]
        L.or_twirl.argtypes = [C.c_double, C.c_double, C.c_double, dp]
        L.or_free.argtypes = [C.c_void_p]
        L.or_stats.argtypes = [C.c_void_p, u64p]
        L.or_leaf.restype = C.c_uint32
        L.or_leaf.argtypes = [C.c_void_p, C.c_uint64, u64p, u64p, u32p, C.c_uint32]
        L.or_serialize.restype = C.c_uint64
        L.or_serialize.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64]
        L.or_apply_gate.argtypes = [dp, C.c_uint32, C.c_void_p, C.c_int]
        L.or_replay.argtypes = [C.c_uint32, C.c_void_p, C.c_uint64, u32p, C.c_uint32, C.c_int, C.c_int, dp]
        L.or_replay_leaf.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, dp]
        L.or_replay_leaf_core.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, dp]
        L.or_terminal_mask.restype = C.c_uint64
        L.or_terminal_mask.argtypes = [C.c_void_p, C.c_uint64]
        L.or_sample_state.argtypes = [dp, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64, C.c_double,
                                      u64p, C.POINTER(C.c_uint8)]
        L.or_run.argtypes = [C.c_void_p, C.c_void_p, C.c_double, u64p, C.POINTER(C.c_uint8)]
        _lib = L
    return _lib


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def ops_array(ops: Sequence[Tuple[int, int, int, float]]) -> np.ndarray:
    a = np.zeros(max(len(ops), 1), dtype=OP_DTYPE)
    for i, (k, q0, q1, th) in enumerate(ops):
        a[i] = (k, q0, q1, 0, th)
    return a


def philox(ctr: Sequence[int], key: Sequence[int]) -> List[int]:
    c = np.array(ctr, dtype=np.uint32)
    k = np.array(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    lib().or_philox(_ptr(c, C.c_uint32), _ptr(k, C.c_uint32), _ptr(o, C.c_uint32))
    return [int(x) for x in o]


SITE_DTYPE = np.dtype([("pos", "<u4"), ("q", "<u4"), ("tI", "<u8"), ("tX", "<u8"), ("tY", "<u8"), ("tZ", "<u8")])


def site_table(n, ops, p1, p2, pm) -> np.ndarray:
    a = ops_array(ops)
    m = lib().or_site_table(n, a.ctypes.data, len(ops), p1, p2, pm, None)
    out = np.zeros(max(m, 1), dtype=SITE_DTYPE)
    lib().or_site_table(n, a.ctypes.data, len(ops), p1, p2, pm, out.ctypes.data)
    return out[:m]


def _chan_array(chan) -> np.ndarray:
    c = np.array([x for t in chan for x in t], dtype=np.float64)
    assert c.shape == (9,)
    return c


def site_table_chan(n, ops, chan) -> np.ndarray:
    """Sites for general Pauli channels chan = ((pX,pY,pZ) 1q, (..) 2q, (..) readout)."""
    a = ops_array(ops)
    c = _chan_array(chan)
    m = lib().or_site_table_chan(n, a.ctypes.data, len(ops), _ptr(c, C.c_double), None)
    out = np.zeros(max(m, 1), dtype=SITE_DTYPE)
    lib().or_site_table_chan(n, a.ctypes.data, len(ops), _ptr(c, C.c_double), out.ctypes.data)
    return out[:m]


def twirl(t: float, T1: float, T2: float):
    """Eq. 2: Pauli-twirled decoherence (pX, pY, pZ), or None when unphysical / invalid."""
    o = np.zeros(3)
    rc = lib().or_twirl(t, T1, T2, _ptr(o, C.c_double))
    return None if rc else tuple(float(x) for x in o)


def sample_er(n, ops, p1, p2, pm, seed, shot) -> List[Tuple[int, int]]:
    a = ops_array(ops)
    cap = 4096
    buf = np.zeros(2 * cap, dtype=np.uint32)
    hw = lib().or_sample_er(n, a.ctypes.data, len(ops), p1, p2, pm, seed, shot, _ptr(buf, C.c_uint32), cap)
    assert hw <= cap
    return [(int(buf[2 * i]), int(buf[2 * i + 1])) for i in range(hw)]


def canonicalize(n, ops, insertions: Sequence[Tuple[int, int, int]]) -> List[Tuple[int, int, int]]:
    """insertions: (pos, q, P) 'P right after gate pos' sorted by pos -> canonical triples."""
    a = ops_array(ops)
    ins = np.array([x for t in insertions for x in t] or [0], dtype=np.uint32)
    cap = 3 * n + len(insertions) + 8
    out = np.zeros(3 * cap, dtype=np.uint32)
    k = lib().or_canonicalize(n, a.ctypes.data, len(ops), _ptr(ins, C.c_uint32), len(insertions),
                              _ptr(out, C.c_uint32), cap)
    assert k <= cap
    return [(int(out[3 * i]), int(out[3 * i + 1]), int(out[3 * i + 2])) for i in range(k)]


def dfs_cmp(a, b) -> int:
    aa = np.array([x for t in a for x in t] or [0], dtype=np.uint32)
    bb = np.array([x for t in b for x in t] or [0], dtype=np.uint32)
    return lib().or_dfs_cmp(_ptr(aa, C.c_uint32), len(a), _ptr(bb, C.c_uint32), len(b))


def prune(counts, a_num=1, a_den=100, beta=100, enabled=True, seed=1):
    c = np.array(counts, dtype=np.uint64)
    oc = np.zeros(max(len(c), 1), dtype=np.uint64)
    cl = np.zeros(max(len(c), 1), dtype=np.uint8)
    st = np.zeros(4, dtype=np.uint64)
    lib().or_prune(_ptr(c, C.c_uint64), len(c), a_num, a_den, beta, int(enabled), seed,
                   _ptr(oc, C.c_uint64), _ptr(cl, C.c_uint8), _ptr(st, C.c_uint64))
    return oc[:len(c)], cl[:len(c)], dict(zip(["p0", "n_sig", "n_insig", "n_selected"], map(int, st)))


def apply_gate(state: np.ndarray, n: int, g, inverse=False):
    a = ops_array([g])
    assert state.dtype == np.complex128 and state.flags.c_contiguous
    rc = lib().or_apply_gate(state.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)), n, a.ctypes.data, int(inverse))
    assert rc == 0


def replay(n, ops, triples, before_gate=True, state: Optional[np.ndarray] = None) -> np.ndarray:
    a = ops_array(ops)
    tr = np.array([x for t in triples for x in t] or [0], dtype=np.uint32)
    init = state is None
    if state is None:
        state = np.zeros(1 << n, dtype=np.complex128)
    rc = lib().or_replay(n, a.ctypes.data, len(ops), _ptr(tr, C.c_uint32), len(triples), int(before_gate),
                         int(init), state.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)))
    assert rc == 0
    return state


def sample_state(state: np.ndarray, n: int, seed: int, leaf: int, n_draws: int, edge_eps: float = 1e-9):
    out = np.zeros(max(n_draws, 1), dtype=np.uint64)
    edge = np.zeros(max(n_draws, 1), dtype=np.uint8)
    lib().or_sample_state(state.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)), n, seed, leaf, n_draws,
                          edge_eps, _ptr(out, C.c_uint64), _ptr(edge, C.c_uint8))
    return out[:n_draws], edge[:n_draws].astype(bool)


class Tree:
    """The oracle's ECM + TEM tree (DFS-ordered leaves after pruning)."""

    STAT_NAMES = ["S1", "S2", "S3", "p0", "n_sig", "n_insig", "n_selected", "n_leaves", "n_ops"]

    def __init__(self, n, ops, p1, p2, pm, shots, seed, alpha=(1, 100), beta=100, prune=True, chan=None):
        """chan: None (depolarizing p1/p2 + readout bit flip pm) or three (pX, pY, pZ) triples for
        the 1q-gate, 2q-gate and readout sites (Eq. 2)."""
        self.n, self.ops, self.seed = n, list(ops), seed
        self._ops = ops_array(ops)
        h = C.c_void_p()
        if chan is not None:
            c = _chan_array(chan)
            rc = lib().or_build_chan(n, self._ops.ctypes.data, len(ops), _ptr(c, C.c_double), shots, seed,
                                     alpha[0], alpha[1], beta, int(prune), C.byref(h))
        else:
            rc = lib().or_build(n, self._ops.ctypes.data, len(ops), p1, p2, pm, shots, seed, alpha[0], alpha[1],
                                beta, int(prune), C.byref(h))
        if rc != 0:
            raise ValueError(f"or_build failed rc={rc}")
        self.h = h

    @classmethod
    def from_config(cls, cfg, prune=True):
        nz = cfg.noise
        return cls(cfg.n, cfg.ops, nz.p1, nz.p2, nz.p_meas, cfg.shots, cfg.seed, cfg.alpha, cfg.beta, prune,
                   chan=getattr(nz, "pauli", None))

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_free(self.h)
            self.h = None

    def stats(self) -> dict:
        o = np.zeros(9, dtype=np.uint64)
        lib().or_stats(self.h, _ptr(o, C.c_uint64))
        return dict(zip(self.STAT_NAMES, map(int, o)))

    @property
    def n_leaves(self) -> int:
        return self.stats()["n_leaves"]

    def leaf(self, l: int):
        cap = 4096
        buf = np.zeros(3 * cap, dtype=np.uint32)
        cnt, off = C.c_uint64(), C.c_uint64()
        k = lib().or_leaf(self.h, l, C.byref(cnt), C.byref(off), _ptr(buf, C.c_uint32), cap)
        assert k <= cap
        tr = [(int(buf[3 * i]), int(buf[3 * i + 1]), int(buf[3 * i + 2])) for i in range(k)]
        return tr, int(cnt.value), int(off.value)

    def serialize(self) -> bytes:
        size = lib().or_serialize(self.h, None, 0)
        buf = (C.c_uint8 * size)()
        lib().or_serialize(self.h, buf, size)
        return bytes(buf)

    def replay_leaf(self, l: int) -> np.ndarray:
        st = np.zeros(1 << self.n, dtype=np.complex128)
        rc = lib().or_replay_leaf(self.h, self._ops.ctypes.data, l, st.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)))
        assert rc == 0
        return st

    def replay_leaf_core(self, l: int) -> np.ndarray:
        """The state leaf l is sampled from: its triples before the readout only (reading #7)."""
        st = np.zeros(1 << self.n, dtype=np.complex128)
        rc = lib().or_replay_leaf_core(self.h, self._ops.ctypes.data, l,
                                       st.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)))
        assert rc == 0
        return st

    def terminal_mask(self, l: int) -> int:
        """Readout flips of leaf l (its terminal X triples) as a bit mask."""
        return int(lib().or_terminal_mask(self.h, l))

    def sample_leaf(self, core_state, l: int, edge_eps=1e-9):
        """Leaf l's draws from its core state (replay_leaf_core), flipped by its terminal mask."""
        _, cnt, _ = self.leaf(l)
        k, edge = sample_state(core_state, self.n, self.seed, l, cnt, edge_eps)
        return k ^ np.uint64(self.terminal_mask(l)), edge

    def run(self, edge_eps=1e-9):
        S = self.stats()["S1"]
        slots = np.zeros(S, dtype=np.uint64)
        edge = np.zeros(S, dtype=np.uint8)
        rc = lib().or_run(self.h, self._ops.ctypes.data, edge_eps, _ptr(slots, C.c_uint64), _ptr(edge, C.c_uint8))
        assert rc == 0
        return slots, edge.astype(bool)
