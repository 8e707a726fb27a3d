"""Sparse state-vector replay -- TEST INFRASTRUCTURE ONLY (see tusq_oracle.c's header).

The same definition as the dense oracle's replay (Eq. 1: every gate is a
matrix acting on its qubits' amplitude pairs; frozen Paulis are applied right before gate pos,
DESIGN.md readings #7, #12), but the state is a dict {basis index: amplitude} holding the
nonzero amplitudes only.  Adder leaves stay sparse (a basis state up to Toffoli cores that a
Pauli error leaves half-open), so a 30-qubit leaf replays in milliseconds here where the dense
oracle needs minutes; that is what lets the GPU tests check every amplitude of many full-size
C4 leaves.  Pinned against the dense oracle (tests/test_oracle_pins.py::test_sparse_replay_*):
random circuits over the full gate set, and the noiseless Adder closed form.

Plain Python: one gate at a time, in circuit order; no fusion, no reordering.
"""
from __future__ import annotations

import cmath
import math
from typing import Dict, List, Sequence, Tuple

from workloads import circuits as W

State = Dict[int, complex]

R2 = 1.0 / math.sqrt(2.0)


def _mat(kind: int, th: float, inverse: bool):
    """2x2 matrix [[a, b], [c, d]] of a one-qubit gate (readings: S:56 for RZ; P(t) = diag(1, e^it))."""
    if inverse:
        if kind in (W.RX, W.RY, W.RZ, W.P):
            th = -th
        kind = {W.S: W.SDG, W.SDG: W.S, W.T: W.TDG, W.TDG: W.T}.get(kind, kind)
    if kind == W.H:
        return (R2, R2, R2, -R2)
    if kind == W.X:
        return (0, 1, 1, 0)
    if kind == W.Y:
        return (0, -1j, 1j, 0)
    if kind == W.Z:
        return (1, 0, 0, -1)
    if kind == W.S:
        return (1, 0, 0, 1j)
    if kind == W.SDG:
        return (1, 0, 0, -1j)
    if kind == W.T:
        return (1, 0, 0, complex(R2, R2))
    if kind == W.TDG:
        return (1, 0, 0, complex(R2, -R2))
    if kind == W.RX:
        c, s = math.cos(th / 2), math.sin(th / 2)
        return (c, -1j * s, -1j * s, c)
    if kind == W.RY:
        c, s = math.cos(th / 2), math.sin(th / 2)
        return (c, -s, s, c)
    if kind == W.RZ:
        return (cmath.exp(-0.5j * th), 0, 0, cmath.exp(0.5j * th))
    if kind == W.P:
        return (1, 0, 0, cmath.exp(1j * th))
    if kind == W.I:
        return (1, 0, 0, 1)
    raise ValueError(kind)


def apply_gate(psi: State, g, inverse: bool = False) -> State:
    kind, q0, q1, th = g
    out: State = {}
    if kind == W.CX:   # |c t> -> |c, t ^ c>
        for i, a in psi.items():
            j = i ^ (1 << q1) if (i >> q0) & 1 else i
            out[j] = out.get(j, 0) + a
        return out
    if kind in (W.CZ, W.CP):
        ph = -1.0 if kind == W.CZ else cmath.exp(1j * (-th if inverse else th))
        for i, a in psi.items():
            out[i] = a * ph if ((i >> q0) & 1 and (i >> q1) & 1) else a
        return out
    a00, a01, a10, a11 = _mat(kind, th, inverse)
    b = 1 << q0
    for i, a in psi.items():
        if (i >> q0) & 1:   # input bit 1: contributes a01 to |0>, a11 to |1>
            i0, i1 = i ^ b, i
            u0, u1 = a01 * a, a11 * a
        else:
            i0, i1 = i, i | b
            u0, u1 = a00 * a, a10 * a
        if u0 != 0:
            out[i0] = out.get(i0, 0) + u0
        if u1 != 0:
            out[i1] = out.get(i1, 0) + u1
    return out


def replay(ops: Sequence[Tuple[int, int, int, float]], triples: Sequence[Tuple[int, int, int]], init: int = 0,
           drop_below: float = 0.0) -> State:
    """Replay a canonical leaf from |init>: at each pos the frozen Paulis of pos (ascending q),
    then gate pos; pos = len(ops) holds the terminal triples.  Amplitudes whose modulus falls to
    <= drop_below are removed (0.0: only exact zeros)."""
    psi: State = {init: 1.0 + 0j}
    L = len(ops)
    tr = sorted(triples)
    k = 0
    for pos in range(L + 1):
        while k < len(tr) and tr[k][0] == pos:
            _, q, p = tr[k]
            psi = apply_gate(psi, (p, q, 0, 0.0))
            k += 1
        if pos < L:
            psi = apply_gate(psi, ops[pos])
            psi = {i: a for i, a in psi.items() if abs(a) > drop_below}
    return psi


def core_triples(triples, L: int) -> List[Tuple[int, int, int]]:
    """A leaf's triples before the readout (pos < L): what its state vector executes (reading #7)."""
    return [t for t in triples if t[0] < L]


def sample(psi: State, seed: int, leaf: int, n_draws: int, edge_eps: float = 1e-9, mask: int = 0):
    """Inverse-CDF draws from |amp|^2 of a sparse state, exactly as the dense oracle's
    or_sample_state (reading #9): p_k = re*re + im*im, C(k) a Neumaier-compensated
    sequential sum in index order, draw j uses Philox counter (j, leaf_lo, leaf_hi, 0x53000000),
    t = ((x >> 11) 2^-53) C(N-1), outcome min{k : C(k) > t}; edge if within edge_eps of C(k-1)
    or C(k).  Zero amplitudes leave a Neumaier sum unchanged (sum + 0 = sum, compensation + 0),
    so summing the nonzero entries in index order gives the dense C(k) at every nonzero k, and
    min{k : C(k) > t} is always a nonzero entry.  Outcomes are XORed with `mask` (the leaf's
    readout flips, reading #7).  Returns (outcomes, edge flags) as lists."""
    import numpy as np

    from oracle import oracle as O
    keys = sorted(psi)
    cum = []
    s = comp = 0.0
    last_pos = -1
    for k in keys:
        a = psi[k]
        re, im = float(a.real), float(a.imag)
        pk = re * re + im * im
        tt = s + pk
        if abs(s) >= abs(pk):
            comp += (s - tt) + pk
        else:
            comp += (pk - tt) + s
        s = tt
        cum.append(s + comp)
        if pk > 0:
            last_pos = k
    T = s + comp
    key = [seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF]
    out, edge = [], []
    for j in range(n_draws):
        w = O.philox([j & 0xFFFFFFFF, leaf & 0xFFFFFFFF, (leaf >> 32) & 0xFFFFFFFF, 0x53000000], key)
        x = w[0] | (w[1] << 32)
        t = float(np.float64(x >> 11) * np.float64(2.0 ** -53)) * T
        hit = None
        prev = 0.0
        for k, c in zip(keys, cum):
            if c > t:
                hit = (k, min(t - prev, c - t) < edge_eps)
                break
            prev = c
        if hit is None:
            hit = (last_pos, True)
        out.append(hit[0] ^ mask)
        edge.append(hit[1])
    return out, edge
