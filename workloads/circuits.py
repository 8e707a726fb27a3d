"""Seeded synthetic input generators shared by the oracle and the CUDA path.

This module holds circuits, noise settings and shot counts ONLY: no part of the
TUSQ method (no noise sampling, no commutation, no gate arithmetic) lives here.
Both `oracle/` and `paper_2508_04880_b200/` consume its op lists; neither
imports the other.

Op encoding (mirrors `include/tusq.h` `tusq_op`, 24 bytes):
    (kind, q0, q1, theta)   q0 = control for two-qubit gates, q1 = target.
Qubit 0 is the least-significant bit of the amplitude index.

Generators follow DESIGN.md readings #13 (Adder), #14 (QFT) and the paper's GHZ
description.
"""
from __future__ import annotations

import math
import struct
from dataclasses import dataclass, field
from typing import List, Tuple

# gate kinds -- PAPER.md P:211 (1q + CNOT basis), plus P, CZ, CP
I, X, Y, Z, H, S, SDG, T, TDG, RX, RY, RZ, P, CX, CZ, CP = range(16)
KIND_NAMES = ["I", "X", "Y", "Z", "H", "S", "SDG", "T", "TDG",
              "RX", "RY", "RZ", "P", "CX", "CZ", "CP"]
TWO_QUBIT = {CX, CZ, CP}
PARAM = {RX, RY, RZ, P, CP}

Op = Tuple[int, int, int, float]


def op(kind: int, q0: int, q1: int = 0, theta: float = 0.0) -> Op:
    return (int(kind), int(q0), int(q1), float(theta))


def pack_ops(ops: List[Op]) -> bytes:
    """Pack into the 24-byte C struct layout {u32 kind, q0, q1, pad; f64 theta}."""
    return b"".join(struct.pack("<IIIId", k, a, b, 0, t) for (k, a, b, t) in ops)


# ---------------------------------------------------------------- Adder (E2)
def ccx(a: int, b: int, t: int) -> List[Op]:
    """Toffoli in the 1q+CX basis, 15 gates (reading #13)."""
    return [op(H, t), op(CX, b, t), op(TDG, t), op(CX, a, t), op(T, t),
            op(CX, b, t), op(TDG, t), op(CX, a, t), op(T, b), op(T, t),
            op(H, t), op(CX, a, b), op(T, a), op(TDG, b), op(CX, a, b)]


def maj(x: int, y: int, w: int) -> List[Op]:
    return [op(CX, w, y), op(CX, w, x)] + ccx(x, y, w)


def uma(x: int, y: int, w: int) -> List[Op]:
    return ccx(x, y, w) + [op(CX, w, x), op(CX, x, y)]


def adder_operands(k: int) -> Tuple[int, int]:
    mask = (1 << k) - 1
    return 0x5555555555555555 & mask, mask


def adder(k: int) -> Tuple[int, List[Op]]:
    """Cuccaro ripple-carry adder (one ancilla), n = 2k+2.

    Layout (reading #13): q0 = c_in, b_i = 2i+1, a_i = 2i+2, z = 2k+1.
    Operands a = 0x5555.. & (2^k-1), b = 2^k-1 loaded with X gates
    (a-bit before b-bit per i).  L = 37 / 392 / 498 for k = 1 / 11 / 14.
    """
    n = 2 * k + 2
    a_val, b_val = adder_operands(k)

    def bq(i):
        return 2 * i + 1

    def aq(i):
        return 2 * i + 2
    z = 2 * k + 1
    ops: List[Op] = []
    for i in range(k):
        if (a_val >> i) & 1:
            ops.append(op(X, aq(i)))
        if (b_val >> i) & 1:
            ops.append(op(X, bq(i)))
    ops += maj(0, bq(0), aq(0))
    for i in range(1, k):
        ops += maj(aq(i - 1), bq(i), aq(i))
    ops.append(op(CX, aq(k - 1), z))
    for i in range(k - 1, 0, -1):
        ops += uma(aq(i - 1), bq(i), aq(i))
    ops += uma(0, bq(0), aq(0))
    return n, ops


def adder_expected_output(k: int) -> int:
    """Classical result index of the noiseless adder: b <- a+b (mod 2^k), z <- carry."""
    a_val, b_val = adder_operands(k)
    s = a_val + b_val
    idx = 0
    for i in range(k):
        if (a_val >> i) & 1:
            idx |= 1 << (2 * i + 2)
        if (s >> i) & 1:
            idx |= 1 << (2 * i + 1)
    if (s >> k) & 1:
        idx |= 1 << (2 * k + 1)
    return idx


# ---------------------------------------------------------------- GHZ (E3)
def ghz(n: int) -> Tuple[int, List[Op]]:
    """H on qubit 0 then CX(0, i) for i = 1..n-1."""
    return n, [op(H, 0)] + [op(CX, 0, i) for i in range(1, n)]


# ---------------------------------------------------------------- QFT (reading #14)
QFT_INPUT = 0x5A5A5A5A5A5A5A5A


def qft_input(n: int) -> int:
    return QFT_INPUT & ((1 << n) - 1)


def qft(n: int, native_cp: bool = False) -> Tuple[int, List[Op]]:
    """X-load of x, then for j = n-1..0: H(j), CP(pi/2^(j-k)) (control k, target j)
    for k = j-1..0; no final swaps.  Default CP is decomposed into the 1q+CX basis
    as P(t/2)_t, CX(k,j), P(-t/2)_j, CX(k,j), P(t/2)_k (circuit order)."""
    x = qft_input(n)
    ops: List[Op] = [op(X, q) for q in range(n) if (x >> q) & 1]
    for j in range(n - 1, -1, -1):
        ops.append(op(H, j))
        for k in range(j - 1, -1, -1):
            th = math.pi / (1 << (j - k))
            if native_cp:
                ops.append(op(CP, k, j, th))
            else:
                ops += [op(P, j, 0, th / 2), op(CX, k, j), op(P, j, 0, -th / 2),
                        op(CX, k, j), op(P, k, 0, th / 2)]
    return n, ops


# ---------------------------------------------------------------- QAOA
def qaoa(n: int, layers: int, seed: int = 1) -> Tuple[int, List[Op]]:
    """Supermarq-style QAOA block: H on every qubit, then per layer one parameterized
    single-qubit layer on all qubits (RX, then RZ) followed by CNOT entanglers (a linear chain).
    Angles are uniform in [0, 2 pi) from a seeded generator (the paper gives none)."""
    import numpy as np
    rng = np.random.default_rng(seed)
    ops: List[Op] = [op(H, q) for q in range(n)]
    for _ in range(layers):
        th = rng.uniform(0, 2 * math.pi, size=n)
        ph = rng.uniform(0, 2 * math.pi, size=n)
        ops += [op(RX, q, 0, float(th[q])) for q in range(n)]
        ops += [op(RZ, q, 0, float(ph[q])) for q in range(n)]
        ops += [op(CX, q, q + 1) for q in range(n - 1)]
    return n, ops


# ---------------------------------------------------------------- Bernstein-Vazirani
def bv_secret(n: int) -> int:
    return 0x2D2D2D2D2D2D2D2D & ((1 << (n - 1)) - 1)


def bv(n: int) -> Tuple[int, List[Op]]:
    """Bernstein-Vazirani on n-1 data qubits + ancilla n-1 (the delta study of P:509-516): X and H on
    the ancilla, H on the data, CX(i -> ancilla) for each secret bit, H on every qubit.  Noiseless
    output: the secret on the data qubits and 1 on the ancilla (bv_expected_output)."""
    s = bv_secret(n)
    a = n - 1
    ops: List[Op] = [op(X, a)] + [op(H, q) for q in range(n)]
    ops += [op(CX, q, a) for q in range(n - 1) if (s >> q) & 1]
    ops += [op(H, q) for q in range(n)]
    return n, ops


def bv_expected_output(n: int) -> int:
    return bv_secret(n) | (1 << (n - 1))


# ---------------------------------------------------------------- configs
@dataclass
class Noise:
    p1: float = 1e-3      # depolarizing after every 1q gate (paper convention 1-p, p/3 x3)
    p2: float = 1e-2      # depolarizing on each qubit of a 2q gate (reading #1)
    p_meas: float = 0.0   # bit flip before readout on every qubit (reading #4)
    # general Pauli channels (Eq. 2): ((pX,pY,pZ) 1q gates, (..) 2q-gate qubits, (..) readout);
    # when set, p1/p2/p_meas are ignored
    pauli: tuple = None


@dataclass
class Config:
    name: str
    n: int
    ops: List[Op]
    noise: Noise
    shots: int
    seed: int = 1
    alpha: Tuple[int, int] = (1, 100)   # P:336, alpha = 0.01 as a rational
    beta: int = 100
    meta: dict = field(default_factory=dict)


ADDER_NOISE = Noise(1e-3, 1e-2, 0.0)
MEAS_NOISE = Noise(1e-3, 1e-2, 1e-2)


def config(name: str, seed: int = 1) -> Config:
    if name == "C1":
        n, ops = adder(1)
        return Config("C1", n, ops, ADDER_NOISE, 1024, seed, meta={"k": 1})
    if name == "C2a":
        n, ops = ghz(16)
        return Config("C2a", n, ops, MEAS_NOISE, 8192, seed)
    if name == "C2b":
        n, ops = qft(16)
        return Config("C2b", n, ops, MEAS_NOISE, 8192, seed)
    if name == "C3":
        n, ops = adder(11)
        return Config("C3", n, ops, ADDER_NOISE, 8192, seed, meta={"k": 11})
    if name == "C4":
        n, ops = adder(14)
        return Config("C4", n, ops, ADDER_NOISE, 8192, seed, meta={"k": 14})
    if name == "C5":
        n, ops = qft(34, native_cp=True)
        return Config("C5", n, ops, MEAS_NOISE, 8192, seed)
    if name == "Q13":   # P:455 QAOA at its smallest size with twirled decoherence (Eq. 2) -- SURVEY 8(f)#4
        n, ops = qaoa(13, 2, seed)
        return Config("Q13", n, ops, TWIRL_NOISE, 8192, seed)
    raise KeyError(name)


# Eq. 2 twirled decoherence for an idle time t = T1 / 50, T2 = T1 (pX = pY = pZ =
# (1 - e^{-0.02}) / 4 each), composed by the caller into the 1q/2q/readout channels; the numbers
# are inputs here -- tusq_twirl_decoherence / the oracle's or_twirl compute the same map
TWIRL_NOISE = Noise(pauli=((0.004950331673311187, 0.004950331673311187, 0.004950331673311187),
                           (0.004950331673311187, 0.004950331673311187, 0.004950331673311187),
                           (0.01, 0.0, 0.0)))


def random_circuit(rng, n: int, n_gates: int, kinds=None) -> List[Op]:
    """Random circuit over the full gate set (seeded numpy Generator)."""
    kinds = kinds if kinds is not None else list(range(16))
    ops: List[Op] = []
    for _ in range(n_gates):
        k = int(rng.choice(kinds))
        if k in TWO_QUBIT:
            if n < 2:
                continue
            a, b = rng.choice(n, size=2, replace=False)
            ops.append(op(k, int(a), int(b), float(rng.uniform(-math.pi, math.pi)) if k in PARAM else 0.0))
        else:
            q = int(rng.integers(n))
            ops.append(op(k, q, 0, float(rng.uniform(-math.pi, math.pi)) if k in PARAM else 0.0))
    return ops
