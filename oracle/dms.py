"""Density-matrix simulation for tiny n -- TEST INFRASTRUCTURE ONLY.

Independent of the C oracle and of the CUDA path: plain numpy, complex128.
rho' = U rho U^dagger for gates, rho' = sum_P p_P P rho P for Pauli channels
("rho' = sum_i K_i rho K_i^dagger", depolarizing expansion
(1-p) rho + p/3 (X rho X + Y rho Y + Z rho Z)); P(k) = <k|rho|k>.
Gate matrices are written out here from their textbook definitions, not shared
with any other module.
"""
from __future__ import annotations

import numpy as np

s2 = 1 / np.sqrt(2)
PAULIS = {
    0: np.eye(2, dtype=complex),
    1: np.array([[0, 1], [1, 0]], dtype=complex),
    2: np.array([[0, -1j], [1j, 0]], dtype=complex),
    3: np.array([[1, 0], [0, -1]], dtype=complex),
}


def mat1(kind: int, th: float) -> np.ndarray:
    c, s = np.cos(th / 2), np.sin(th / 2)
    return {
        0: PAULIS[0], 1: PAULIS[1], 2: PAULIS[2], 3: PAULIS[3],
        4: np.array([[1, 1], [1, -1]], dtype=complex) * s2,
        5: np.diag([1, 1j]), 6: np.diag([1, -1j]),
        7: np.diag([1, np.exp(1j * np.pi / 4)]), 8: np.diag([1, np.exp(-1j * np.pi / 4)]),
        9: np.array([[c, -1j * s], [-1j * s, c]]),
        10: np.array([[c, -s], [s, c]], dtype=complex),
        11: np.diag([np.exp(-1j * th / 2), np.exp(1j * th / 2)]),
        12: np.diag([1, np.exp(1j * th)]),
    }[kind].astype(complex)


def full_1q(n: int, q: int, u: np.ndarray) -> np.ndarray:
    """Embed a 1q matrix on qubit q (qubit 0 = least significant bit)."""
    m = np.array([[1.0]], dtype=complex)
    for j in range(n - 1, -1, -1):
        m = np.kron(m, u if j == q else np.eye(2))
    return m


def full_gate(n: int, g) -> np.ndarray:
    kind, q0, q1, th = g
    N = 1 << n
    if kind in (13, 14, 15):
        U = np.zeros((N, N), dtype=complex)
        for i in range(N):
            c, t = (i >> q0) & 1, (i >> q1) & 1
            if kind == 13:
                U[i ^ (c << q1), i] = 1
            elif kind == 14:
                U[i, i] = -1 if (c and t) else 1
            else:
                U[i, i] = np.exp(1j * th) if (c and t) else 1
        return U
    return full_1q(n, q0, mat1(kind, th))


def statevector(n: int, ops, insert_after=None, insert_before=None) -> np.ndarray:
    """Dense matrix-chain product from |0..0>, with optional Pauli
    insertions (pos, q, P) right after gate pos (pos = len(ops): at the end) or
    right before gate pos (pos = len(ops): at the end)."""
    psi = np.zeros(1 << n, dtype=complex)
    psi[0] = 1
    after, before = {}, {}
    for (pos, q, p) in (insert_after or []):
        after.setdefault(pos, []).append((q, p))
    for (pos, q, p) in (insert_before or []):
        before.setdefault(pos, []).append((q, p))
    for pos in range(len(ops) + 1):
        for (q, p) in before.get(pos, []):
            psi = full_1q(n, q, PAULIS[p]) @ psi
        if pos < len(ops):
            psi = full_gate(n, ops[pos]) @ psi
        for (q, p) in after.get(pos, []):
            psi = full_1q(n, q, PAULIS[p]) @ psi
    return psi


def channel(rho: np.ndarray, n: int, q: int, probs) -> np.ndarray:
    """Pauli channel (p_I, p_X, p_Y, p_Z) on qubit q."""
    out = np.zeros_like(rho)
    for p, w in enumerate(probs):
        if w:
            P = full_1q(n, q, PAULIS[p])
            out += w * (P @ rho @ P.conj().T)
    return out


def dms_run(n: int, ops, p1: float, p2: float, pm: float) -> np.ndarray:
    """Exact noisy output distribution: one depolarizing channel per (gate, qubit)
    after the gate (readings #1, #2) and a bit flip before readout (reading #4)."""
    N = 1 << n
    rho = np.zeros((N, N), dtype=complex)
    rho[0, 0] = 1
    for g in ops:
        U = full_gate(n, g)
        rho = U @ rho @ U.conj().T
        if g[0] in (13, 14, 15):
            if p2 > 0:
                for q in (g[1], g[2]):
                    rho = channel(rho, n, q, (1 - p2, p2 / 3, p2 / 3, p2 / 3))
        elif p1 > 0:
            rho = channel(rho, n, g[1], (1 - p1, p1 / 3, p1 / 3, p1 / 3))
    if pm > 0:
        for q in range(n):
            rho = channel(rho, n, q, (1 - pm, pm, 0, 0))
    return np.real(np.diag(rho)).copy()


def dms_run_chan(n: int, ops, chan1, chan2, chanm) -> np.ndarray:
    """Exact noisy output distribution for general Pauli channels (Eq. 2): chan1 =
    (pX, pY, pZ) after every 1q gate, chan2 on each qubit of every 2q gate, chanm before readout."""
    N = 1 << n
    rho = np.zeros((N, N), dtype=complex)
    rho[0, 0] = 1

    def probs(c):
        return (1 - sum(c), c[0], c[1], c[2])
    for g in ops:
        U = full_gate(n, g)
        rho = U @ rho @ U.conj().T
        if g[0] in (13, 14, 15):
            if any(chan2):
                for q in (g[1], g[2]):
                    rho = channel(rho, n, q, probs(chan2))
        elif any(chan1):
            rho = channel(rho, n, g[1], probs(chan1))
    if any(chanm):
        for q in range(n):
            rho = channel(rho, n, q, probs(chanm))
    return np.real(np.diag(rho)).copy()
