#!/usr/bin/env python
"""Per-kernel HBM bandwidth at n = 30: K1 dense 1q at q = 0, 1-4, >= 5; K2 diagonal;
K3 CX / CZ; K4 Pauli string; K5 fused group (one Adder group); K6 block sums + draws; K7 init.
Each kernel is launched through the C ABI (tusq_apply_ops / tusq_init_basis / tusq_sample) and
timed with CUDA events on the launching stream after warm-up; achieved = algorithmic bytes / time.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2508_04880_b200 as T  # noqa: E402
from workloads import circuits as W  # noqa: E402


def timeit(fn, reps=5, warm=2):
    s = torch.cuda.current_stream()
    for _ in range(warm):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps


def main():
    n = int(os.environ.get("KB_N", "30"))
    prec = int(os.environ.get("KB_PREC", "128"))
    s = 16 if prec == 128 else 8
    N = 1 << n
    dt = torch.complex128 if prec == 128 else torch.complex64
    st = torch.zeros(N, dtype=dt, device="cuda")
    T.init_basis(st, n, prec, 0)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    rows = []

    def rec(name, bytes_, sec):
        gbs = bytes_ / sec / 1e9
        rows.append({"kernel": name, "ms": sec * 1e3, "GB/s": round(gbs, 1), "frac": round(gbs / peak, 3)})

    stream = torch.cuda.current_stream()
    U = T.APPLY_UNFUSED
    for q in (0, 1, 3, 5, 12, n - 1):
        rec(f"K1 H q={q}", 2 * N * s, timeit(lambda: T.apply_ops(st, n, prec, [W.op(W.H, q)], U, stream)))
    rec("K1 RX q=7", 2 * N * s, timeit(lambda: T.apply_ops(st, n, prec, [W.op(W.RX, 7, 0, 0.3)], U, stream)))
    for q in (0, 9):
        rec(f"K2 T q={q}", N * s, timeit(lambda: T.apply_ops(st, n, prec, [W.op(W.T, q)], U, stream)))
    rec("K2 RZ q=9", 2 * N * s, timeit(lambda: T.apply_ops(st, n, prec, [W.op(W.RZ, 9, 0, 0.3)], U, stream)))
    rec("K3 CX 3->17", N * s, timeit(lambda: T.apply_ops(st, n, prec, [W.op(W.CX, 3, 17)], U, stream)))
    rec("K3 CX 0->1", N * s, timeit(lambda: T.apply_ops(st, n, prec, [W.op(W.CX, 0, 1)], U, stream)))
    rec("K3 CZ 4,20", N * s / 2, timeit(lambda: T.apply_ops(st, n, prec, [W.op(W.CZ, 4, 20)], U, stream)))
    rec("K4 XYZ string", 2 * N * s,
        timeit(lambda: T.apply_ops(st, n, prec, [W.op(W.X, 2), W.op(W.Y, 11), W.op(W.Z, 25)], U, stream)))
    rec("K4 Z string", N * s, timeit(lambda: T.apply_ops(st, n, prec, [W.op(W.Z, 5), W.op(W.Z, 26)], U, stream)))
    # one fused Adder group (4 MAJ blocks on qubits 10..18) = one sweep
    _, ops = W.adder(14)
    grp = [g for g in ops if g[0] != W.X][4 * 17: 8 * 17]
    rec(f"K5 fused ({len(grp)} gates)", 2 * N * s, timeit(lambda: T.apply_ops(st, n, prec, grp, 0, stream)))
    # K5 cost anatomy: the bare sweep, register work without / with one transpose
    variants = {
        "K5 sweep (1 diagonal)": [W.op(W.T, 5)],
        "K5 10 H, 1 phase": [W.op(W.H, q) for q in (3, 4, 5, 6, 7)] * 2,
        "K5 9 H, 2 phases": [W.op(W.H, q) for q in (3, 4, 5, 6, 7, 8, 9, 10, 11)],
        "K5 15 H, 3 phases": [W.op(W.H, q) for q in (3, 4, 5, 6, 7, 8, 9, 10, 11, 3, 4, 5, 6, 7, 8)],
        "K5 20 H, 4 phases": [W.op(W.H, q) for q in (3, 4, 5, 6, 7, 8, 9, 10, 11, 3, 4, 5, 6, 7, 8, 9, 10, 11, 3, 4)],
        "K5 5 H on 12-16 (tile span 2^17)": [W.op(W.H, q) for q in (12, 13, 14, 15, 16)],
        "K5 5 H on 20-24 (tile span 2^25)": [W.op(W.H, q) for q in (20, 21, 22, 23, 24)],
        "K5 5 H on 25-29 (tile span 2^30)": [W.op(W.H, q) for q in (25, 26, 27, 28, 29)],
        "K5 8 DK (T/CX runs), 1 phase": [g for q in (3, 5) for g in
                                         (W.op(W.CX, q, q + 1), W.op(W.T, q + 1), W.op(W.CX, q, q + 1),
                                          W.op(W.TDG, q))] * 4,
        "K5 4 Toffoli (CU records)": [g for g in W.adder(14)[1] if g[0] != W.X][4 * 17 + 2: 4 * 17 + 17],
        # tile span vs transposes: 9 H over 9 consecutive qubits, 2 phases (pages per tile 1 / 8 / 512)
        "K5 9 H on 8-16, 2 phases": [W.op(W.H, q) for q in range(8, 17)],
        "K5 9 H on 14-22, 2 phases": [W.op(W.H, q) for q in range(14, 23)],
        "K5 9 H on 20-28, 2 phases": [W.op(W.H, q) for q in range(20, 29)],
    }
    gx = [g for g in W.adder(14)[1] if g[0] != W.X]
    for k in (8, 9, 10):
        variants[f"K5 4 MAJ on qubits {2 * k}-{2 * k + 8}"] = gx[k * 17:(k + 4) * 17]
    for name, g in variants.items():
        rec(name, 2 * N * s, timeit(lambda: T.apply_ops(st, n, prec, g, 0, stream)))
    # the same groups launched alternately (as in a replay): per-launch times
    ga, gb = gx[4 * 17:8 * 17], gx[9 * 17:13 * 17]
    ta, tb = [], []
    for it in range(6):
        for g, lst in ((ga, ta), (gb, tb)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            T.apply_ops(st, n, prec, g, 0, stream)
            e1.record(stream)
            torch.cuda.synchronize()
            lst.append(e0.elapsed_time(e1) / 1e3)
    rec("K5 4 MAJ 8-16 alternating", 2 * N * s, sorted(ta)[len(ta) // 2])
    rec("K5 4 MAJ 18-26 alternating", 2 * N * s, sorted(tb)[len(tb) // 2])
    rec("K7 init", N * s, timeit(lambda: T.init_basis(st, n, prec, 5, 1.0, 0.0, stream)))
    out = torch.zeros(8, dtype=torch.int64, device="cuda")
    rec("K6 sample (block sums + scan + 8 draws)", N * s, timeit(lambda: T.sample(st, n, prec, 8, 1, 0, out, stream)))
    print(json.dumps({"n": n, "precision": prec, "peak_GBs": peak, "kernels": rows}, indent=1))


if __name__ == "__main__":
    main()
