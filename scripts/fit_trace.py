#!/usr/bin/env python
"""Least-squares per-record costs from a TUSQ_TRACE_LAUNCHES trace: ms ~ c0 + sum_k c_k * count_k."""
import re
import sys

import numpy as np

rows = []
for line in open(sys.argv[1]):
    if not line.startswith("[launch]"):
        continue
    ms = float(line.split()[1])
    kv = dict(re.findall(r"\b(H|DK|CX|D|XP|XY|T|O|CU)(\d+)", line))
    init = int(re.search(r"init (\d)", line).group(1))
    rows.append((ms, init, kv))
keys = ["H", "DK", "CX", "D", "XP", "XY", "T", "O", "CU"]
keys = [k for k in keys if any(int(r[2].get(k, 0)) for r in rows)]
A = np.array([[1.0, r[1]] + [float(r[2].get(k, 0)) for k in keys] for r in rows])
y = np.array([r[0] for r in rows])
c, *_ = np.linalg.lstsq(A, y, rcond=None)
print(f"launches {len(rows)}  mean {y.mean():.3f} ms  total {y.sum():.1f} ms")
for name, v in zip(["const", "init"] + keys, c):
    print(f"  {name:6s} {v:7.3f} ms")
res = y - A @ c
print(f"  rms residual {np.sqrt((res ** 2).mean()):.3f} ms")
