#!/usr/bin/env python
"""One noiseless QFT30 (native CP) through the fused path: its K5 launches are the QFT groups
(C2b / C5 shapes) for ncu.  Prints per-launch times (CUDA events around tusq_apply_ops)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2508_04880_b200 as T  # noqa: E402
from workloads import circuits as W  # noqa: E402

n, ops = W.qft(30, native_cp=True)
st = torch.zeros(1 << n, dtype=torch.complex128, device="cuda")
T.init_basis(st, n, 128, 0)
s = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(2):
    e0.record(s)
    T.apply_ops(st, n, 128, ops, 0, s)
    e1.record(s)
    torch.cuda.synchronize()
    print(f"QFT30 pass {rep}: {e0.elapsed_time(e1):.1f} ms for {len(ops)} gates")
