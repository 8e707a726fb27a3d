#!/usr/bin/env python
"""K5 micro-benchmarks at n = 30 through tusq_run_tree on one-leaf noiseless circuits (noise 0:
the tree is the single all-I leaf, every call resets): how the fused sweep's cost depends on
whether it starts from a reset (write-only) or a load, on the tile's qubits, and on the layout
policy.  Per-launch times from TUSQ_EXEC_PROFILE events; the first call of each case is warm-up."""
import json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2508_04880_b200 as T
from workloads import circuits as W

n = 30
st = torch.empty(1 << n, dtype=torch.complex128, device="cuda")
out = np.zeros(1, dtype=np.uint64)


def case(name, ops, reps=3):
    tree = T.build_error_tree(n, ops, 0.0, 0.0, 0.0, 1, 1, prune=False)
    T.run_tree(tree, 128, d_state=st, flags=T.EXEC_NO_SAMPLE, out_slots=out)
    ms, launches, fused = [], 0, 0
    for _ in range(reps):
        _, s = T.run_tree(tree, 128, d_state=st, flags=T.EXEC_NO_SAMPLE | T.EXEC_PROFILE, out_slots=out)
        ms.append(s["gate_kernel_seconds"] * 1e3)
        launches, fused = s["gate_kernel_launches"], s["fused_launches"]
    r = {"case": name, "ms_total": float(np.median(ms)), "launches": launches, "fused": fused,
         "ms_per_launch": float(np.median(ms)) / max(launches, 1)}
    print(json.dumps(r), flush=True)
    return r


H = lambda qs: [W.op(W.H, q) for q in qs]
rows = []
# a reset group alone (write-only sweep): the tile's write runs
rows.append(case("init + 9 H on 3-11 (contiguous tile)", H(range(3, 12))))
rows.append(case("init + 9 H on 20-28 (128 B runs)", H(range(20, 29))))
rows.append(case("init + 5 H on 25-29 (2 KiB runs)", H(range(25, 30))))
# two groups: a reset group then a loaded group (the remap decides the layout between them)
rows.append(case("init 9 H 3-11, then 9 H 20-28", H(range(3, 12)) + H(range(20, 29))))
rows.append(case("init 9 H 20-28, then 9 H 3-11", H(range(20, 29)) + H(range(3, 12))))
rows.append(case("init 9 H 12-20, then 9 H 21-29", H(range(12, 21)) + H(range(21, 30))))
# four groups along a ladder
rows.append(case("ladder 4 groups", H(range(3, 12)) + H(range(10, 19)) + H(range(17, 26)) + H(range(21, 30))))
rows.append(case("ladder 6 groups", H(range(3, 12)) + H(range(10, 19)) + H(range(17, 26)) + H(range(21, 30))
                 + H(range(12, 21)) + H(range(3, 12))))
json.dump(rows, open(os.path.join(ROOT, "gpurun_out", "k5_micro.json"), "w"), indent=1)
