#!/usr/bin/env python
"""K5 sweeps on DENSE states: one-leaf noiseless circuits at n = 30 through tusq_run_tree with
per-launch events (TUSQ_EXEC_PROFILE).  A prefix of H on every qubit makes the state dense (after
it every tile may be nonzero, so the case's groups are ordinary full sweeps); the case's K5 time is
(prefix + case) - (prefix), median of 3."""
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
H = lambda qs: [W.op(W.H, q) for q in qs]
pre = H(range(n))


def kms(ops):
    tree = T.build_error_tree(n, ops, 0.0, 0.0, 0.0, 1, 1, prune=False)
    T.run_tree(tree, 128, d_state=st, flags=T.EXEC_NO_SAMPLE, out_slots=out)
    v = []
    for _ in range(3):
        _, s = T.run_tree(tree, 128, d_state=st, flags=T.EXEC_NO_SAMPLE | T.EXEC_PROFILE, out_slots=out)
        v.append((s["gate_kernel_seconds"] * 1e3, s["fused_launches"]))
    v.sort()
    return v[1]


cfg = W.config("C4")
_, qft = W.qft(n, native_cp=True)
cases = [("9 H on 3-11", H(range(3, 12))), ("9 H on 20-28", H(range(20, 29))), ("5 H on 25-29", H(range(25, 30))),
         ("C4 ops 40-140", cfg.ops[40:140]), ("C4 ops 250-350", cfg.ops[250:350]), ("C4 ops 400-498", cfg.ops[400:]),
         ("QFT30 pass", qft)]
base, bl = kms(pre)
res = [{"case": "prefix H(0..29)", "ms": base, "launches": bl}]
print(json.dumps(res[0]), flush=True)
for name, ops in cases:
    t, l = kms(pre + ops)
    r = {"case": name, "ms": t - base, "launches": l - bl, "ms_per_launch": (t - base) / max(l - bl, 1)}
    print(json.dumps(r), flush=True)
    res.append(r)
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "k5_dense.json"), "w"), indent=1)
