#!/usr/bin/env python
"""Run one C4 DFS leaf batch through tusq_run_tree (a target for ncu): python scripts/c4_batch.py [begin] [count]."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2508_04880_b200 as T
from workloads import circuits as W
cfg = W.config(os.environ.get("C4B_CONFIG", "C4"))
nz = cfg.noise
t = T.build_error_tree(cfg.n, cfg.ops, nz.p1, nz.p2, nz.p_meas, cfg.shots, cfg.seed)
b = int(sys.argv[1]) if len(sys.argv) > 1 else t.n_leaves // 3
k = int(sys.argv[2]) if len(sys.argv) > 2 else 8
st = torch.empty(1 << cfg.n, dtype=torch.complex128, device="cuda")
out = np.zeros(cfg.shots, dtype=np.uint64)
_, s = T.run_tree(t, 128, d_state=st, leaf_begin=b, leaf_end=b + k, out_slots=out)
torch.cuda.synchronize()
print({k_: s[k_] for k_ in ("leaves", "fused_launches", "device_seconds", "sweeps")})
