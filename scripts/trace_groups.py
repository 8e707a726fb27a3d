#!/usr/bin/env python
"""Per-launch K5 timing vs group shape (TUSQ_TRACE_LAUNCHES): run a few C4 leaf batches."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["TUSQ_TRACE_LAUNCHES"] = "1"
import torch
import paper_2508_04880_b200 as T
from workloads import circuits as W
cfg = W.config("C4"); nz = cfg.noise
tree = T.build_error_tree(cfg.n, cfg.ops, nz.p1, nz.p2, nz.p_meas, cfg.shots, cfg.seed)
st = torch.empty(1 << cfg.n, dtype=torch.complex128, device="cuda")
nl = tree.n_leaves
for b in (0, nl // 3, 2 * nl // 3):
    T.run_tree(tree, 128, d_state=st, leaf_begin=b, leaf_end=b + 24, flags=T.EXEC_PROFILE)
