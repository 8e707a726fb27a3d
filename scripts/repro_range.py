#!/usr/bin/env python
"""Debug aid: run one DFS leaf range of a config through tusq_run_tree (no sampling) and compare
the final state with the oracle.  usage: repro_range.py CONFIG PREC FLAGS LO HI"""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2508_04880_b200 as T
from oracle import oracle as O
from workloads import circuits as W
name, prec, flags, lo, hi = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
cfg = W.config(name)
nz = cfg.noise
t = T.build_error_tree(cfg.n, cfg.ops, nz.p1, nz.p2, nz.p_meas, cfg.shots, cfg.seed)
d = torch.zeros(1 << cfg.n, dtype=torch.complex128 if prec == 128 else torch.complex64, device="cuda")
T.run_tree(t, prec, d_state=d, leaf_begin=lo, leaf_end=hi, flags=flags | T.EXEC_NO_SAMPLE)
torch.cuda.synchronize()
ref = O.Tree.from_config(cfg).replay_leaf_core(hi - 1)
print("err", float(np.abs(d.cpu().numpy() - ref).max()))
