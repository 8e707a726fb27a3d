#!/usr/bin/env python
"""Debug aid: C3 (24q Adder) rollback leaves through tusq_run_tree, each run in a fresh process
state is not needed -- prints per (prec, flags, leaf) the max amplitude error against the oracle or
the CUDA error.  Library chosen by TUSQ_LIB_NAME.  usage: python scripts/repro_c3.py [config]"""
import os, sys, traceback
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2508_04880_b200 as T
from oracle import oracle as O
from workloads import circuits as W

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
cfg = W.config(name)
nz = cfg.noise
t = T.build_error_tree(cfg.n, cfg.ops, nz.p1, nz.p2, nz.p_meas, cfg.shots, cfg.seed)
ot = O.Tree.from_config(cfg)
nl = t.n_leaves
rng = np.random.default_rng(3)
picks = sorted({0, 1, nl - 1, *[int(x) for x in rng.integers(0, nl, size=3)]})
print(T.LIB_PATH, "leaves", nl, "picks", picks, flush=True)
refs = {l: ot.replay_leaf_core(l) for l in picks}
for prec in (128, 64):
    for flags in (0, T.EXEC_NO_RESET):
        for l in picks:
            d = torch.zeros(1 << cfg.n, dtype=torch.complex128 if prec == 128 else torch.complex64, device="cuda")
            lo = max(0, l - 40)
            try:
                T.run_tree(t, prec, d_state=d, leaf_begin=lo, leaf_end=l + 1, flags=flags | T.EXEC_NO_SAMPLE)
                torch.cuda.synchronize()
                err = float(np.abs(d.cpu().numpy() - refs[l]).max())
                print(f"prec {prec} flags {flags} leaf {l}: err {err:.3e}", flush=True)
            except Exception as e:
                print(f"prec {prec} flags {flags} leaf {l}: FAIL {e}", flush=True)
                sys.exit(1)
