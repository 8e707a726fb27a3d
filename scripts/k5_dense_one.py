"""ncu target: H on all 30 qubits (a dense state), then C4 ops 40-140 (two ordinary dense Adder
sweeps, ~5.7 ms each in scripts/k5_dense.py), one noiseless leaf through tusq_run_tree."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2508_04880_b200 as T
from workloads import circuits as W
n = 30
ops = [W.op(W.H, q) for q in range(n)] + W.config("C4").ops[40:140]
st = torch.empty(1 << n, dtype=torch.complex128, device="cuda")
tree = T.build_error_tree(n, ops, 0.0, 0.0, 0.0, 1, 1, prune=False)
T.run_tree(tree, 128, d_state=st, flags=T.EXEC_NO_SAMPLE, out_slots=np.zeros(1, dtype=np.uint64))
torch.cuda.synchronize()
