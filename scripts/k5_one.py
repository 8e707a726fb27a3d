"""One K5 micro case (scripts/k5_micro.py) for ncu: python scripts/k5_one.py <first> <last> [<first2> <last2>]
-> noiseless one-leaf circuit H(first..last) [+ H(first2..last2)] at n = 30, run twice (reset each time)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2508_04880_b200 as T
from workloads import circuits as W
a = [int(x) for x in sys.argv[1:]]
ops = [W.op(W.H, q) for q in range(a[0], a[1] + 1)]
if len(a) > 3:
    ops += [W.op(W.H, q) for q in range(a[2], a[3] + 1)]
st = torch.empty(1 << 30, dtype=torch.complex128, device="cuda")
tree = T.build_error_tree(30, ops, 0.0, 0.0, 0.0, 1, 1, prune=False)
for _ in range(2):
    T.run_tree(tree, 128, d_state=st, flags=T.EXEC_NO_SAMPLE, out_slots=np.zeros(1, dtype=np.uint64))
torch.cuda.synchronize()
