"""K5 debug: random circuits through apply_ops vs the oracle at several n, under debug knobs
(build: TUSQ_LIB_NAME=libtusq_dbg.so TUSQ_NVCC_FLAGS=-DTUSQ_DEBUG_KNOBS)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2508_04880_b200 as T
from oracle import oracle as O
from workloads import circuits as W
print(T.LIB_PATH, os.environ.get("TUSQ_DBG_GRID"), os.environ.get("TUSQ_DBG_IDENTITY"), flush=True)
for n in [int(x) for x in os.environ.get("DBG_NS", "14,16,21,22").split(",")]:
    rng = np.random.default_rng(n)
    worst = 0
    for trial in range(3):
        ops = W.random_circuit(rng, n, 120)
        st = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
        st /= np.linalg.norm(st)
        ref = st.copy()
        for g in ops:
            O.apply_gate(ref, n, g)
        d = torch.from_numpy(st).cuda()
        T.apply_ops(d, n, 128, ops)
        torch.cuda.synchronize()
        worst = max(worst, float(np.abs(d.cpu().numpy() - ref).max()))
    # adder ladder (multi-group, all-X)
    k = (n - 2) // 2
    m, ops = W.adder(k)
    d = torch.zeros(1 << m, dtype=torch.complex128, device="cuda")
    T.init_basis(d, m, 128, 0)
    T.apply_ops(d, m, 128, ops)
    torch.cuda.synchronize()
    v = d.cpu().numpy()
    idx = W.adder_expected_output(k)
    e2 = abs(v[idx] - 1) + np.abs(np.delete(v, idx)).max()
    print(f"n={n} random max err {worst:.3e}  adder(m={m}) err {e2:.3e}", flush=True)
