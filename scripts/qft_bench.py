#!/usr/bin/env python
"""K5 on QFT groups (C2b / C5 shapes): one noiseless native-CP QFT through tusq_run_tree (the all-I
leaf: a reset sweep, then the loaded groups) at n = 30 c128 and n = 34 c64, per-launch times from
TUSQ_EXEC_PROFILE events, and the fraction of the copy peak per loaded sweep."""
import json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2508_04880_b200 as T
from workloads import circuits as W

peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6553.9
out = np.zeros(1, dtype=np.uint64)
res = []
for n, prec in ((30, 128), (34, 64)):
    if len(sys.argv) > 1 and str(n) not in sys.argv[1:]:
        continue
    _, ops = W.qft(n, native_cp=True)
    st = torch.empty(1 << n, dtype=torch.complex128 if prec == 128 else torch.complex64, device="cuda")
    tree = T.build_error_tree(n, ops, 0.0, 0.0, 0.0, 1, 1, prune=False)
    T.run_tree(tree, prec, d_state=st, flags=T.EXEC_NO_SAMPLE, out_slots=out)
    _, s = T.run_tree(tree, prec, d_state=st, flags=T.EXEC_NO_SAMPLE | T.EXEC_PROFILE, out_slots=out)
    sweep = 2.0 * (1 << n) * (16 if prec == 128 else 8)
    ms, nl = s["gate_kernel_seconds"] * 1e3, s["gate_kernel_launches"]
    r = {"n": n, "prec": prec, "fused_launches": s["fused_launches"], "gate_kernel_ms": ms, "gate_kernel_launches": nl,
         "gate_kernel_GB": s["gate_kernel_bytes"] / 1e9,
         "achieved_GBs": s["gate_kernel_bytes"] / max(s["gate_kernel_seconds"], 1e-12) / 1e9}
    r["frac"] = r["achieved_GBs"] / peak
    r["ideal_ms_per_loaded_sweep"] = sweep / peak / 1e6
    print(json.dumps(r), flush=True)
    res.append(r)
    del st
    torch.cuda.empty_cache()
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "qft_bench.json"), "w"), indent=1)
