#!/usr/bin/env python
"""K5 launch anatomy on C4 (debug-knob build): runs DFS leaf batches with per-launch CUDA events and
prints per-variant totals plus a least-squares fit of launch time against the group shape.
Env: TUSQ_LIB_NAME=libtusq_dbg.so, TUSQ_DBG_TRACE=1 (set here), knobs TUSQ_DBG_CAP / _IDENTITY."""
import json, os, re, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import os, sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_2508_04880_b200 as T
from workloads import circuits as W
cfg = W.config("C4"); nz = cfg.noise
t = T.build_error_tree(cfg.n, cfg.ops, nz.p1, nz.p2, nz.p_meas, cfg.shots, cfg.seed)
st = torch.empty(1 << cfg.n, dtype=torch.complex128, device="cuda")
nl = t.n_leaves
out = np.zeros(cfg.shots, dtype=np.uint64)
T.run_tree(t, 128, d_state=st, leaf_begin=0, leaf_end=4, out_slots=out)   # warm-up
tot = 0.0; n = 0
for f in (0.1, 0.35, 0.6, 0.85):
    b = int(nl * f)
    _, s = T.run_tree(t, 128, d_state=st, leaf_begin=b, leaf_end=b + 40, flags=T.EXEC_PROFILE, out_slots=out)
    tot += s["device_seconds"]; n += s["fused_launches"]
print("RESULT", tot, n, flush=True)
''' % ROOT


def run(env_extra):
    env = dict(os.environ, TUSQ_LIB_NAME="libtusq_dbg.so", TUSQ_DBG_TRACE="1", **env_extra)
    p = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=900)
    rows, pend = [], {}
    for line in p.stderr.splitlines():
        if line.startswith("[k5]"):
            kv = line.split()[1:]
            d = {kv[i]: kv[i + 1] for i in range(0, len(kv) - 1, 2)}
            pend[int(d["idx"])] = d
        elif line.startswith("[t]"):
            _, i, cat, ms = line.split()
            if int(i) in pend:
                d = pend.pop(int(i))
                d["ms"] = float(ms)
                rows.append(d)
        if line.startswith("[t] 0 "):
            pass
    res = [l for l in p.stdout.splitlines() if l.startswith("RESULT")]
    return rows, res, p.stderr[-2000:] if not res else ""


def fit(rows):
    import numpy as np
    keys = ["XP", "H", "DK", "CX", "D", "CU", "CCX", "TP", "XY"]
    X = np.array([[1.0, float(r["contig"]), float(r["oop"])] + [float(r[k]) for k in keys] for r in rows])
    y = np.array([r["ms"] for r in rows])
    c, *_ = np.linalg.lstsq(X, y, rcond=None)
    return dict(zip(["base", "contig", "oop"] + keys, [round(float(v), 3) for v in c]))


if __name__ == "__main__":
    out = {}
    variants = [("remap_cap9 (default)", {}), ("remap12", {"TUSQ_DBG_CAP": "12"}),
                ("identity_cap9 (round 1)", {"TUSQ_DBG_IDENTITY": "1"}),
                ("remap_wcontig", {"TUSQ_DBG_WCONTIG": "1"})]
    if os.environ.get("K5T_ONLY_DEFAULT"):
        variants = variants[:1]
    for name, env in variants:
        rows, res, err = run(env)
        import numpy as np
        ms = [r["ms"] for r in rows]
        out[name] = {"result": res, "launches": len(rows), "avg_ms": float(np.mean(ms)) if ms else None,
                     "sum_ms": float(np.sum(ms)) if ms else None,
                     "avg_xpose": float(np.mean([int(r["XP"]) for r in rows])) if rows else None,
                     "fit": fit(rows) if len(rows) > 20 else None, "err": err,
                     "mean_counts": {k: float(np.mean([float(r[k]) for r in rows])) for k in
                                     ("recs", "ph", "XP", "H", "DK", "CX", "D", "CU", "CCX", "TP", "XY", "oop",
                                      "contig", "gtab")} if rows else None,
                     "rows": [[r["ms"], r["recs"], r["XP"], r["H"], r["DK"], r["CX"], r["CU"], r["CCX"], r["XY"],
                               r["oop"], r["contig"], r["init"], r["gtab"], r["nlive"], r["vmask"], r["ns"]] for r in rows]}
        print(name, json.dumps({k: v for k, v in out[name].items() if k != "rows"}), flush=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "k5_trace.json"), "w"), indent=1)
