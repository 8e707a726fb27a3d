#!/usr/bin/env python
"""Profile one K5 launch of a chosen kind in a C4 leaf batch: the debug-knob build's launch trace
(TUSQ_DBG_TRACE) finds the index of the first launch matching the kind, then ncu --set full
captures that k_fused launch from the release build.
usage: ncu_pick.py KIND OUT [begin count]   KIND: vmask | live | full | heavy | init"""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
kind, out = sys.argv[1], sys.argv[2]
b, k = (sys.argv[3], sys.argv[4]) if len(sys.argv) > 4 else ("2600", "40")
env = dict(os.environ, TUSQ_LIB_NAME="libtusq_dbg.so", TUSQ_DBG_TRACE="1")
p = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "c4_batch.py"), b, k], env=env, capture_output=True,
                   text=True)
idx = None
i = -1
for line in (l for l in p.stderr.splitlines() if l.startswith("[k5")):
    if line.startswith("[k5r]"):   # a replay launch (sums-only sampling): counted, never picked
        i += 1
        continue
    kv = line.split()[1:]
    d = {kv[j]: kv[j + 1] for j in range(0, len(kv) - 1, 2)}
    if d.get("ns") == "1" and d.get("oop") == "0":   # sums from K6 block sums: no k_fused launch
        continue
    i += 1
    full = int(d["nlive"]) == (1 << 18)
    match = {"heavy": full and int(d["recs"]) >= 15 and d.get("ns") == "0", "vmask": full and d["vmask"] == "1", "live": not full and d["init"] == "0", "init": d["init"] == "1",
             "full": full and d["vmask"] == "0"}[kind]
    if match:
        idx = i
        print("picked", i, line, flush=True)
        break
if idx is None:
    sys.exit("no launch of kind " + kind)
cmd = ["ncu", "--set", "full", "--clock-control", "none", "--import-source", "on", "-k", "regex:k_fused", "-s", str(idx),
       "-c", "1", "-o", out, sys.executable, os.path.join(ROOT, "scripts", "c4_batch.py"), b, k]
sys.exit(subprocess.run(cmd).returncode)
