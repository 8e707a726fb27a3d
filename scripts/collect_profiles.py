#!/usr/bin/env python
"""Copy the judged evidence of one GPU session (gpurun_out/<tag>) into profiles/ (tracked):
bench JSON line, kernel microbench, ncu launch-list shares, ncu --set full summaries."""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    tag, prefix = sys.argv[1], sys.argv[2]
    src = os.path.join(ROOT, "gpurun_out", tag)
    dst = os.path.join(ROOT, "profiles")
    os.makedirs(dst, exist_ok=True)
    bench = os.path.join(src, "bench.log")
    if os.path.exists(bench):
        line = [l for l in open(bench).read().splitlines() if l.startswith("{")][-1]
        open(os.path.join(dst, f"{prefix}_bench.json"), "w").write(line + "\n")
    if os.path.exists(os.path.join(src, "kernels.json")):
        shutil.copy(os.path.join(src, "kernels.json"), os.path.join(dst, f"{prefix}_kernel_microbench.json"))
    if os.path.exists(os.path.join(src, "launches.csv")):
        shutil.copy(os.path.join(src, "launches.csv"), os.path.join(dst, f"{prefix}_ncu_launches.csv"))
    for rep, name in (("prof_fused.ncu-rep", "ncu_k_fused_in_bench"), ("prof_maj.ncu-rep", "ncu_k_fused_maj_group")):
        p = os.path.join(src, rep)
        if os.path.exists(p):
            subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), p,
                            os.path.join(src, "launches.csv") if os.path.exists(os.path.join(src, "launches.csv")) else "-",
                            os.path.join(dst, f"{prefix}_{name}.json"), "34359738368"], check=False,
                           stdout=subprocess.DEVNULL)
    print(sorted(f for f in os.listdir(dst) if f.startswith(prefix)))


if __name__ == "__main__":
    main()
