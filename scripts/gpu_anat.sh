#!/bin/bash
# K5 cost anatomy: kernel microbench variants + a launch trace of C4 leaf batches.
cd $GRAFT_REPO_ROOT
TAG=${1:-anat}
O=gpurun_out/$TAG
mkdir -p $O
timeout 300 python scripts/kernel_bench.py > $O/kernels.json 2> $O/kernels.err
timeout 600 python scripts/trace_groups.py 2> $O/trace.txt > /dev/null
python scripts/fit_trace.py $O/trace.txt > $O/fit.txt 2>&1
python - <<'P' "$O"
import json, sys
d = json.load(open(sys.argv[1] + "/kernels.json"))
for k in d["kernels"]:
    if k["kernel"].startswith("K5"): print(k)
P
cat $O/fit.txt
