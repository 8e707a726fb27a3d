#!/bin/bash
# ncu --set full of two specific K5 launches of the C4 trace replay (launch indices $2 and $3)
cd $GRAFT_REPO_ROOT
O=gpurun_out/$1
mkdir -p $O
for s in $2 $3; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s $s -c 1 -o $O/launch_$s \
    python scripts/trace_groups.py > $O/ncu_$s.log 2>&1
done
echo done
