#!/bin/bash
# A/B of library builds / env settings without tests: bench + kernel microbench per variant.
# usage: gpu_ab2.sh TAG "label:ENV=..;ENV2=.." ...
cd $GRAFT_REPO_ROOT
TAG=$1; shift
O=gpurun_out/$TAG
mkdir -p $O
for v in "$@"; do
  label=${v%%:*}; envs=${v#*:}
  ( IFS=';'; for e in $envs; do export "$e"; done
    timeout 600 python bench.py --steps 5 --warmup 3 --leaves-per-step 64 --no-cpu-baseline > $O/bench_$label.log 2>&1
    timeout 300 python scripts/kernel_bench.py > $O/kern_$label.json 2>&1 )
  grep '^{' $O/bench_$label.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(sys.argv[1], d["value"], d["roofline"]["frac"], d["roofline"]["avg_launch_ms"])' $label >> $O/ab.txt
done
cat $O/ab.txt
