#!/bin/bash
# Quick A/B GPU session: fused-path parity subset, then bench variants (env / library builds).
# usage: gpu_ab.sh TAG "label1:ENV=..;ENV2=.." "label2:TUSQ_LIB_NAME=libtusq_rb4.so" ...
cd $GRAFT_REPO_ROOT
TAG=$1; shift
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider \
  -k "fused or adder or leaf_amplitudes or c4_full or run_tree_slots" > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu.log
for v in "$@"; do
  label=${v%%:*}; envs=${v#*:}
  ( IFS=';'; for e in $envs; do export "$e"; done
    timeout 600 python bench.py --steps 5 --warmup 3 --leaves-per-step 64 --no-cpu-baseline > $O/bench_$label.log 2>&1 )
  grep '^{' $O/bench_$label.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(sys.argv[1], d["value"], d["roofline"]["frac"], d["roofline"]["avg_launch_ms"])' $label >> $O/ab.txt
done
cat $O/ab.txt
