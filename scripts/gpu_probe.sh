#!/bin/bash
# Probe session: K5 anatomy under ncu (2 vs 3 phases), launch-trace fit, sharded bench on one GPU.
cd $GRAFT_REPO_ROOT
TAG=${1:-probe}
O=gpurun_out/$TAG
mkdir -p $O
timeout 300 python scripts/kernel_bench.py > $O/kernels.json 2> $O/kernels.err
for L in 21 28; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused -s $L -c 1 -o /tmp/prof_l$L \
    python scripts/kernel_bench.py > $O/ncu_l$L.log 2>&1
  ncu -i /tmp/prof_l$L.ncu-rep --page raw --csv > $O/raw_l$L.csv 2>/dev/null
  ncu -i /tmp/prof_l$L.ncu-rep --page source --csv --print-source cuda,sass > $O/src_l$L.csv 2>/dev/null
  gzip -f $O/src_l$L.csv
done
timeout 600 python scripts/trace_groups.py > $O/trace.log 2>&1
python scripts/fit_trace.py $O/trace.log > $O/fit.txt 2>&1
timeout 900 python bench.py --config C3 --mode sharded --shards 8 --no-cpu-baseline > $O/bench_c3_sharded8.log 2>&1
timeout 900 python bench.py --config C3 --no-cpu-baseline > $O/bench_c3_replica.log 2>&1
echo done
