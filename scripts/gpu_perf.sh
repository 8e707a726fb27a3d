#!/bin/bash
# Perf-only GPU session: kernel microbench, bench (auto), ncu launch list + full capture of k_fused.
cd $GRAFT_REPO_ROOT
TAG=${1:-perf}
O=gpurun_out/$TAG
mkdir -p $O
timeout 300 python scripts/kernel_bench.py > $O/kernels.json 2> $O/kernels.err
timeout 600 python bench.py --steps 5 --warmup 3 --leaves-per-step 64 --no-cpu-baseline > $O/bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --leaves-per-step 64 --no-cpu-baseline > $O/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s ${NCU_SKIP:-12} -c 1 -o $O/prof_fused \
  python bench.py --steps 1 --warmup 3 --leaves-per-step 64 --no-cpu-baseline > $O/ncu_full.log 2>&1
echo done
# the isolated Adder MAJ group (kernel microbench K5) under a full capture
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 0 -c 1 -o $O/prof_maj \
  python scripts/kernel_bench.py > $O/ncu_maj.log 2>&1
echo done2
