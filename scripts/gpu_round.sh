#!/bin/bash
# One GPU session: tests, smoke, kernel microbench, bench (modes), ncu launch list + full capture.
# usage: bash scripts/gpu_round.sh <tag> [tests]
cd $GRAFT_REPO_ROOT
TAG=${1:-run}
mkdir -p gpurun_out/$TAG
O=gpurun_out/$TAG
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > $O/env.log 2>&1
if [ "$2" == "tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $O/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> $O/pytest_gpu.log
  timeout 300 python __graft_entry__.py --smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
fi
timeout 300 python scripts/kernel_bench.py > $O/kernels.json 2> $O/kernels.err
for m in auto strict loose; do
  TUSQ_TILE_MODE=$m timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$m.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 6 -c 1 -o $O/prof_fused \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_full.log 2>&1
echo done
