#!/bin/bash
# Full GPU session: tests + smoke, kernel microbench, bench (default + --full C4), ncu launch list
# and one --set full capture of k_fused inside the bench.   usage: gpu_session.sh TAG
cd $GRAFT_REPO_ROOT
TAG=${1:-session}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > $O/env.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 300 python scripts/kernel_bench.py > $O/kernels.json 2> $O/kernels.err
timeout 900 python bench.py > $O/bench.log 2>&1
timeout 900 python bench.py --steps 1 --warmup 3 --full --no-cpu-baseline > $O/bench_full.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s ${NCU_SKIP:-12} -c 1 -o /tmp/prof_fused \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_full.log 2>&1
cp /tmp/prof_fused.ncu-rep $O/ 2>/dev/null; echo done
# sharded mode on one GPU (local communicator) and the C5 config at c64 (128 GiB: fits one B200)
timeout 900 python bench.py --config C3 --mode sharded --shards 8 --no-cpu-baseline > $O/bench_c3_sharded8.log 2>&1
timeout 900 python bench.py --config C5 --precision 64 --leaves-per-step 16 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_c5_c64_replica.log 2>&1
timeout 1200 python bench.py --config C5 --precision 64 --mode sharded --shards 8 --leaves-per-step 16 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_c5_c64_sharded8.log 2>&1
echo done2
