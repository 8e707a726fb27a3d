#!/bin/bash
# GPU session: tests + smoke, then the perf session (kernel microbench, bench, ncu).
cd $GRAFT_REPO_ROOT
TAG=${1:-full}
O=gpurun_out/$TAG
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
bash scripts/gpu_perf.sh $TAG
