#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/s2l; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider \
  -k "random_circuits or run_tree_slots or leaf_amplitudes or sharded or single_gate" > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --config C5 --precision 64 --leaves-per-step 16 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_c5_c64_replica.log 2>&1
echo done
