#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/s2j; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider \
  -k "fused or adder or leaf_amplitudes or c4_full or run_tree_slots or sharded" > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --config C5 --precision 64 --leaves-per-step 16 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_c5_c64_replica.log 2>&1
timeout 1200 python bench.py --config C5 --precision 64 --mode sharded --shards 8 --leaves-per-step 16 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_c5_c64_sharded8.log 2>&1
for v in "cap9:X=1" "cap8:TUSQ_HI_CAP=8"; do
  label=${v%%:*}; e=${v#*:}
  env $e timeout 600 python bench.py --steps 5 --warmup 3 --leaves-per-step 64 --no-cpu-baseline > $O/bench_$label.log 2>&1
done
echo done
