#!/bin/bash
# Round-end style verification: full GPU test suite, smoke, default bench.
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-verify}; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.log 2>&1
echo done
