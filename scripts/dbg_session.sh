#!/bin/bash
# K5 debug session (debug-knob build libtusq_dbg.so): random circuits / Adder vs the oracle under
# grid caps and forced identity layouts, then the small-n batched path's parity tests.
export TUSQ_LIB_NAME=libtusq_dbg.so
O=gpurun_out/${1:-dbg}; mkdir -p $O
DBG_NS=14,16,21,22,24 timeout 600 python scripts/dbg_k5.py > $O/a.txt 2>&1
TUSQ_DBG_GRID=1 DBG_NS=14,16,17 timeout 600 python scripts/dbg_k5.py > $O/b.txt 2>&1
TUSQ_DBG_GRID=3 DBG_NS=16,21 timeout 600 python scripts/dbg_k5.py > $O/c.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "C1 or C2a or rollback or small" -p no:cacheprovider > $O/small.txt 2>&1
for f in $O/*.txt; do echo "== $f"; tail -n 6 $f; done
