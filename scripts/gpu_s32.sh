O=gpurun_out/s32; mkdir -p $O
for k in 13 3 6 9; do TUSQ_LIB_NAME=libtusq_dbg.so TUSQ_DBG_TS_L0=$k timeout 600 python scripts/k5_dense.py > $O/dense_$k.txt 2>&1; done
for k in 13 9; do TUSQ_DBG_TS_L0=$k K5T_ONLY_DEFAULT=1 timeout 900 python scripts/k5_trace.py > $O/trace_$k.txt 2>&1; cp gpurun_out/k5_trace.json $O/trace_$k.json; done
tail -n 7 $O/dense_*.txt
