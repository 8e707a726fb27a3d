O=gpurun_out/s30; mkdir -p $O
K5T_ONLY_DEFAULT=1 timeout 900 python scripts/k5_trace.py > $O/trace.txt 2>&1; cp gpurun_out/k5_trace.json $O/store.json
TUSQ_DBG_NOSTORE=1 K5T_ONLY_DEFAULT=1 timeout 900 python scripts/k5_trace.py > $O/trace_ns.txt 2>&1; cp gpurun_out/k5_trace.json $O/nostore.json
