O=gpurun_out/s14; mkdir -p $O
TUSQ_LIB_NAME=libtusq_dbg.so TUSQ_DBG_TRACE=1 CUDA_LAUNCH_BLOCKING=1 timeout 300 python scripts/repro_range.py C3 128 0 147 188 > $O/trace.txt 2>&1
tail -n 30 $O/trace.txt
