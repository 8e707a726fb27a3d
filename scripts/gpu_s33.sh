O=gpurun_out/s33; mkdir -p $O
timeout 600 python scripts/k5_dense.py > $O/dense_default.txt 2>&1
TUSQ_LIB_NAME=libtusq_dbg.so TUSQ_DBG_TS_L0=13 timeout 600 python scripts/k5_dense.py > $O/dense_nots.txt 2>&1
bash scripts/gpu_session.sh s33 "bench" --steps 10 --warmup 3 --no-cpu-baseline
cat $O/dense_default.txt $O/dense_nots.txt
