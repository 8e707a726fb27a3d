O=gpurun_out/s19; mkdir -p $O
timeout 600 python scripts/qft_bench.py > $O/qft_new.txt 2>&1
TUSQ_LIB_NAME=libtusq_dbg.so timeout 600 python scripts/qft_bench.py > $O/qft_old.txt 2>&1
bash scripts/gpu_session.sh s19 "tests"
cat $O/qft_new.txt $O/qft_old.txt
