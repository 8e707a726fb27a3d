O=gpurun_out/s50; mkdir -p $O
for b in 1 2 1000000; do TUSQ_LIB_NAME=libtusq_dbg.so TUSQ_DBG_RESET_BIAS=$b timeout 1200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$b.log 2>&1; echo "bias $b: $(grep -o '"value": [0-9.]*' $O/bench_$b.log | head -1)"; done
