O=gpurun_out/s37; mkdir -p $O
export TUSQ_LIB_NAME=libtusq_rb4.so
timeout 300 python scripts/repro_c3.py C3 > $O/repro.txt 2>&1; grep -c err $O/repro.txt; grep FAIL $O/repro.txt
timeout 600 python scripts/k5_dense.py > $O/dense.txt 2>&1
timeout 600 python scripts/qft_bench.py > $O/qft.txt 2>&1
timeout 1200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench.log 2>&1
cat $O/dense.txt; grep -o '"value": [0-9.]*' $O/bench.log | head -1
