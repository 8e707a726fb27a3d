O=gpurun_out/s31; mkdir -p $O
timeout 300 python scripts/repro_c3.py C3 > $O/repro.txt 2>&1; grep -c "err" $O/repro.txt; grep FAIL $O/repro.txt
K5T_ONLY_DEFAULT=1 timeout 900 python scripts/k5_trace.py > $O/trace.txt 2>&1; cp gpurun_out/k5_trace.json $O/trace.json
timeout 600 python scripts/k5_micro.py > $O/micro.txt 2>&1
timeout 600 python scripts/qft_bench.py > $O/qft.txt 2>&1
bash scripts/gpu_session.sh s31 "tests bench" --steps 10 --warmup 3 --no-cpu-baseline
cat $O/micro.txt $O/qft.txt
