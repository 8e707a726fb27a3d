O=gpurun_out/s18; mkdir -p $O
timeout 300 python scripts/repro_c3.py C3 > $O/repro.txt 2>&1; tail -n 3 $O/repro.txt
K5T_ONLY_DEFAULT=1 timeout 900 python scripts/k5_trace.py > $O/trace.txt 2>&1; cp gpurun_out/k5_trace.json $O/ 2>/dev/null
timeout 600 python scripts/k5_micro.py > $O/micro.txt 2>&1
bash scripts/gpu_session.sh s18 "bench" --steps 10 --warmup 3 --no-cpu-baseline
cat $O/micro.txt; tail -2 $O/trace.txt
