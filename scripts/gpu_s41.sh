O=gpurun_out/s41; mkdir -p $O
timeout 300 python scripts/repro_c3.py C3 > $O/repro.txt 2>&1; grep -c err $O/repro.txt; grep FAIL $O/repro.txt
K5T_ONLY_DEFAULT=1 timeout 900 python scripts/k5_trace.py > $O/trace.txt 2>&1; cp gpurun_out/k5_trace.json $O/trace.json
bash scripts/gpu_session.sh s41 "tests bench" --steps 10 --warmup 3 --no-cpu-baseline
