O=gpurun_out/s27; mkdir -p $O
K5T_ONLY_DEFAULT=1 timeout 900 python scripts/k5_trace.py > $O/trace.txt 2>&1; cp gpurun_out/k5_trace.json $O/ 2>/dev/null
bash scripts/gpu_session.sh s27 "tests bench" --steps 10 --warmup 3 --no-cpu-baseline
