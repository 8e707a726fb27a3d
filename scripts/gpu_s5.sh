O=gpurun_out/s5; mkdir -p $O
bash scripts/gpu_session.sh s5 "tests bench kb" --steps 10 --warmup 3 --no-cpu-baseline
timeout 1200 python scripts/k5_trace.py > $O/trace.txt 2>&1; cp gpurun_out/k5_trace.json $O/
