O=gpurun_out/s6; mkdir -p $O
bash scripts/gpu_session.sh s6 "tests smoke bench" --steps 10 --warmup 3
timeout 1200 python scripts/k5_trace.py > $O/trace.txt 2>&1; cp gpurun_out/k5_trace.json $O/
