O=gpurun_out/s44; mkdir -p $O
timeout 600 python scripts/k5_dense.py > $O/dense.txt 2>&1
K5T_ONLY_DEFAULT=1 timeout 900 python scripts/k5_trace.py > $O/trace.txt 2>&1; cp gpurun_out/k5_trace.json $O/trace.json
bash scripts/gpu_session.sh s44 "bench" --steps 10 --warmup 3 --no-cpu-baseline
cat $O/dense.txt
