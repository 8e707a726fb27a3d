O=gpurun_out/s21; mkdir -p $O
timeout 600 python scripts/qft_bench.py > $O/qft.txt 2>&1
K5T_ONLY_DEFAULT=1 timeout 900 python scripts/k5_trace.py > $O/trace.txt 2>&1; cp gpurun_out/k5_trace.json $O/ 2>/dev/null
bash scripts/gpu_session.sh s21 "tests"
cat $O/qft.txt; tail -1 $O/trace.txt | cut -c1-300
