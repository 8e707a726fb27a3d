O=gpurun_out/s51; mkdir -p $O
bash scripts/gpu_session.sh s51 "tests smoke bench"
timeout 1200 python bench.py --precision 64 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c4_c64.log 2>&1
grep -o '"value": [0-9.e-]*' $O/bench*.log
