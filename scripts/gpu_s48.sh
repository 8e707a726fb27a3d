O=gpurun_out/s48; mkdir -p $O
bash scripts/gpu_session.sh s48 "tests smoke bench"
for c in C1 C2a C2b C3; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_$c.log 2>&1; done
timeout 1200 python bench.py --precision 64 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c4_c64.log 2>&1
grep -o '"value": [0-9.e-]*' $O/bench_*.log
