O=gpurun_out/s52; mkdir -p $O
for c in C1 C2a C2b C3; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_$c.log 2>&1; done
timeout 300 python scripts/c4_batch.py 2000 800 > $O/batch.txt 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python scripts/c4_batch.py 2000 800 > $O/ncu.log 2>&1
K5T_ONLY_DEFAULT=1 timeout 900 python scripts/k5_trace.py > $O/trace.txt 2>&1; cp gpurun_out/k5_trace.json $O/trace.json
grep -o '"value": [0-9.e-]*' $O/bench_*.log; cat $O/batch.txt
