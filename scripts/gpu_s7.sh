#!/bin/bash
# Round-2 evidence session: delta study, bench lines for the other configs, per-kernel ncu
# bandwidth list (n = 30), one ncu --set full capture of K5 inside a C4 batch.
O=gpurun_out/s7; mkdir -p $O
timeout 1500 python scripts/delta_study.py --out $O/delta_study.json > $O/delta.log 2>&1; echo "delta rc=$?" >> $O/rc.txt
for c in C1 C2a C2b C3; do
  timeout 600 python bench.py --config $c --steps 4 --warmup 2 --no-cpu-baseline > $O/bench_$c.log 2>&1; echo "bench $c rc=$?" >> $O/rc.txt
done
timeout 900 python bench.py --config C4 --precision 64 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_C4_c64.log 2>&1; echo "bench C4 c64 rc=$?" >> $O/rc.txt
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/kb_launches.csv python scripts/kernel_bench.py > $O/kb_ncu.log 2>&1; echo "kb ncu rc=$?" >> $O/rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 20 -c 2 -o $O/k5_full python scripts/c4_batch.py 2600 8 > $O/ncu_full.log 2>&1; echo "ncu full rc=$?" >> $O/rc.txt
cat $O/rc.txt
