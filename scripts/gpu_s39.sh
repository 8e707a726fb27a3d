O=gpurun_out/s39; mkdir -p $O
K5T_ONLY_DEFAULT=1 timeout 900 python scripts/k5_trace.py > $O/trace.txt 2>&1; cp gpurun_out/k5_trace.json $O/trace.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file $O/launches.csv python scripts/c4_batch.py 2600 300 > $O/ncu.log 2>&1
timeout 300 python scripts/c4_batch.py 2600 300 > $O/batch.txt 2>&1
cat $O/batch.txt
