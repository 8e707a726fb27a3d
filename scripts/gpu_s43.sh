O=gpurun_out/s43; mkdir -p $O
timeout 300 python scripts/c4_batch.py 2000 800 > $O/batch.txt 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python scripts/c4_batch.py 2000 800 > $O/ncu.log 2>&1
cat $O/batch.txt; wc -l $O/launches.csv
