O=gpurun_out/s34; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/list.csv python scripts/qft_dense_one.py > $O/l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 3 -c 1 -o $O/qftd python scripts/qft_dense_one.py > $O/n.log 2>&1
grep -c k_fused $O/list.csv
