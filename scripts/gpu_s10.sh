O=gpurun_out/s10; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 -o $O/init9H python scripts/k5_one.py 3 11 > $O/a.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 -o $O/init5H python scripts/k5_one.py 25 29 > $O/b.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 3 -c 1 -o $O/load9H python scripts/k5_one.py 3 11 20 28 > $O/c.log 2>&1
ls $O
