O=gpurun_out/s46; mkdir -p $O
timeout 900 python scripts/ncu_pick.py heavy $O/heavy 2600 160 > $O/heavy.log 2>&1
python scripts/ncu_summary.py $O/heavy.ncu-rep - $O/ncu_heavy.json > /dev/null 2>&1
grep picked $O/heavy.log
