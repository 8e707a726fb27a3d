O=gpurun_out/s45; mkdir -p $O
timeout 900 python scripts/ncu_pick.py full $O/full > $O/full.log 2>&1
python scripts/ncu_summary.py $O/full.ncu-rep - $O/ncu_full.json > /dev/null 2>&1
