O=gpurun_out/s28; mkdir -p $O
timeout 900 python scripts/ncu_pick.py vmask $O/vmask > $O/vmask.log 2>&1
timeout 900 python scripts/ncu_pick.py full $O/full > $O/full.log 2>&1
grep picked $O/*.log
