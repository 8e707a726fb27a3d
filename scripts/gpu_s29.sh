O=gpurun_out/s29; mkdir -p $O
timeout 900 python scripts/ncu_pick.py vmask $O/vmask > $O/vmask.log 2>&1
grep picked $O/*.log
