#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/s2m; mkdir -p $O
timeout 300 python scripts/qft_groups.py > $O/qft.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/qft_launches.csv python scripts/qft_groups.py > $O/qft_ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 -o /tmp/prof_qft python scripts/qft_groups.py > $O/qft_ncu.log 2>&1
cp /tmp/prof_qft.ncu-rep $O/ 2>/dev/null
echo done
