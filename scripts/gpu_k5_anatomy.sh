O=gpurun_out/s4; mkdir -p $O
timeout 1500 python scripts/k5_trace.py > $O/trace.txt 2>&1
cp gpurun_out/k5_trace.json $O/ 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 12 -c 4 -o $O/k5_full python scripts/c4_batch.py 2600 6 > $O/ncu.log 2>&1
echo ncu rc=$? >> $O/ncu.log
tail -n 12 $O/trace.txt
