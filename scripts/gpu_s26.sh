O=gpurun_out/s26; mkdir -p $O
K5T_ONLY_DEFAULT=1 timeout 900 python scripts/k5_trace.py > $O/trace.txt 2>&1; cp gpurun_out/k5_trace.json $O/ 2>/dev/null
tail -2 $O/trace.txt | cut -c1-300
