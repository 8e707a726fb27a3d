O=gpurun_out/s20; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 2 -c 2 -o $O/qft30 python scripts/qft_bench.py 30 > $O/ncu.log 2>&1
echo rc=$?
