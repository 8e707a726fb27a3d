O=gpurun_out/s42; mkdir -p $O
bash scripts/gpu_session.sh s42 "tests smoke bench ncu"
timeout 900 python scripts/ncu_pick.py full $O/full > $O/full.log 2>&1
timeout 600 python scripts/k5_dense.py > $O/dense.txt 2>&1
timeout 600 python scripts/qft_bench.py > $O/qft.txt 2>&1
K5T_ONLY_DEFAULT=1 timeout 900 python scripts/k5_trace.py > $O/trace.txt 2>&1; cp gpurun_out/k5_trace.json $O/trace.json
timeout 600 python scripts/kernel_bench.py > $O/kb.json 2> $O/kb.err
python scripts/ncu_summary.py $O/k_fused_full.ncu-rep $O/launches.csv $O/ncu_in_bench.json > /dev/null 2>&1
python scripts/ncu_summary.py $O/full.ncu-rep - $O/ncu_full.json > /dev/null 2>&1
rm -f $O/k_fused_full.ncu-rep
du -sh gpurun_out; ls -la $O
