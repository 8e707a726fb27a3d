O=gpurun_out/s35; mkdir -p $O
bash scripts/gpu_session.sh s35 "tests smoke bench ncu" --steps 10 --warmup 3
timeout 900 python scripts/ncu_pick.py vmask $O/vmask > $O/vmask.log 2>&1
timeout 900 python scripts/ncu_pick.py full $O/full > $O/full.log 2>&1
timeout 600 python scripts/k5_dense.py > $O/dense.txt 2>&1
timeout 600 python scripts/qft_bench.py > $O/qft.txt 2>&1
K5T_ONLY_DEFAULT=1 timeout 900 python scripts/k5_trace.py > $O/trace.txt 2>&1; cp gpurun_out/k5_trace.json $O/trace.json
