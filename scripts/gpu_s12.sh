O=gpurun_out/s12; mkdir -p $O
timeout 600 python scripts/k5_micro.py > $O/micro.txt 2>&1
bash scripts/gpu_session.sh s12 "tests smoke bench" --steps 10 --warmup 3
cat $O/micro.txt | tail -20
