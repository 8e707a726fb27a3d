O=gpurun_out/s11; mkdir -p $O
timeout 600 python scripts/k5_micro.py > $O/micro.txt 2>&1
bash scripts/gpu_session.sh s11 "tests bench" --steps 10 --warmup 3 --no-cpu-baseline
cat $O/micro.txt
