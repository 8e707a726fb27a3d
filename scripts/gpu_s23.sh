O=gpurun_out/s23; mkdir -p $O
bash scripts/gpu_session.sh s23 "tests bench" --steps 10 --warmup 3 --no-cpu-baseline
