O=gpurun_out/s8; mkdir -p $O
bash scripts/gpu_session.sh s8 "tests smoke bench" --steps 10 --warmup 3
bash scripts/gpu_s7.sh
