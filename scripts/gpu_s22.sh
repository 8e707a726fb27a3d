O=gpurun_out/s22; mkdir -p $O
timeout 300 python scripts/repro_c3.py C3 > $O/repro.txt 2>&1; tail -n 4 $O/repro.txt
bash scripts/gpu_session.sh s22 "tests bench" --steps 10 --warmup 3 --no-cpu-baseline
