O=gpurun_out/s16; mkdir -p $O
timeout 300 python scripts/repro_c3.py C3 > $O/repro.txt 2>&1; tail -n 3 $O/repro.txt
timeout 600 python scripts/k5_micro.py > $O/micro.txt 2>&1
bash scripts/gpu_session.sh s16 "tests smoke bench" --steps 10 --warmup 3
cat $O/micro.txt | tail -20
