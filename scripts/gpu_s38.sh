O=gpurun_out/s38; mkdir -p $O
timeout 300 python scripts/repro_c3.py C3 > $O/repro.txt 2>&1; grep -c err $O/repro.txt; grep FAIL $O/repro.txt
bash scripts/gpu_session.sh s38 "tests smoke bench" --steps 10 --warmup 3 --no-cpu-baseline
