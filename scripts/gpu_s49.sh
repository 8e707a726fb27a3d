O=gpurun_out/s49; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "no_live" -p no:cacheprovider -rA > $O/pytest.log 2>&1; echo rc=$?
timeout 2400 python bench.py --no-live --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_nolive.log 2>&1
tail -3 $O/pytest.log; grep -o '"value": [0-9.e-]*' $O/bench_nolive.log | head -1
