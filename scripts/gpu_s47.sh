O=gpurun_out/s47; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "c3_all_slots" -p no:cacheprovider -rA > $O/pytest.log 2>&1; echo rc=$?
tail -5 $O/pytest.log
