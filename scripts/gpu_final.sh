# round-end style verification: GPU tests, smoke, the default bench line (with the CPU baseline)
O=gpurun_out/final; mkdir -p $O
bash scripts/gpu_session.sh final "tests smoke bench"
