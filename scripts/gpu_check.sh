cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(nvidia-smi; free -g; nproc; python -c "import torch;print(torch.cuda.get_device_name())") > gpurun_out/env.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --cpu-seconds 15 > gpurun_out/bench_c4.log 2>&1
echo done
