set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import torch;print(torch.cuda.get_device_name(0))"
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke_exit=$?
timeout 900 python -m pytest tests -m "gpu and not slow" -q -rs -s > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench_exit=$?
tail -3 gpurun_out/pytest_gpu.log
tail -2 gpurun_out/bench.log
