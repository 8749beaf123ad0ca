# One GPU call: smoke, GPU tests, bench, ncu launch list (after the same command exited 0).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; grep -m1 "model name" /proc/cpuinfo
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke_exit=$?
timeout 900 python -m pytest tests -m "gpu" -q -rs -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$?
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench_exit=$?
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1; echo ncu_exit=$?
tail -3 gpurun_out/pytest_gpu.log
tail -2 gpurun_out/bench.log
