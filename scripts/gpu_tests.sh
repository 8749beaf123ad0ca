# GPU tests (optionally a -k filter in $1) + a short bench line.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; grep -m1 "model name" /proc/cpuinfo
python -m paper_1905_07311_b200.build > gpurun_out/build.log 2>&1; echo build_exit=$?
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke_exit=$?
timeout 2400 python -m pytest tests -m "gpu" -q -rs ${1:+-k "$1"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$?
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench_exit=$?
tail -15 gpurun_out/pytest_gpu.log
tail -1 gpurun_out/bench.log
