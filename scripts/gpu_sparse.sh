# Sparse path on the GPU: parity tests, then the C5 bench line (phases) and a launch list.
set -x
timeout 900 python -m pytest tests/test_gpu_sparse.py -q -x -rs ${1:+-k "$1"} > gpurun_out/pytest_sparse.log 2>&1; echo pytest_exit=$?
timeout 600 python bench.py --algo sparse --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_sparse.log 2>&1; echo bench_exit=$?
grep -E "passed|failed|FAILED|Error|assert" gpurun_out/pytest_sparse.log | tail -20
tail -c 1500 gpurun_out/bench_sparse.log
