# Quick GPU iteration: smoke, kernel + algorithm parity tests (not slow), a short bench.
set -x
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke_exit=$?
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -rs ${1:+-k "$1"} > gpurun_out/pytest_quick.log 2>&1; echo pytest_exit=$?
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_quick.log 2>&1; echo bench_exit=$?
tail -3 gpurun_out/smoke.log
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_quick.log | tail -30
tail -2 gpurun_out/bench_quick.log
