# Quick GPU iteration: kernel + algorithm parity tests (not slow) and a short bench.
set -x
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x -rs > gpurun_out/pytest_quick.log 2>&1; echo pytest_exit=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_quick.log 2>&1; echo bench_exit=$?
tail -3 gpurun_out/pytest_quick.log
tail -1 gpurun_out/bench_quick.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['phase_ms'], d['roofline']['frac'])"
