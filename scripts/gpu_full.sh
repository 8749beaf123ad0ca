# Full GPU suite (incl. slow full-size parity) + default bench line.
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke_exit=$?
timeout 3300 python -m pytest tests -m gpu -q -rs --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$?
grep -E "passed|failed" gpurun_out/pytest_gpu.log | tail -3
grep -E "^FAILED|^ERROR" gpurun_out/pytest_gpu.log | head -20
