# adaptive + sparse + hosvd bench lines (short)
timeout 900 python bench.py --algo adaptive --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_adaptive.log 2>&1; echo adaptive_exit=$?
timeout 600 python bench.py --algo sparse --steps 5 --warmup 3 > gpurun_out/bench_sparse.log 2>&1; echo sparse_exit=$?
timeout 600 python bench.py --algo hosvd --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_hosvd.log 2>&1; echo hosvd_exit=$?
for f in adaptive sparse hosvd; do echo "== $f"; tail -3 gpurun_out/bench_$f.log | cut -c1-600; python - <<PY
import json
try:
    d=json.loads(open("gpurun_out/bench_$f.log").read().strip().splitlines()[-1]); print(d.get("ms_per_step"), d.get("value"), d.get("phase_ms"))
except Exception as e: print("parse", e)
PY
done
