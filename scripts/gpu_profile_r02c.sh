# Round-2 (final session) breakdowns: adaptive phase times, and the ncu launch lists of one
# R-HOSVD call and one adaptive call (each run first without ncu).
set -x
mkdir -p gpurun_out
timeout 600 python scripts/adaptive_phases.py > gpurun_out/c_adaptive_phases.log 2>&1; echo ap_exit=$?
CMD="python bench.py --algo hosvd --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-phases"
timeout 300 $CMD > gpurun_out/c_hosvd.json 2> gpurun_out/c_hosvd.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c_hosvd_launches.csv $CMD > gpurun_out/c_ncu_hosvd.log 2>&1; echo hl_exit=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c_adaptive_launches.csv python scripts/adaptive_once.py > gpurun_out/c_ncu_adaptive.log 2>&1; echo al_exit=$?
