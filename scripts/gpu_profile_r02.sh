# Round-2 evidence: default bench line, the other algorithms' lines, the ncu launch list of the
# default bench (after the same command exited 0), saved under gpurun_out/ for profiles/.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv
nproc; grep -m1 "model name" /proc/cpuinfo
timeout 900 python bench.py > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err; echo default_exit=$?
timeout 900 python bench.py --algo sparse --steps 10 --warmup 3 > gpurun_out/r02_bench_sparse.json 2> gpurun_out/r02_bench_sparse.err; echo sparse_exit=$?
timeout 900 python bench.py --algo adaptive --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02_bench_adaptive.json 2> gpurun_out/r02_bench_adaptive.err; echo adaptive_exit=$?
timeout 900 python bench.py --impl reference --steps 1 --warmup 3 > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.err; echo ref_exit=$?
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-phases"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv $CMD > gpurun_out/ncu.log 2>&1; echo ncu_exit=$?
for f in default sparse adaptive reference; do tail -c 600 gpurun_out/r02_bench_$f.json; echo; done
