# iterate: algorithm parity tests, default + hosvd bench, launch list of one eager R-STHOSVD step
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_algorithms.py -q -x > gpurun_out/t_alg.log 2>&1; echo "rc=$?" >> gpurun_out/t_alg.log
timeout 300 python bench.py > gpurun_out/bench_d.json 2> gpurun_out/bench_d.err
timeout 300 python bench.py --algo hosvd > gpurun_out/bench_h.json 2> gpurun_out/bench_h.err
[ -n "$WITH_ADAPTIVE" ] && timeout 600 python bench.py --algo adaptive --steps 3 > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-phases"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/d_launches.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo list_exit=$?
