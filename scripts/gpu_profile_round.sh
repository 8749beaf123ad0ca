# Round profile capture: full bench line, ncu launch list and ncu --set full captures of the
# dominant kernels (each ncu run only after the same command exited 0 without ncu).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo bench_exit=$?
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo list_exit=$?
timeout 300 python scripts/run_c4_once.py 1 > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"sketch_tc_mn|bpass_ozaki|ttm_dmma|gram_eig|cholqr2|sketch_dfma" -c 12 -o gpurun_out/c4_full -f python scripts/run_c4_once.py 1 > gpurun_out/ncu_full.log 2>&1; echo full_exit=$?
tail -1 gpurun_out/bench_full.log
