# Round-2 (late) evidence: bench lines of every algorithm, the ncu launch list of the default
# bench, and one ncu --set full capture of the C4 hot kernels (each ncu run only after the same
# command exited 0 without ncu).  Outputs under gpurun_out/ (copied to profiles/ by hand).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv
nproc; grep -m1 "model name" /proc/cpuinfo
timeout 900 python bench.py > gpurun_out/p_default.json 2> gpurun_out/p_default.err; echo default_exit=$?
timeout 900 python bench.py --algo sparse > gpurun_out/p_sparse.json 2> gpurun_out/p_sparse.err; echo sparse_exit=$?
timeout 900 python bench.py --algo adaptive --steps 2 --no-e2e > gpurun_out/p_adaptive.json 2> gpurun_out/p_adaptive.err; echo adaptive_exit=$?
timeout 900 python bench.py --impl reference --steps 1 --warmup 3 > gpurun_out/p_reference.json 2> gpurun_out/p_reference.err; echo ref_exit=$?
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-phases"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p_launches.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo list_exit=$?
timeout 300 python scripts/run_c4_once.py 1 > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"sketch_tc_mn|bpass_ozaki|ttm_dmma|gram_eig|cholqr2|sketch_dfma|factor_" -c 16 -o gpurun_out/p_c4_full -f python scripts/run_c4_once.py 1 > gpurun_out/ncu_full.log 2>&1; echo full_exit=$?
for f in default sparse adaptive reference; do tail -c 300 gpurun_out/p_$f.json; echo; done
