# Evidence at the round-2 HEAD (the -m gpu suite is run separately): smoke, bench lines of every
# algorithm, the launch list of one eager default step and one ncu --set full capture of the
# C4 kernels (each ncu run only after its command exited 0 without ncu).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/g_smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/g_smoke.log
timeout 600 python bench.py > gpurun_out/g_default.json 2> gpurun_out/g_default.err
timeout 600 python bench.py --algo hosvd > gpurun_out/g_hosvd.json 2> gpurun_out/g_hosvd.err
timeout 600 python bench.py --algo sparse > gpurun_out/g_sparse.json 2> gpurun_out/g_sparse.err
timeout 900 python bench.py --algo adaptive --steps 3 > gpurun_out/g_adaptive.json 2> gpurun_out/g_adaptive.err
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-phases"
timeout 300 $CMD > gpurun_out/g_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g_launches.csv $CMD > gpurun_out/g_ncu_list.log 2>&1; echo list_exit=$?
timeout 300 python scripts/run_c4_once.py 1 > gpurun_out/g_plain2.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"sketch_tc_mna|bpass_ozaki|ttm_dmma|gram_eig|cholqr2|sketch_dfma|omega_fold|slab_gram" -c 16 -o gpurun_out/g_c4_full -f python scripts/run_c4_once.py 1 > gpurun_out/g_ncu_full.log 2>&1; echo full_exit=$?
