# Sketch iteration: quick tests, bench, sketch timing (both variants), ncu capture of the sketch.
bash scripts/gpu_quick.sh
timeout 300 python scripts/prof_sketch.py 800 0 60 20 > gpurun_out/sk.log 2>&1
RTUCKER_SKETCH_SMEM_A=1 timeout 300 python scripts/prof_sketch.py 800 0 60 20 >> gpurun_out/sk.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sketch_tc -c 1 -o gpurun_out/sk_full -f python scripts/prof_sketch.py 800 0 60 1 > gpurun_out/ncu_sk.log 2>&1; echo ncu_exit=$?
cat gpurun_out/sk.log
