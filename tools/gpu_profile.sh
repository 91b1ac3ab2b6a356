#!/bin/bash
# Profiling recipe run on the GPU box (B200_PROFILING.md): bench, launch list, full capture.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/gpu.txt
timeout 300 python bench.py --steps 200 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -2 gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/launches.csv python tools/profile_step.py > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:composite_kernel -s 2 -c 1 \
    -o gpurun_out/composite python tools/profile_step.py > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"preprocess_kernel|onesweep_kernel|duplicate_kernel" -s 6 -c 4 \
    -o gpurun_out/others python tools/profile_step.py > gpurun_out/ncu_full2.log 2>&1
ls -la gpurun_out
