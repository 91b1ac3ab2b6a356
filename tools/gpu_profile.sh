#!/bin/bash
# Profiling recipe (B200_PROFILING.md), run on the GPU box. Outputs in gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/gpu.txt
timeout 300 python bench.py --steps 200 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
# launch list of a short render sequence (cold-cache, serialised: compare shares)
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python tools/profile_step.py > gpurun_out/ncu_launch.log 2>&1
# full capture of every kernel of the 3rd frame (warm): skip the first 2 frames' launches
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"composite_kernel|preprocess_kernel|onesweep_kernel|duplicate_kernel|hist_kernel|tile_setup|scan_|tile_ranges" \
    -s ${NCU_SKIP:-30} -c ${NCU_COUNT:-15} -o gpurun_out/full python tools/profile_step.py > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
