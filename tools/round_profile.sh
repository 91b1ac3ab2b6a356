#!/bin/bash
# Round profile: benches of every workload, the reference arm, the ncu launch
# list and full captures (config 2 frame, config 3 backward, config 4).
# Run on the GPU box: gpurun -- 'bash tools/round_profile.sh'. Outputs in gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/gpu.txt
timeout 300 python bench.py --steps 200 --warmup 5 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
for w in cfg3 cfg3i cfg4 cfg5; do
  timeout 600 python bench.py --workload $w --steps ${STEPS:-30} --warmup 5 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python tools/profile_step.py > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"composite_kernel|preprocess_kernel|onesweep_kernel|duplicate_|pair_counts|hist_kernel|tile_setup|scan_|tile_ranges|tile_order" \
    -s ${NCU_SKIP:-30} -c ${NCU_COUNT:-16} -o gpurun_out/full python tools/profile_step.py > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"epilogue|composite_backward|l1_kernel" \
    -s 9 -c 3 -o gpurun_out/bwd python tools/explore_cfg3.py > gpurun_out/ncu_bwd.log 2>&1
VIEWS=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"composite_kernel|onesweep|preprocess|duplicate_" \
    -s 12 -c 8 -o gpurun_out/cfg4 python tools/explore_cfg4.py > gpurun_out/ncu_cfg4.log 2>&1
ls -la gpurun_out
