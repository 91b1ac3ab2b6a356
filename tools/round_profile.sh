#!/bin/bash
# Round profile: the GPU test suite, smoke, benches of every workload, the
# reference arm, the drop-in bench, the ncu launch list and full captures
# (config-2 frame, config-3 backward, config-4 view). Run on the GPU box:
#   gpurun -- 'bash tools/round_profile.sh'      (outputs in gpurun_out/)
# then here: python tools/summarize_ncu.py rNN
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/gpu.txt
if [ -z "$SKIP_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q --durations=20 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
fi
timeout 400 python bench.py --steps 200 --warmup 5 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
for w in cfg3 cfg3i cfg4 cfg5; do
  timeout 600 python bench.py --workload $w --steps ${STEPS:-30} --warmup 5 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python tools/profile_step.py > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"composite_kernel|preprocess_kernel|onesweep_kernel|duplicate_|pair_counts|hist_kernel|tile_setup|scan_|tile_ranges|tile_order" \
    -s ${NCU_SKIP:-30} -c ${NCU_COUNT:-16} -o gpurun_out/full python tools/profile_step.py > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"epilogue|composite_backward|composite_kernel|l1_kernel" \
    -s 12 -c 4 -o gpurun_out/bwd python tools/ab_stage.py cfg3 2 > gpurun_out/ncu_bwd.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"composite|onesweep|preprocess|duplicate_|merge_huge|pair_counts" \
    -s 20 -c 12 -o gpurun_out/cfg4 python tools/ab_stage.py cfg4 2 > gpurun_out/ncu_cfg4.log 2>&1
ls -la gpurun_out
