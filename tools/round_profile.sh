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
# summarise on the box (the reports themselves exceed gpurun's 64 MiB return)
mkdir -p gpurun_out/prof
PROF_DIR=gpurun_out/prof python tools/summarize_ncu.py ${TAG:-r02} > gpurun_out/prof/summary.log 2>&1
python tools/hotspots.py gpurun_out/full.ncu-rep "composite_kernel" 40 > gpurun_out/prof/hotspots_composite_cfg2.md 2>&1
python tools/hotspots.py gpurun_out/cfg4.ncu-rep "composite_coop" 40 > gpurun_out/prof/hotspots_composite_cfg4.md 2>&1
python tools/hotspots.py gpurun_out/bwd.ncu-rep "composite_backward" 30 > gpurun_out/prof/hotspots_backward_cfg3.md 2>&1
for k in composite_kernel composite_coop_kernel; do
  for r in full cfg4; do python tools/sass_histogram.py --ncu gpurun_out/$r.ncu-rep $k >> gpurun_out/prof/sass_exec_$r.md 2>&1; done
done
python tools/ncu_regions.py gpurun_out/full.ncu-rep composite_kernel "{'phaseA':('raster.cu',0,0)}" > /dev/null 2>&1
for r in full bwd cfg4; do xz -T0 -9 -c gpurun_out/$r.ncu-rep > gpurun_out/prof/$r.ncu-rep.xz 2>/dev/null; done
du -sh gpurun_out/prof/*.xz
rm -f gpurun_out/*.ncu-rep
while [ "$(du -sm gpurun_out | cut -f1)" -gt 56 ]; do rm -f "$(ls -S gpurun_out/prof/*.xz | head -1)"; done
du -sh gpurun_out; ls -la gpurun_out gpurun_out/prof
