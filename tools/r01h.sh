mkdir -p gpurun_out; rm -f gpurun_out/variants.log
timeout 120 python tools/stage_time.py >> gpurun_out/variants.log 2>&1
SVR_RANK_ORDER=0 timeout 120 python tools/stage_time.py >> gpurun_out/variants.log 2>&1
SVR_FRAMES=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rank.csv python tools/profile_step.py > /dev/null 2>&1
