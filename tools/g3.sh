mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "forward or dropin" > gpurun_out/pytest_fwd.log 2>&1
timeout 120 python tools/quick_time.py > gpurun_out/quick.log 2>&1
VIEWS=0,77 timeout 300 python tools/explore_cfg4.py > gpurun_out/cfg4b.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:composite_backward -s 3 -c 1 -o gpurun_out/bwd python tools/explore_cfg3.py > gpurun_out/ncu_bwd.log 2>&1
