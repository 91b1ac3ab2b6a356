mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1
timeout 120 python tools/quick_time.py > gpurun_out/quick.log 2>&1
timeout 120 python tools/explore_cfg3.py > gpurun_out/cfg3.log 2>&1
VIEWS=0,77 timeout 300 python tools/explore_cfg4.py > gpurun_out/cfg4.log 2>&1
VIEWS=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"onesweep|composite_kernel|duplicate|hist_kernel" -s 12 -c 12 -o gpurun_out/cfg4 python tools/explore_cfg4.py > gpurun_out/ncu_cfg4.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"epilogue|composite_backward" -s 6 -c 2 -o gpurun_out/bwd2 python tools/explore_cfg3.py > gpurun_out/ncu_bwd2.log 2>&1
