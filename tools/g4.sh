mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1
SVR_RANK_KEYS=0 timeout 300 python -m pytest tests -m gpu -x -q -k "entries or sort or multi_pattern" > gpurun_out/pytest_norank.log 2>&1
timeout 120 python tools/quick_time.py > gpurun_out/quick.log 2>&1
timeout 120 python tools/explore_cfg3.py > gpurun_out/cfg3.log 2>&1
VIEWS=0,77 timeout 300 python tools/explore_cfg4.py > gpurun_out/cfg4.log 2>&1
