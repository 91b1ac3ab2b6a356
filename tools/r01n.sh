mkdir -p gpurun_out
timeout 300 python tools/explore_cfg3.py > gpurun_out/cfg3.log 2>&1
timeout 900 python -m pytest tests/test_gpu_backward.py tests/test_gpu_dropin.py -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
