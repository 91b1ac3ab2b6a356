#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
for v in minb1 minb2 minb3 minb4; do
  echo "== $v" >> gpurun_out/variants.log
  SVR_LIB=variants/libsvr_$v.so timeout 120 python tools/quick_time.py >> gpurun_out/variants.log 2>&1
done
