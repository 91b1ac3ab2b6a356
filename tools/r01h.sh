mkdir -p gpurun_out; rm -f gpurun_out/variants.log
for v in laneq cpasync; do
  echo "== $v" >> gpurun_out/variants.log
  SVR_LIB=variants/libsvr_$v.so timeout 120 python tools/quick_time.py >> gpurun_out/variants.log 2>&1
done
timeout 900 python -m pytest tests/ -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
