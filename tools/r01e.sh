mkdir -p gpurun_out
timeout 600 python tools/dbg_cfg4.py 5 > gpurun_out/dbg4.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
for v in old minb1 minb3 minb4; do
  echo "== $v" >> gpurun_out/variants.log
  SVR_LIB=variants/libsvr_$v.so timeout 120 python tools/quick_time.py >> gpurun_out/variants.log 2>&1
done
