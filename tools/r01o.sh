mkdir -p gpurun_out; rm -f gpurun_out/epi.log
for v in epi_a epi_c; do echo $v >> gpurun_out/epi.log; SVR_LIB=variants/libsvr_$v.so timeout 300 python tools/explore_cfg3.py 2>&1 | tail -1 >> gpurun_out/epi.log; done
SVR_LIB=variants/libsvr_epi_c.so timeout 900 python -m pytest tests/ -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
