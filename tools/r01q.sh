mkdir -p gpurun_out; rm -f gpurun_out/bwd.log
for v in ${VARIANTS}; do echo $v >> gpurun_out/bwd.log; SVR_LIB=variants/libsvr_$v.so timeout 300 python tools/explore_cfg3.py 2>&1 | tail -1 | cut -c1-60 >> gpurun_out/bwd.log; done
