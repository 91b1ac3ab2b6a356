mkdir -p gpurun_out
for v in oldfix minb4; do
SVR_LIB=variants/libsvr_$v.so timeout 900 python tools/prec_sweep.py > gpurun_out/prec_$v.log 2>&1
done
