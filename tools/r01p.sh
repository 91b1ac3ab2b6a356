mkdir -p gpurun_out; rm -f gpurun_out/variants.log
for v in poly3 pre8; do SVR_LIB=variants/libsvr_$v.so timeout 120 python tools/stage_time.py >> gpurun_out/variants.log 2>&1; done
SVR_FRAMES=2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"composite_kernel" -s 1 -c 1 -o gpurun_out/comp_poly python tools/profile_step.py > /dev/null 2>&1
