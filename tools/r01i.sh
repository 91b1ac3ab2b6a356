mkdir -p gpurun_out
SVR_FRAMES=2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"composite_kernel" -s 1 -c 1 -o gpurun_out/comp_new python tools/profile_step.py > gpurun_out/ncu_comp.log 2>&1
