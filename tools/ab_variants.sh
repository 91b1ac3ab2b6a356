# A/B of built variants (tools/build_variant.sh): per-stage device times -> gpurun_out/abv.txt
mkdir -p gpurun_out
for w in ${WL:-cfg2}; do
  for v in default ${VARIANTS}; do
    if [ "$v" = default ]; then timeout 300 python tools/ab_stage.py $w 40 | sed "s/^/$v /" >> gpurun_out/abv.txt 2>&1;
    else SVR_LIB=variants/libsvr_$v.so timeout 300 python tools/ab_stage.py $w 40 | sed "s/^/$v /" >> gpurun_out/abv.txt 2>&1; fi
  done
done
