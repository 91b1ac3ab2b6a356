mkdir -p gpurun_out; rm -f gpurun_out/variants.log
for v in ${VARIANTS:-ab2}; do
echo "== $v" >> gpurun_out/variants.log
SVR_LIB=variants/libsvr_$v.so timeout 120 python tools/stage_time.py >> gpurun_out/variants.log 2>&1
SVR_LIB=variants/libsvr_$v.so timeout 600 python bench.py --workload cfg4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 5 > gpurun_out/b4.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/b4.json').read().strip().splitlines()[-1]); print('cfg4', round(d['value'],2), {k:round(v,3) for k,v in d['stage_ms_per_step'].items() if v>0})" >> gpurun_out/variants.log
done
[ -n "$TESTS" ] && timeout 900 python -m pytest tests/ -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo done
