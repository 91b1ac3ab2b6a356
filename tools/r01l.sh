mkdir -p gpurun_out; rm -f gpurun_out/variants.log
for v in os9 os9m3; do
SVR_LIB=variants/libsvr_$v.so timeout 120 python tools/stage_time.py >> gpurun_out/variants.log 2>&1
SVR_LIB=variants/libsvr_$v.so timeout 600 python bench.py --workload cfg4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 5 > gpurun_out/b4.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/b4.json').read().strip().splitlines()[-1]); print('$v cfg4', round(d['value'],2), {k:round(v,3) for k,v in d['stage_ms_per_step'].items() if v>0})" >> gpurun_out/variants.log
done
SVR_LIB=variants/libsvr_os9.so timeout 900 python -m pytest tests/ -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
