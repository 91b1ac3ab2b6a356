mkdir -p gpurun_out; rm -f gpurun_out/pdl.log
for w in cfg3 cfg3i; do for p in 1 0; do SVR_PDL=$p timeout 300 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/b_pdl$p.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/b_pdl$p.json').read().strip().splitlines()[-1]); print('$w pdl $p', round(d['value'],1), round(d['e2e']['value'],1), d['ms_per_step'])" >> gpurun_out/pdl.log; done; done
timeout 900 python -m pytest tests/ -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
