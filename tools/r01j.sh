mkdir -p gpurun_out
for r in 1 0; do
SVR_RANK_ORDER=$r timeout 600 python bench.py --workload cfg4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 5 > gpurun_out/bench_cfg4_r$r.json 2> gpurun_out/bench_cfg4_r$r.err
done
