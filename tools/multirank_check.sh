#!/bin/bash
# Exercises bench.py's multi-rank path (view sharding, max-over-ranks timing,
# rank-0 JSON line, the training all-reduce) with 2 ranks on ONE GPU over gloo.
# Not a scaling number: both ranks share the device.
mkdir -p gpurun_out
for w in ${MR_WORKLOADS:-cfg2 cfg3}; do
SVR_BENCH_DEVICE=0 SVR_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 10 --warmup 3 --e2e-steps 10 --workload $w \
  > gpurun_out/multirank_$w.json 2> gpurun_out/multirank_$w.err; echo "rc $w $?" >> gpurun_out/multirank_$w.err
done
SVR_BENCH_DEVICE=0 SVR_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 2 --impl reference --steps 2 --warmup 3 \
  > gpurun_out/multirank_ref.json 2> gpurun_out/multirank_ref.err
