#!/bin/bash
# N>1 code paths of bench.py with 2 ranks sharing one GPU (gloo test mode)
export BENCH_DIST_BACKEND=gloo
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
for c in c2 c3 c5; do
  timeout 600 $R bench.py --gpus 2 --config $c --steps 2 --warmup 3 --no-primitives --no-cpu-baseline > gpurun_out/mr_$c.log 2>&1
  echo "$c rc=$?"; grep '^{' gpurun_out/mr_$c.log | tail -1 | cut -c1-300; tail -2 gpurun_out/mr_$c.log | cut -c1-300
done
timeout 600 $R bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/mr_ref.log 2>&1; echo "ref rc=$?"; grep '^{' gpurun_out/mr_ref.log | cut -c1-200
