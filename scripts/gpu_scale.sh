#!/bin/bash
# Multi-GPU bench pass: gpurun --gpus N -- bash scripts/gpu_scale.sh <tag> <N...>
tag=${1:-scale}
shift
mkdir -p gpurun_out
for n in "$@"; do
  if [ "$n" = "1" ]; then
    timeout 900 python bench.py --no-cpu > gpurun_out/bench_${tag}_n1.json 2> gpurun_out/bench_${tag}_n1.err
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29900 + n)) bench.py --gpus $n --no-cpu > gpurun_out/bench_${tag}_n$n.json 2> gpurun_out/bench_${tag}_n$n.err
  fi
  echo "rc=$?" >> gpurun_out/bench_${tag}_n$n.err
done
