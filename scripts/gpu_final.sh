#!/bin/bash
# Round-end evidence on one GPU: tests, smoke, both bench arms, the bench's ncu launch list.
#   gpurun --timeout 3600 -- bash scripts/gpu_final.sh <tag>
tag=${1:-final}
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
bash scripts/gpu_pass.sh $tag ref
timeout 1200 $NCU --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/launches_bench_$tag.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-mmdit \
  > gpurun_out/ncu_launch_$tag.log 2>&1
echo "ncu_rc=$?" >> gpurun_out/ncu_launch_$tag.log
