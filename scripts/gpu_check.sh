#!/bin/bash
# One GPU-box pass: parity tests, per-kernel microbenchmarks, the contract bench line.
#   gpurun -- bash scripts/gpu_check.sh <tag> [extra kernel_bench --only groups...]
tag=${1:-check}
shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$tag.log 2>&1
echo "pytest_rc=$?" >> gpurun_out/pytest_gpu_$tag.log
for g in "$@"; do
  timeout 300 python scripts/kernel_bench.py --only $g >> gpurun_out/kb_$tag.log 2>&1
done
timeout 600 python bench.py --no-cpu > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
echo "bench_rc=$?" >> gpurun_out/bench_$tag.err
