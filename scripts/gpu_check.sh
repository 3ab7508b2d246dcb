#!/bin/bash
# One GPU-box pass: parity tests, per-kernel microbenchmarks, the contract bench line.
#   gpurun -- bash scripts/gpu_check.sh [tag]
tag=${1:-check}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$tag.log 2>&1
echo "pytest_rc=$?" >> gpurun_out/pytest_gpu_$tag.log
timeout 300 python scripts/kernel_bench.py --only gemm-n2048 > gpurun_out/kb_$tag.log 2>&1
timeout 300 python scripts/kernel_bench.py --only gemm >> gpurun_out/kb_$tag.log 2>&1
timeout 300 python scripts/kernel_bench.py --only attn >> gpurun_out/kb_$tag.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
echo "bench_rc=$?" >> gpurun_out/bench_$tag.err
