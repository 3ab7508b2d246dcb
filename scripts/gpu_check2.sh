#!/bin/bash
tag=${1:-check}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$tag.log 2>&1
echo "pytest_rc=$?" >> gpurun_out/pytest_gpu_$tag.log
for ht in 1 0; do
  echo "== half_tail=$ht" >> gpurun_out/kb_$tag.log
  AQB_GEMM_HALF_TAIL=$ht timeout 300 python scripts/kernel_bench.py --only gemm-n2048 >> gpurun_out/kb_$tag.log 2>&1
  AQB_GEMM_HALF_TAIL=$ht timeout 300 python scripts/kernel_bench.py --only gemm >> gpurun_out/kb_$tag.log 2>&1
  AQB_GEMM_HALF_TAIL=$ht timeout 300 python scripts/kernel_bench.py --only gemm-small >> gpurun_out/kb_$tag.log 2>&1
done
timeout 300 python scripts/kernel_bench.py --only attn >> gpurun_out/kb_$tag.log 2>&1
timeout 600 python bench.py --no-cpu > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
echo "bench_rc=$?" >> gpurun_out/bench_$tag.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm2 -o gpurun_out/ncu_gemm_proj_$tag python scripts/kernel_bench.py --only gemm-proj --ncu > gpurun_out/ncu_$tag.log 2>&1
