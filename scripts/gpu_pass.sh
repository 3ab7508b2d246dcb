#!/bin/bash
# One GPU-box pass: parity tests, smoke, the contract bench line (+ optional reference arm).
#   gpurun -- bash scripts/gpu_pass.sh <tag> [ref]
tag=${1:-pass}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$tag.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_$tag.log 2>&1
echo "pytest_rc=$?" >> gpurun_out/pytest_gpu_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1
echo "smoke_rc=$?" >> gpurun_out/smoke_$tag.log
timeout 1200 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
echo "bench_rc=$?" >> gpurun_out/bench_$tag.err
if [ "$2" = "ref" ]; then
  timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err
  echo "ref_rc=$?" >> gpurun_out/bench_ref_$tag.err
fi
