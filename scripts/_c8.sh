mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r1f.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_gpu_r1f.log
for sq in 1 0; do
  echo "== splitqk=$sq" >> gpurun_out/attn_sqk.log
  AQB_ATTN_SPLITQK=$sq timeout 300 python scripts/kernel_bench.py --only attn >> gpurun_out/attn_sqk.log 2>&1
done
timeout 300 python scripts/kernel_bench.py --only gemm-small > gpurun_out/gemm_small_r1f.log 2>&1
timeout 600 python bench.py --no-cpu > gpurun_out/bench_r1f.json 2> gpurun_out/bench_r1f.err
