for v in auto 2cta256 2cta128 1cta256 1cta128; do
  if [ $v = auto ]; then timeout 300 python scripts/gemm_bench.py > gpurun_out/gemm_$v.jsonl 2>&1
  else AQB_GEMM_VARIANT=$v timeout 300 python scripts/gemm_bench.py > gpurun_out/gemm_$v.jsonl 2>&1; fi
done
