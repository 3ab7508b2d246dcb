# AQB_GEMM_VARIANT sweep of kernel_bench cases (--only gemm-variants; gemm-small for the 1/4 and 1/8 shards)
for v in default 2cta256 2cta128; do
  if [ $v = default ]; then unset AQB_GEMM_VARIANT; else export AQB_GEMM_VARIANT=$v; fi
  timeout 120 python scripts/kernel_bench.py --only gemm-variants | sed "s/^{/{\"variant\": \"$v\", /" >> gpurun_out/kb_gemm_variants2.log 2>&1
done
