mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm2 -c 8 -o gpurun_out/ncu_gemm_small python scripts/kernel_bench.py --only gemm-small --ncu > gpurun_out/ncu_gemm_small.log 2>&1
