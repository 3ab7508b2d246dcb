timeout 600 python -m pytest tests/test_kernels_gpu.py -q -k "attention" > gpurun_out/pytest_attn_mb2.log 2>&1; echo rc=$? >> gpurun_out/pytest_attn_mb2.log
timeout 300 python scripts/kernel_bench.py --only attn-cross > gpurun_out/kb_cross2.log 2>&1
