mkdir -p gpurun_out
AQB_ATTN_STREAMK=1 timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -x -q -k "attention" > gpurun_out/pytest_sk_forced.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sk_forced.log
AQB_ATTN_STREAMK=1 timeout 600 python -m pytest tests/test_model_gpu.py -m gpu -x -q > gpurun_out/pytest_sk_forced_model.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sk_forced_model.log
for sk in 0 1; do
  echo "== streamk=$sk" >> gpurun_out/attn_sk.log
  AQB_ATTN_STREAMK=$sk timeout 300 python scripts/kernel_bench.py --only attn-ranks >> gpurun_out/attn_sk.log 2>&1
done
