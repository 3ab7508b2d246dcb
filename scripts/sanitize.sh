#!/bin/bash
# compute-sanitizer over every kernel class (tiny shapes) and the 2-rank peer exchange.
#   gpurun -- bash scripts/sanitize.sh
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 $CS --tool $tool --print-limit 50 python scripts/sanitize_kernels.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
done
# 2 ranks on one GPU: peer barrier, scatter epilogues, TMA reduce-add into peer memory
for tool in memcheck synccheck; do
  AQB_OVERSUBSCRIBE=1 timeout 1800 $CS --tool $tool --target-processes all --print-limit 50 \
    python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29811 \
    tests/mp_parity.py --parallel ulysses --cases single --out gpurun_out/sanitize_mp_$tool.jsonl \
    > gpurun_out/sanitize_mp_ulysses_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_mp_ulysses_$tool.log
  AQB_OVERSUBSCRIBE=1 timeout 1800 $CS --tool $tool --target-processes all --print-limit 50 \
    python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29812 \
    tests/mp_parity.py --parallel tp --cases single --out gpurun_out/sanitize_mp_tp_$tool.jsonl \
    > gpurun_out/sanitize_mp_tp_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_mp_tp_$tool.log
done
