# 8-rank parity (ranks share the box's GPUs round-robin, gloo plumbing, p2p exchange unchanged)
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 8"
for par in ulysses tp; do
  AQB_OVERSUBSCRIBE=1 timeout 1500 $R --master-port 29801 tests/mp_parity.py --parallel $par \
    --out gpurun_out/mp_p8_$par.jsonl > gpurun_out/mp_p8_$par.log 2>&1; echo "rc=$?" >> gpurun_out/mp_p8_$par.log
done
