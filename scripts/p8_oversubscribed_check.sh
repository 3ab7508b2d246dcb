# 8-rank correctness on a 4-GPU box (2 ranks per GPU, gloo plumbing, p2p exchange unchanged)
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 8"
AQB_OVERSUBSCRIBE=1 timeout 1500 $R --master-port 29801 scripts/ulysses_check.py > gpurun_out/ucheck_p8_os.log 2>&1; echo "rc=$?" >> gpurun_out/ucheck_p8_os.log
AQB_OVERSUBSCRIBE=1 timeout 1200 $R --master-port 29802 scripts/tp_check.py > gpurun_out/tpcheck_p8_os.log 2>&1; echo "rc=$?" >> gpurun_out/tpcheck_p8_os.log
