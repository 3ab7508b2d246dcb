R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_model_gpu.py -m gpu -x -q -k "tp_sp" > gpurun_out/pytest_tp_mm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tp_mm.log
timeout 900 $R --nproc-per-node 2 --master-port 29731 scripts/tp_check.py > gpurun_out/tpcheck_mm_p2.log 2>&1; echo "rc=$?" >> gpurun_out/tpcheck_mm_p2.log
AQB_OVERSUBSCRIBE=1 timeout 900 $R --nproc-per-node 8 --master-port 29732 scripts/tp_check.py > gpurun_out/tpcheck_mm_p8_oversub.log 2>&1; echo "rc=$?" >> gpurun_out/tpcheck_mm_p8_oversub.log
