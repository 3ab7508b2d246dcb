mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $R --nproc-per-node 2 --master-port 29631 scripts/ulysses_check.py > gpurun_out/ucheck_p2_r1h.log 2>&1; echo "rc=$?" >> gpurun_out/ucheck_p2_r1h.log
timeout 600 $R --nproc-per-node 2 --master-port 29632 scripts/tp_check.py > gpurun_out/tpcheck_p2_r1h.log 2>&1; echo "rc=$?" >> gpurun_out/tpcheck_p2_r1h.log
timeout 900 $R --nproc-per-node 2 --master-port 29633 bench.py --gpus 2 --no-cpu > gpurun_out/bench_n2_r1h.json 2> gpurun_out/bench_n2_r1h.err
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r1h.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_gpu_r1h.log
