mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r1i.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_gpu_r1i.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench_r1i_n1.json 2> gpurun_out/bench_r1i_n1.err
timeout 900 $R --nproc-per-node 4 --master-port 29671 bench.py --gpus 4 --no-cpu > gpurun_out/bench_r1i_n4.json 2> gpurun_out/bench_r1i_n4.err
timeout 600 $R --nproc-per-node 2 --master-port 29672 bench.py --gpus 2 --no-cpu --no-mmdit > gpurun_out/bench_r1i_n2.json 2> gpurun_out/bench_r1i_n2.err
