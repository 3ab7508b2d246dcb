R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 $R --nproc-per-node 4 --master-port 29741 bench.py --gpus 4 --no-cpu --parallel tp > gpurun_out/bench_tp_n4.json 2> gpurun_out/bench_tp_n4.err
