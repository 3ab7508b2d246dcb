R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python bench.py > gpurun_out/bench_f5_n1.json 2> gpurun_out/bench_f5_n1.err
timeout 900 $R --nproc-per-node 2 --master-port 29771 bench.py --gpus 2 > gpurun_out/bench_f5_n2.json 2> gpurun_out/bench_f5_n2.err
timeout 1200 $R --nproc-per-node 4 --master-port 29772 bench.py --gpus 4 > gpurun_out/bench_f5_n4.json 2> gpurun_out/bench_f5_n4.err
timeout 900 $R --nproc-per-node 4 --master-port 29773 scripts/ulysses_check.py > gpurun_out/ucheck_f5_n4.log 2>&1; echo "rc=$?" >> gpurun_out/ucheck_f5_n4.log
