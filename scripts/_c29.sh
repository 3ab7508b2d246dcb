mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_final.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_final.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_final.log
timeout 600 python bench.py > gpurun_out/bench_final_n1.json 2> gpurun_out/bench_final_n1.err
timeout 900 $R --nproc-per-node 2 --master-port 29701 bench.py --gpus 2 > gpurun_out/bench_final_n2.json 2> gpurun_out/bench_final_n2.err
timeout 1200 $R --nproc-per-node 4 --master-port 29702 bench.py --gpus 4 > gpurun_out/bench_final_n4.json 2> gpurun_out/bench_final_n4.err
timeout 900 $R --nproc-per-node 4 --master-port 29703 scripts/ulysses_check.py > gpurun_out/ucheck_final_n4.log 2>&1; echo "rc=$?" >> gpurun_out/ucheck_final_n4.log
timeout 900 $R --nproc-per-node 4 --master-port 29704 scripts/tp_check.py > gpurun_out/tpcheck_final_n4.log 2>&1; echo "rc=$?" >> gpurun_out/tpcheck_final_n4.log
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python scripts/profile_step.py > gpurun_out/ncu_launch_final.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm2 -c 2 -o gpurun_out/ncu_qkv_final python scripts/kernel_bench.py --only qkv --ncu > gpurun_out/ncu_qkv_final.log 2>&1
