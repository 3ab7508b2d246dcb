mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_r1g_n1.json 2> gpurun_out/bench_r1g_n1.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1g.csv python scripts/profile_step.py > gpurun_out/ncu_launch_r1g.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm2 -c 4 -o gpurun_out/ncu_gemm_r1g python scripts/kernel_bench.py --only gemm --ncu > gpurun_out/ncu_gemm_r1g.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_fwd -c 1 -o gpurun_out/ncu_attn_r1g python scripts/kernel_bench.py --only attn --ncu > gpurun_out/ncu_attn_r1g.log 2>&1
