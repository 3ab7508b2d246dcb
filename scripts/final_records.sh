# Round-end records on a 4-GPU box: bench N=1/2/4 (full JSON line), the reference arm,
# Ulysses parity at P=4, the ncu launch list of the bench command and an ncu --set full
# capture of the attention kernels (self 7800x7800x16 and cross 7800x256x16).
T=${1:-f6}
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python bench.py > gpurun_out/bench_${T}_n1.json 2> gpurun_out/bench_${T}_n1.err
timeout 900 $R --nproc-per-node 2 --master-port 29771 bench.py --gpus 2 > gpurun_out/bench_${T}_n2.json 2> gpurun_out/bench_${T}_n2.err
timeout 1200 $R --nproc-per-node 4 --master-port 29772 bench.py --gpus 4 > gpurun_out/bench_${T}_n4.json 2> gpurun_out/bench_${T}_n4.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_${T}_ref.json 2> gpurun_out/bench_${T}_ref.err
timeout 900 $R --nproc-per-node 4 --master-port 29773 tests/mp_parity.py --parallel ulysses --out gpurun_out/mp_${T}_n4.jsonl > gpurun_out/ucheck_${T}_n4.log 2>&1; echo "rc=$?" >> gpurun_out/ucheck_${T}_n4.log
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2600 --csv \
  --log-file gpurun_out/launches_bench_${T}.csv python bench.py --steps 1 --warmup 3 --no-mmdit --no-cpu > gpurun_out/ncu_launch_${T}.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -c 2 \
  -o gpurun_out/attn_${T} python scripts/kernel_bench.py --only attn --ncu > gpurun_out/ncu_attn_${T}.log 2>&1
