mkdir -p gpurun_out
rm -f gpurun_out/ucheck_bisect.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for cfg in "AQB_X=1" "AQB_GEMM_GATE_ADD=0" "AQB_GEMM_GATE_ADD=0 AQB_GEMM_HALF_TAIL=0" "AQB_GEMM_VARIANT=2cta256" "AQB_PDL=0"; do
  echo "== $cfg" >> gpurun_out/ucheck_bisect.log
  env $cfg timeout 600 $R --nproc-per-node 2 --master-port 29641 scripts/ulysses_check.py 2>&1 | grep '^{' | grep p2p >> gpurun_out/ucheck_bisect.log
done
