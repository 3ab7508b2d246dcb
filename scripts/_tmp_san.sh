bash scripts/sanitize.sh
NCU=/usr/local/cuda/bin/ncu
for c in "xproj 1950 2048 2048" "proj 1950 2048 2048" "fc2 1950 2048 8192"; do
  set -- $c
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemm -s 4 -c 1 -o gpurun_out/ncu_gemm_$1_$2 -f python scripts/gemm_bench.py --ncu $1 $2 $3 $4 > gpurun_out/ncu_gemm_$1_$2.log 2>&1
done
