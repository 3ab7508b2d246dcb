#!/bin/bash
# In-model sweep of the env switches under the board power cap (config 2, N=1, no MM-DiT):
#   gpurun -- bash scripts/knob_sweep.sh <tag>
tag=${1:-sweep}
mkdir -p gpurun_out
out=gpurun_out/knob_sweep_$tag.jsonl
: > $out
run() {
  line=$(env "$@" timeout 300 python bench.py --no-mmdit --no-cpu 2>/dev/null | tail -1)
  python -c "import json,sys; d=json.loads(sys.argv[2]); print(json.dumps({'env': sys.argv[1], 'value': d['value'], 'sm_mhz': d['clocks']['sm_mhz'], 'attn': d['kernels']['attention']['tflops'], 'norm_gbs': d['kernels']['norm_modulate']['gbs']}))" "$*" "$line" >> $out
}
run AQB_X=default
for p in 0 2 4; do run AQB_ATTN_POLY=$p; done
for v in 2 8; do run AQB_NORM_VPT=$v; done
for c in 4 12; do run AQB_NORM_CTAS_PER_SM=$c; done
run AQB_X=default
