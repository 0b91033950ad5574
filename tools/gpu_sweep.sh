#!/bin/bash
# Measurement rows beyond the headline: batch sweep, g = 8 split parts on
# one GPU (the real multi-part splitter + exchange copy kernels), C1, C4 with a partial
# feature cache (misses staged from host memory), C3 with the layer-1 weight-gradient
# launch captured by ncu.  Usage: tools/gpu_sweep.sh TAG
TAG=${1:-r}
mkdir -p gpurun_out
run() {  # name, args...
  local name=$1; shift
  timeout ${BENCH_TIMEOUT:-900} python bench.py "$@" > gpurun_out/${TAG}_sweep_${name}.json 2> gpurun_out/${TAG}_sweep_${name}.err
  echo "$name rc=$? $(python -c "import json,sys; d=json.load(open('gpurun_out/${TAG}_sweep_${name}.json')); print(round(d['ms_per_step'],4), 'ms', '%.3g' % d['value'], d['unit'], 'frac', d.get('roofline',{}).get('frac'), 'parity', (d.get('parity') or {}).get('ok'))" 2>/dev/null)"
}
run c2_b1024 --config c2
run c2_b4096 --config c2 --batch 4096 --steps 10
run c2_b16384 --config c2 --batch 16384 --steps 6 --warmup 3
run c2_g8 --config c2 --parts 8
run c1 --config c1
run c2_cache025 --config c2 --cache 0.25
free -g > gpurun_out/${TAG}_free.txt; nproc >> gpurun_out/${TAG}_free.txt
MEMG=$(free -g | awk '/Mem:/ {print $7}')
if [ "${MEMG:-0}" -gt 150 ]; then  # C4's 57 GB host feature matrix (mapped) + graph
  run c4_cache0125 --config c4 --cache 0.125 --steps 10 --warmup 3
else
  echo "c4_cache0125 skipped: ${MEMG} GB available"
fi
run c3 --config c3
