#!/bin/bash
# Extra measurement rows: C4 split into 8 parts on one GPU (each part's feature
# cache holds its own partition: north_star's "8 GPUs with partitioned feature
# cache" with the exchanges as copy kernels), and the C2 batch sweep continued.
# Usage: tools/gpu_extra.sh TAG
TAG=${1:-r}
mkdir -p gpurun_out
run() {
  local name=$1; shift
  timeout ${BENCH_TIMEOUT:-1500} python bench.py "$@" > gpurun_out/${TAG}_extra_${name}.json 2> gpurun_out/${TAG}_extra_${name}.err
  echo "$name rc=$? $(python -c "import json; d=json.load(open('gpurun_out/${TAG}_extra_${name}.json')); print(round(d['ms_per_step'],4), 'ms', '%.3g' % d['value'], d['unit'], 'frac', d.get('roofline',{}).get('frac'), 'parity', (d.get('parity') or {}).get('ok'))" 2>/dev/null)"
}
run c4_g8 --config c4 --parts 8 --steps 10 --warmup 3 --no-api-leg
run c2_b65536 --config c2 --batch 65536 --steps 5 --warmup 3 --no-api-leg
run c3_b4096 --config c3 --batch 4096 --steps 10 --warmup 3 --no-api-leg
