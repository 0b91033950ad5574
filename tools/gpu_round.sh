#!/bin/bash
# One gpurun call: GPU parity tests, the C2 bench line, the ncu launch list and
# one --set full capture of the layer-1 kernels.  Usage: tools/gpu_round.sh TAG [CONFIG]
TAG=${1:-r}
CFG=${2:-c2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py --config $CFG > gpurun_out/${TAG}_bench_${CFG}.json 2> gpurun_out/${TAG}_bench_${CFG}.err; echo "bench rc=$?"
tail -c 600 gpurun_out/${TAG}_bench_${CFG}.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_${CFG}.csv \
   python bench.py --config $CFG --profile --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${KREGEX:-k_sage_layer|k_sage_wgrad|k_sage_final|k_tspmm|k_reduce_partials}" -c ${KCOUNT:-8} \
   -o gpurun_out/${TAG}_full_${CFG} -f python bench.py --config $CFG --profile --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
