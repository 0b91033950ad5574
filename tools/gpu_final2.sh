#!/bin/bash
# Round-2 evidence in one gpurun call: GPU tests, smoke, sanitizers on the round-2
# kernels, the bench sweep, the reference arm, ncu launch lists and full captures.
# Usage: tools/gpu_final2.sh TAG
TAG=${1:-r}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,pcie.link.gen.current,pcie.link.width.current --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
T_MEM="tests/test_gpu_partition.py tests/test_gpu_gat.py tests/test_gpu_api.py tests/test_gpu_sage.py tests/test_gpu_tspmm.py" \
T_RACE="tests/test_gpu_gat.py tests/test_gpu_partition.py tests/test_gpu_sage.py" MEM_TIMEOUT=1200 RACE_TIMEOUT=1200 \
  bash tools/gpu_sanitize.sh ${TAG}
bash tools/gpu_sweep.sh ${TAG}
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err; echo "ref rc=$?"
timeout 1500 python bench.py --config c4 --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err; echo "c4 rc=$?"
for c in c2 c3; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_${c}.csv \
     python bench.py --config $c --profile --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu launches $c rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_sage_layer|k_sage_wgrad|k_sage_final|k_sage_scatter|k_reduce_partials" -c 7 \
   -o gpurun_out/${TAG}_full_c2 -f python bench.py --config c2 --profile --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu full c2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_gat_project_tc|k_gat_agg|k_gat_bwd_dst|k_gat_wgrad_dst|k_gat_wgrad_mma|k_gat_bwd_src" -c 14 \
   -o gpurun_out/${TAG}_full_c3 -f python bench.py --config c3 --profile --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu full c3 rc=$?"
