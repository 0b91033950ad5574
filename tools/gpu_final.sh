#!/bin/bash
# End-of-round evidence: C2 round (tests, bench, launch list, ncu full), C3 bench + tensor-pipe capture,
# reference arm, C4 bench.  Usage: tools/gpu_final.sh TAG
TAG=${1:-r}
bash tools/gpu_round.sh $TAG c2
timeout 600 python bench.py --config c3 > gpurun_out/${TAG}_bench_c3.json 2>gpurun_out/${TAG}_bench_c3.err; echo "c3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_gat_project_tc|k_gat_wgrad_mma|k_gat_agg|k_gat_bwd_src" -c 8 \
   -o gpurun_out/${TAG}_full_c3 -f python bench.py --config c3 --profile --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2>gpurun_out/${TAG}_bench_ref.err; echo "ref rc=$?"
timeout 1200 python bench.py --config c4 --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_c4.json 2>gpurun_out/${TAG}_bench_c4.err; echo "c4 rc=$?"
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/${TAG}_smoke.log
