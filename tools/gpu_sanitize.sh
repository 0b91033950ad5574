#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over GPU parity tests.  Usage: tools/gpu_sanitize.sh TAG
TAG=${1:-r}
mkdir -p gpurun_out
CS="compute-sanitizer --target-processes all --error-exitcode 99 --print-limit 50"
T_MEM=${T_MEM:-"tests/test_gpu_split.py tests/test_gpu_sage.py tests/test_gpu_gat.py tests/test_gpu_cache_miss.py tests/test_gpu_small_rows.py tests/test_gpu_tspmm.py tests/test_gpu_sampler.py tests/test_gpu_graph.py"}
T_RACE=${T_RACE:-"tests/test_gpu_sage.py tests/test_gpu_gat.py tests/test_gpu_split.py"}
timeout ${MEM_TIMEOUT:-1500} $CS --tool memcheck --leak-check no python -m pytest $T_MEM -m gpu -x -q -p no:cacheprovider \
   > gpurun_out/${TAG}_memcheck.log 2>&1; echo "memcheck rc=$?" | tee -a gpurun_out/${TAG}_memcheck.log
tail -4 gpurun_out/${TAG}_memcheck.log
timeout ${RACE_TIMEOUT:-1200} $CS --tool racecheck --racecheck-report hazard python -m pytest $T_RACE -m gpu -x -q -p no:cacheprovider \
   > gpurun_out/${TAG}_racecheck.log 2>&1; echo "racecheck rc=$?" | tee -a gpurun_out/${TAG}_racecheck.log
tail -4 gpurun_out/${TAG}_racecheck.log
timeout ${SYNC_TIMEOUT:-600} $CS --tool synccheck python -m pytest tests/test_gpu_sage.py tests/test_gpu_gat.py -m gpu -x -q -p no:cacheprovider \
   > gpurun_out/${TAG}_synccheck.log 2>&1; echo "synccheck rc=$?" | tee -a gpurun_out/${TAG}_synccheck.log
tail -4 gpurun_out/${TAG}_synccheck.log
