#!/bin/bash
# racecheck with every hazard printed, reduced to its distinct (kernel, line) sites.
# Usage: tools/race_sites.sh TAG test-files...
TAG=$1; shift
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --target-processes all --tool racecheck --racecheck-report hazard --print-limit 0 \
  python -m pytest "$@" -m gpu -q -p no:cacheprovider > /tmp/race_full.log 2>&1
echo "racecheck rc=$?" > gpurun_out/${TAG}_race_sites.txt
grep -E "RACECHECK SUMMARY|passed|failed" /tmp/race_full.log | tail -3 >> gpurun_out/${TAG}_race_sites.txt
grep -E "^=========     (Write|Read) Thread" /tmp/race_full.log | sed -E 's/Thread \([0-9]+,[0-9]+,[0-9]+\)/Thread/; s/\+0x[0-9a-f]+//' \
  | sort | uniq -c | sort -rn >> gpurun_out/${TAG}_race_sites.txt
grep -E "^========= (Warning|Error)" /tmp/race_full.log | sed -E 's/at __shared__ 0x[0-9a-f]+ in block \([0-9,]+\)//' \
  | sort | uniq -c | sort -rn | head -20 >> gpurun_out/${TAG}_race_sites.txt
