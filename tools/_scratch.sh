rm -f gpurun_out/bis.txt
run() { for i in 1 2 3; do SG_PDL_DENY="$1" SG_GAT_PDL=1 timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 20 2>>gpurun_out/e.err | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('deny=$1', d['loss_last'])" >> gpurun_out/bis.txt; done; }
run "none"
run "gat.cu"
run "tspmm.cu,sort.cu"
run "loss.cu,split.cu,features.cu,exchange.cu,dense.cu"
cat gpurun_out/bis.txt
