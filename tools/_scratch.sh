rm -f gpurun_out/nar.txt
for v in 0 1 0 1; do SG_LAYER_NARROW=$v timeout 300 python bench.py --no-cpu-baseline --steps 20 2>>gpurun_out/e.err | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);p=d['phases_ms'];print('narrow=$v', round(d['ms_per_step'],4), d['loss_last'], p['agg+update2'])" >> gpurun_out/nar.txt; done
cat gpurun_out/nar.txt
