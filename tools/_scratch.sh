for nb in 296 592 888 296 592; do SG_NBP=$nb timeout 300 python bench.py --no-cpu-baseline --steps 20 2>>gpurun_out/e.err | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);p=d['phases_ms'];print('nb=$nb', round(d['ms_per_step'],4), d['loss_last'], p['bwd_rows1'], p['reduce'])" >> gpurun_out/nbp.txt; done
cat gpurun_out/nbp.txt
