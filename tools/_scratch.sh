timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for p in 1 1 1; do SG_PDL=$p timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 20 2>>gpurun_out/e.err | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);p=d['phases_ms'];print('pdl=$p', round(d['ms_per_step'],4), d['loss_last'], d['e2e_with_sampling']['ms_per_step'], p['project1'], p['bwd_param1'])"; done
for v in 1; do SG_NO_MMA=1 timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 20 2>>gpurun_out/e.err | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);p=d['phases_ms'];print('nomma', round(d['ms_per_step'],4), d['loss_last'], p['project1'])"; done
