timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do timeout 120 python bench.py --no-cpu-baseline --steps 20 2>gpurun_out/e.err | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(round(d['ms_per_step'],4),'agg1',round(d['roofline']['avg_launch_ms'],4), round(d['roofline']['frac'],3),'e2e',round(d['e2e']['ms_per_step'],4), d['loss_last'], d['gpu_launches'], d['phases_ms'])"; done
