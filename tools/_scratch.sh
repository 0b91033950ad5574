for i in 1 2; do for v in 0 2 3 4; do SG_SAGE_LAYER=$v timeout 300 python bench.py --no-cpu-baseline --steps 20 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('v=$v',round(d['ms_per_step'],4),'agg1',round(d['roofline']['avg_launch_ms'],4),'e2e',round(d['e2e']['ms_per_step'],4))"; done; done
