SG_BENCH_HOST_STAGED=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/n2p.json 2> gpurun_out/n2p.err; echo rc=$?
grep -v "^frame" gpurun_out/n2p.err | grep -v "^\*\*\*\|OMP_NUM" | tail -5; python -c "
import json;d=json.loads(open('gpurun_out/n2p.json').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['e2e'], d['gpu_launches'], d['loss_last'], d['config']['parallelism'], d['phases_ms'])"
