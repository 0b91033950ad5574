"""Host-time breakdown of split_minibatch's direct (pinned-sample) path and of
allreduce_and_step's host SGD, C2-shaped samples. GPU box:
    python tools/api_probe2.py"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2303_13775_b200 as sg  # noqa: E402
from paper_2303_13775_b200 import engine, scheduler  # noqa: E402
from paper_2303_13775_b200.scheduler import DeviceSplit, PackGeometry, _lazy_views  # noqa: E402

n, m = 2_449_029, 61_859_140
graph = sg.generate_powerlaw(n, m, blocks=64, p_local=0.92, seed=0)
labels = sg.synthetic_labels(n, 47, seed=2)
pm = sg.range_partition(n, 1)
cache = sg.full_cache(pm)
feats = sg.FeatureStore.synthetic(n, 100, 1, pad_rows=True)
sampler = sg.NativeSampler(graph)
rng = np.random.default_rng(3)
samples = [sampler.sample(rng.choice(n, 1024, replace=False), [15, 10, 5], i) for i in range(30)]
params = sg.init_params("graphsage", 100, 16, 47, 3, seed=0)
T = {}


def tick(k, t0):
    t1 = time.perf_counter()
    T[k] = T.get(k, 0.0) + t1 - t0
    return t1


def split(smp):
    t = time.perf_counter()
    smp = sg.sampling.as_sample(smp)
    ok = smp.pinned.intact(smp)
    t = tick("intact", t)
    stage = scheduler._h2d_pinned(smp.pinned, torch.device("cuda"))
    t = tick("h2d", t)
    nV, nE = smp.sizes()
    geo = PackGeometry.for_sizes(nV, nE, scope=(len(nE), len(pm.assignment), pm.num_devices))
    t = tick("geometry", t)
    buf = torch.empty(geo.words, dtype=torch.int32, device="cuda")
    t = tick("empty", t)
    used = geo.relayout_from_stage(smp, smp.pinned, stage, buf, nE)
    t = tick("relayout", t)
    VC = int(geo.voff[-1])
    ds = DeviceSplit(None, None, None, geo.cap_nV, geo.cap_nE, pm, cache, True, torch.device("cuda"), host_V=None,
                     defer=True, views=lambda: (buf[geo.o_V:geo.o_V + VC], buf[geo.o_es:geo.o_es + geo.EC],
                                                buf[geo.o_ed:geo.o_ed + geo.EC], buf[:geo.S].view(torch.int64)))
    ds.packed = (buf, used, geo)
    ds.num_targets = len(smp.targets)
    t = tick("DeviceSplit", t)
    r = _lazy_views(ds)
    tick("views", t)
    return r, ok


def step(smp):
    t = time.perf_counter()
    (splits, plan), ok = split(smp)
    t = tick("split", t)
    ex = sg.SplitExecutor(params, splits, plan, feats, labels)
    t = tick("executor", t)
    loss, grads = ex.run()
    t = tick("run", t)
    sg.allreduce_and_step(params, grads, 0.1, len(smp.targets))
    tick("allreduce", t)
    return ok


for smp in samples[:10]:
    assert step(smp)
torch.cuda.synchronize()
T.clear()
t0 = time.perf_counter()
for smp in samples[10:]:
    step(smp)
torch.cuda.synchronize()
t = time.perf_counter() - t0
print(f"loop {1e3 * t / 20:.3f} ms/step: " + ", ".join(f"{k} {1e6 * v / 20:.1f}us" for k, v in T.items()))
hp = params
T.clear()
for _ in range(20):
    t = time.perf_counter()
    a = engine._host_flat(hp)
    t = tick("host_flat", t)
    np.array_equal(a, a.copy())
    tick("array_equal", t)
print(", ".join(f"{k} {1e6 * v / 20:.1f}us" for k, v in T.items()),
      {k: (v.dtype, v.shape) for k, v in list(hp.tensors().items())[:3]})
