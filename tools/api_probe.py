"""Host-cost breakdown of the reference-API loop (split_minibatch ->
SplitExecutor.run -> allreduce_and_step) on C2-shaped samples. GPU box:
    python tools/api_probe.py"""
import cProfile
import os
import pstats
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2303_13775_b200 as sg  # noqa: E402

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
T = {"split": 0.0, "exec_init": 0.0, "run": 0.0, "allreduce": 0.0}


def step(smp):
    t0 = time.perf_counter()
    splits, plan = sg.split_minibatch(smp, pm, cache)
    t1 = time.perf_counter()
    ex = sg.SplitExecutor(params, splits, plan, feats, labels)
    t2 = time.perf_counter()
    loss, grads = ex.run()
    t3 = time.perf_counter()
    sg.allreduce_and_step(params, grads, 0.1, len(smp.targets))
    t4 = time.perf_counter()
    for k, a, b in (("split", t0, t1), ("exec_init", t1, t2), ("run", t2, t3), ("allreduce", t3, t4)):
        T[k] += b - a
    return loss


for smp in samples[:10]:
    step(smp)
torch.cuda.synchronize()
for k in T:
    T[k] = 0.0
t = time.perf_counter()
for smp in samples[10:]:
    step(smp)
torch.cuda.synchronize()
t = time.perf_counter() - t
print(f"api loop: {1e3 * t / 20:.3f} ms/step; " + ", ".join(f"{k} {1e3 * v / 20:.3f}" for k, v in T.items()))
# the same loop with a device synchronise after every call: wall time of each
# call INCLUDING the GPU work it queued
S = {"split+h2d": 0.0, "exec_init": 0.0, "replay": 0.0, "allreduce": 0.0}
for smp in samples[10:]:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    splits, plan = sg.split_minibatch(smp, pm, cache)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ex = sg.SplitExecutor(params, splits, plan, feats, labels)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    loss, grads = ex.run()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    sg.allreduce_and_step(params, grads, 0.1, len(smp.targets))
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    for k, a, b in (("split+h2d", t0, t1), ("exec_init", t1, t2), ("replay", t2, t3), ("allreduce", t3, t4)):
        S[k] += b - a
print("synchronised: " + ", ".join(f"{k} {1e3 * v / 20:.3f}" for k, v in S.items()) +
      f" ms; packed words {splits.device_split.packed[1]}, geometry words {splits.device_split.packed[2].words}")
# pieces of split_minibatch: native pack into the pinned slot; the H2D copy alone
from paper_2303_13775_b200.scheduler import _PINNED, PackGeometry  # noqa: E402
geo = splits.device_split.packed[2]
dst = torch.empty(geo.words, dtype=torch.int32, device="cuda")
tp = th = 0.0
for smp in samples[10:]:
    t0 = time.perf_counter()
    hb, used = _PINNED.pack(geo, smp)
    t1 = time.perf_counter()
    dst[:used].copy_(hb[:used], non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    tp += t1 - t0
    th += t2 - t1
print(f"pack {1e3 * tp / 20:.3f} ms, H2D {1e3 * th / 20:.3f} ms for {4 * used / 1e6:.2f} MB "
      f"({4 * used / (th / 20) / 1e9:.1f} GB/s)")


def h2d_only(buf, k=20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        dst[:used].copy_(buf[:used], non_blocking=True)
        torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t0) / k


print(f"H2D only, ring slot: {h2d_only(hb):.3f} ms")
fresh = torch.empty(geo.words, dtype=torch.int32, pin_memory=True)
fresh.numpy()[:used] = hb.numpy()[:used]
print(f"H2D only, fresh pinned buffer: {h2d_only(fresh):.3f} ms")
print(f"H2D only, ring slot again: {h2d_only(hb):.3f} ms; slot is_pinned {hb.is_pinned()} "
      f"data_ptr {hb.data_ptr():#x} numel {hb.numel()}")
d2 = torch.empty(geo.words, dtype=torch.int32, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    d2[:used].copy_(hb[:used], non_blocking=True)
    torch.cuda.synchronize()
print(f"H2D only into a fresh device buffer: {1e3 * (time.perf_counter() - t0) / 20:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for smp in samples[10:]:
    step(smp)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
