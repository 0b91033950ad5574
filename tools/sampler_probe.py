"""Diagnostic: GPU sampler time on the C2 graph (events), per-kernel under ncu."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2303_13775_b200 as sg  # noqa: E402

graph, labels, train, _ = bench.build_workload(16)
samples, _ = bench.make_samples(graph, train, 6, bench.BATCH, 16)
gs = sg.GpuSampler(graph)
from paper_2303_13775_b200.engine import StaticSample, capacities_for  # noqa: E402
cap_nV, cap_nE = capacities_for(samples)
inp = StaticSample(cap_nV, cap_nE, "cuda")
for i, (t, sd) in enumerate(bench.PLAN):
    tt = torch.from_numpy(np.asarray(t, np.int64)).cuda()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    gs.sample_into(tt, bench.FANOUTS, sd, inp.V, inp.es, inp.ed, inp.sizes, inp.voff, inp.eoff)
    e1.record()
    torch.cuda.synchronize()
    print(f"sample {i}: {e0.elapsed_time(e1) * 1e3:.1f} us, err {int(gs.err.item())}")
