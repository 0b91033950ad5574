"""Partition the products-shape graph (C2: 2.45M vertices, 61.9M edges) into
g = 2 / 4 / 8 parts with the GPU multilevel partitioner; cut and balance vs the
contiguous range map the benchmarks use, and the time. GPU box:
    python tools/partition_scale.py"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2303_13775_b200 as sg  # noqa: E402

n, m = 2_449_029, 61_859_140
graph = sg.generate_powerlaw(n, m, blocks=64, p_local=0.92, seed=0)
out = []
for g in (2, 4, 8):
    torch.cuda.synchronize()
    t = time.perf_counter()
    pm = sg.partition_graph(graph, g, 0.05, seed=1)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    cut = sg.cut_size(graph, pm)
    rng = sg.cut_size(graph, sg.range_partition(n, g))
    rec = {"g": g, "seconds": round(dt, 2), "cut": cut, "cut_frac": cut / m, "range_cut": rng,
           "range_cut_frac": rng / m, "max_part": int(pm.counts().max()), "cap": sg.max_part_size(n, g, 0.05),
           "peak_gpu_GB": round(torch.cuda.max_memory_allocated() / 1e9, 2)}
    print(json.dumps(rec), flush=True)
    out.append(rec)
