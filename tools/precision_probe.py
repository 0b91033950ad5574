"""Precision probe: per-gradient error of the F=200 / D=128 GAT case against the
float64 oracle, with the same metric as tests/helpers.assert_grads_close (shows
how close the analytically-zero attention gradients sit to the 1e-4 bar).
Run from the repo root on a GPU box: python tools/precision_probe.py"""
import os, sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, "tests/golden"); sys.path.insert(0, ".")
from test_gpu_wide import _run
from oracle.coop_oracle import CoopRun
from oracle.model_oracle import glorot_params
from oracle.split_oracle import split_sample
from helpers import rel_err
for g in (1, 2):
    sg, graph, pm, sample, cache, feats, labels, params, splits, ex, loss, grads = _run("gat", g, 200, 128, 9, 95 + g)
    ws, wp = split_sample(sample.layer_vertices, sample.layer_edges, pm.assignment, g, cache.cached)
    ref = CoopRun(glorot_params("gat", 200, 128, 9, 3, seed=5), ws, wp, feats.astype(np.float64), labels)
    rloss, rgrads = ref.run()
    worst = []
    for d in range(g):
        want = rgrads[d]
        gmax = max(float(np.abs(np.asarray(v)).max(initial=0.0)) for v in want.values())
        for k, w in want.items():
            w = np.asarray(w, dtype=np.float64); gg = np.asarray(grads[d][k], dtype=np.float64)
            scale = max(float(np.abs(w).max(initial=0.0)), 1e-3 * gmax, 1e-12)
            worst.append((round(float(np.abs(gg - w).max(initial=0.0)) / scale, 7), d, k, float(np.abs(w).max()) / gmax))
    worst = sorted(worst, reverse=True)[:3]
    print(os.environ.get("SG_NO_MMA", "mma"), g, abs(loss - rloss) / abs(rloss), worst)
