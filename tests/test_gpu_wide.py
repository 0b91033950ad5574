"""Layer widths outside the fused fast paths (hidden 64..256, wide inputs,
hidden*classes > 6144): the generic dense GEMMs (dense.cu) and the multi-pass
classifier keep every layer working like the reference (config.py:91-92
accepts any hidden >= 1). Parity vs the oracle, rel 1e-4."""

import numpy as np
import pytest

from helpers import assert_grads_close, random_partition_case, rel_err
from oracle.coop_oracle import CoopRun, reduce_and_sgd
from oracle.model_oracle import glorot_params
from oracle.multihead_oracle import multihead_run
from oracle.split_oracle import split_sample
from test_gpu_sage import TOL

pytestmark = pytest.mark.gpu


def _run(kind, g, F, hid, C, seed, heads=1, fanouts=(6, 5, 4)):
    import paper_2303_13775_b200 as sg
    graph, pm, sample, cache = random_partition_case(seed, n=4000, m=40000, g=g, batch=96,
                                                     fanouts=fanouts, cache_frac=0.25)
    feats = sg.synthetic_features(graph.num_vertices, F, seed=3)
    labels = sg.synthetic_labels(graph.num_vertices, C, seed=4)
    params = sg.init_params(kind, F, hid, C, len(fanouts), seed=5, heads=heads)
    splits, plan = sg.split_minibatch(sample, pm, cache)
    ex = sg.SplitExecutor(params, splits, plan, feats, labels)
    loss, grads = ex.run()
    return sg, graph, pm, sample, cache, feats, labels, params, splits, ex, loss, grads


@pytest.mark.parametrize("F,hid,C", [(100, 64, 47), (64, 128, 64), (100, 256, 30)])
@pytest.mark.parametrize("g", [1, 2])
def test_sage_wide_matches_oracle(F, hid, C, g):
    sg, graph, pm, sample, cache, feats, labels, params, splits, ex, loss, grads = _run(
        "graphsage", g, F, hid, C, 90 + g)
    ws, wp = split_sample(sample.layer_vertices, sample.layer_edges, pm.assignment, g, cache.cached)
    ref = CoopRun(glorot_params("graphsage", F, hid, C, 3, seed=5), ws, wp, feats.astype(np.float64), labels)
    rloss, rgrads = ref.run()
    assert abs(loss - rloss) <= TOL * abs(rloss)
    for d in range(g):
        assert_grads_close(grads[d], rgrads[d], TOL, d)
        for l in range(1, 4):
            assert rel_err(ex.states[d].h[l], ref.h[d][l]) < TOL, (d, l)


@pytest.mark.parametrize("g", [1, 2])
def test_gat_wide_input_matches_oracle(g):
    """F = 200 input, D = 128: dense projection and weight-gradient path."""
    sg, graph, pm, sample, cache, feats, labels, params, splits, ex, loss, grads = _run(
        "gat", g, 200, 128, 9, 95 + g)
    ws, wp = split_sample(sample.layer_vertices, sample.layer_edges, pm.assignment, g, cache.cached)
    ref = CoopRun(glorot_params("gat", 200, 128, 9, 3, seed=5), ws, wp, feats.astype(np.float64), labels)
    rloss, rgrads = ref.run()
    assert abs(loss - rloss) <= TOL * abs(rloss)
    for d in range(g):
        assert_grads_close(grads[d], rgrads[d], TOL, d)


def test_gat_wide_multihead_matches_oracle():
    sg, graph, pm, sample, cache, feats, labels, params, splits, ex, loss, grads = _run(
        "gat", 2, 200, 32, 9, 97, heads=4)
    rloss, rgrads, _ = multihead_run(sample.layer_vertices, sample.layer_edges,
                                     {k: np.asarray(v, dtype=np.float64) for k, v in params.tensors().items()},
                                     feats.astype(np.float64), labels, 4)
    assert abs(loss - rloss) <= TOL * abs(rloss)
    tot = {k: sum(np.asarray(gd[k], dtype=np.float64) for gd in grads) for k in rgrads}
    assert_grads_close(tot, rgrads, TOL)


def test_wide_captured_step_matches_oracle():
    """The dense fallbacks read every size from device memory: capture-safe."""
    import torch

    import paper_2303_13775_b200 as sg
    from paper_2303_13775_b200.engine import CapturedStep, capacities_for
    graph = sg.generate_powerlaw(20000, 200000, blocks=16, p_local=0.8, seed=9)
    pm = sg.range_partition(graph.num_vertices, 1)
    cache = sg.full_cache(pm)
    F, hid, C, B = 100, 128, 64, 96
    feats = sg.FeatureStore.synthetic(graph.num_vertices, F, seed=1)
    hostX = sg.synthetic_features(graph.num_vertices, F, seed=1).astype(np.float64)
    labels = sg.synthetic_labels(graph.num_vertices, C, seed=2)
    rng = np.random.default_rng(3)
    samples = [sg.sample_minibatch(graph, rng.choice(graph.num_vertices, B, replace=False), [8, 6, 4], rng)
               for _ in range(4)]
    cap_nV, cap_nE = capacities_for(samples, slack=1.1)
    dp = sg.DeviceParams.from_host(sg.init_params("graphsage", F, hid, C, 3, seed=4))
    cs = CapturedStep(dp, pm, cache, feats, torch.from_numpy(labels).cuda(), cap_nV, cap_nE, 0.1 / B)
    cs.capture(samples[0])
    ref = glorot_params("graphsage", F, hid, C, 3, seed=4)
    for i, smp in enumerate(samples):
        if i > 0:
            cs.run(smp)
        ws, wp = split_sample(smp.layer_vertices, smp.layer_edges, pm.assignment, 1, cache.cached)
        rl, rg = CoopRun(ref, ws, wp, hostX, labels).run()
        reduce_and_sgd(ref, rg, 0.1, B)
        if i > 0:
            got = float(cs.out[dp.n].item())
            assert abs(got - rl) <= 1e-4 * abs(rl), (i, got, rl)
    got = dp.to_host().tensors()
    for k in ref:
        assert rel_err(got[k], ref[k]) < 1e-4, k
