"""Partial feature caches on every path (_load_inputs, engine.py:160-167; the
load_gids of scheduler.py:193-203): layer-0 rows missing from the GPU cache
are gathered on the device from the page-locked host matrix
(sg_stage_misses), in the eager exact step AND inside captured CUDA graphs
(CapturedStep, SampledCapturedStep) whose sizes are never read on the host.
Every run is compared with the oracle replaying the same samples."""

import numpy as np
import pytest

from helpers import rel_err
from oracle.coop_oracle import CoopRun, reduce_and_sgd
from oracle.model_oracle import glorot_params
from oracle.multihead_oracle import multihead_run
from oracle.split_oracle import split_sample

pytestmark = pytest.mark.gpu


def _graph(seed=9, n=20000, m=200000):
    import paper_2303_13775_b200 as sg
    return sg.generate_powerlaw(n, m, blocks=16, p_local=0.8, seed=seed)


def test_stage_misses_copies_the_load_list_bit_exact():
    """The staged rows are the host rows of load_gids in the reference's load
    order, for every device of a g = 4 split, padded stride included."""
    import torch

    import paper_2303_13775_b200 as sg
    from paper_2303_13775_b200.scheduler import DeviceSplit
    graph = _graph(seed=3, n=6000, m=60000)
    pm = sg.range_partition(graph.num_vertices, 4)
    cache = sg.build_cache(graph, pm, 0.05)
    rng = np.random.default_rng(1)
    smp = sg.sample_minibatch(graph, rng.choice(graph.num_vertices, 128, replace=False), [6, 4], rng)
    X = sg.synthetic_features(graph.num_vertices, 100, seed=5)
    fs = sg.FeatureStore.from_host(X, cache, pad_rows=True)
    assert fs.row_stride == 128
    ds = DeviceSplit.from_sample(smp, pm, cache)
    fs.stage_misses(ds)
    torch.cuda.synchronize()
    m = ds.host_meta()
    splits, _ = ds.to_reference_types()
    loads = np.concatenate([s.load_gids for s in splits])
    assert len(loads) == int(m.load_off[4]) > 0
    got = fs.table[fs.n_cached:fs.n_cached + len(loads)].cpu().numpy()
    assert np.array_equal(got[:, :100], X[loads])
    assert not got[:, 100:].any()
    ws, _ = split_sample(smp.layer_vertices, smp.layer_edges, pm.assignment, 4, cache.cached)
    assert np.array_equal(loads, np.concatenate([w["load_gids"] for w in ws]))


def _oracle_replay(kind, samples, pm, cache, X, labels, F, hid, C, L, B, lr=0.1):
    ref = glorot_params(kind, F, hid, C, L, seed=4)
    losses = []
    for smp in samples:
        ws, wp = split_sample(smp.layer_vertices, smp.layer_edges, pm.assignment, pm.num_devices,
                              None if cache is None else cache.cached)
        rl, rg = CoopRun(ref, ws, wp, X, labels).run()
        reduce_and_sgd(ref, rg, lr, B)
        losses.append(rl)
    return ref, losses


@pytest.mark.parametrize("kind,frac", [("graphsage", 0.15), ("graphsage", None), ("gat", 0.3)])
def test_captured_step_partial_cache_matches_oracle(kind, frac):
    """CapturedStep (g = 1, one CUDA graph, exact=False) with a partial cache
    (or none): misses are staged inside the graph; loss per step and final
    parameters equal the oracle's."""
    import torch

    import paper_2303_13775_b200 as sg
    from paper_2303_13775_b200.engine import CapturedStep, capacities_for
    graph = _graph()
    pm = sg.range_partition(graph.num_vertices, 1)
    cache = sg.build_cache(graph, pm, frac) if frac is not None else None
    F, C, B, hid = 100, 6, 96, 16
    Xh = sg.synthetic_features(graph.num_vertices, F, seed=1)
    feats = sg.FeatureStore.from_host(Xh, cache, pad_rows=kind == "graphsage")
    labels = sg.synthetic_labels(graph.num_vertices, C, seed=2)
    rng = np.random.default_rng(3)
    samples = [sg.sample_minibatch(graph, rng.choice(graph.num_vertices, B, replace=False), [8, 6, 4], rng)
               for _ in range(5)]
    cap_nV, cap_nE = capacities_for(samples, slack=1.1)
    params = sg.init_params(kind, F, hid, C, 3, seed=4)
    dp = sg.DeviceParams.from_host(params)
    cs = CapturedStep(dp, pm, cache, feats, torch.from_numpy(labels).cuda(), cap_nV, cap_nE, 0.1 / B)
    cs.capture(samples[0])
    losses = [None]
    for smp in samples[1:]:
        cs.run(smp)
        losses.append(float(cs.out[dp.n].item()))
    ref, rlosses = _oracle_replay(kind, samples, pm, cache, Xh.astype(np.float64), labels, F, hid, C, 3, B)
    for i in range(1, len(samples)):
        assert abs(losses[i] - rlosses[i]) <= 1e-4 * abs(rlosses[i]), (i, losses[i], rlosses[i])
    got = dp.to_host().tensors()
    for k in ref:
        assert rel_err(got[k], ref[k]) < 1e-4, k


def test_sampled_captured_step_partial_cache():
    """Sampler + split + miss staging + step in one graph from host targets."""
    import torch

    import paper_2303_13775_b200 as sg
    from paper_2303_13775_b200.engine import SampledCapturedStep, capacities_for
    graph = _graph(seed=5)
    pm = sg.range_partition(graph.num_vertices, 1)
    cache = sg.build_cache(graph, pm, 0.1)
    F, C, B, fan = 64, 6, 96, [8, 6, 4]
    Xh = sg.synthetic_features(graph.num_vertices, F, seed=1)
    feats = sg.FeatureStore.from_host(Xh, cache)
    labels = sg.synthetic_labels(graph.num_vertices, C, seed=2)
    rng = np.random.default_rng(3)
    plan = [(rng.choice(graph.num_vertices, B, replace=False), 77 + i) for i in range(5)]
    ns = sg.NativeSampler(graph)
    samples = [ns.sample(t, fan, sd) for t, sd in plan]
    cap_nV, cap_nE = capacities_for(samples, slack=1.2)
    params = sg.init_params("graphsage", F, 16, C, 3, seed=4)
    dp = sg.DeviceParams.from_host(params)
    cs = SampledCapturedStep(sg.GpuSampler(graph), fan, B, dp, pm, cache, feats,
                             torch.from_numpy(labels).cuda(), cap_nV, cap_nE, 0.1 / B)
    losses = []
    for i, (t, sd) in enumerate(plan):
        if i == 0:
            cs.capture_targets(t, sd)
        else:
            cs.run_targets(t, sd)
        losses.append(float(cs.out[dp.n].item()))
    cs.check()
    ref, rlosses = _oracle_replay("graphsage", samples, pm, cache, Xh.astype(np.float64), labels, F, 16, C, 3, B)
    for i in range(1, len(plan)):
        assert abs(losses[i] - rlosses[i]) <= 1e-4 * abs(rlosses[i]), (i, losses[i], rlosses[i])
    got = dp.to_host().tensors()
    for k in ref:
        assert rel_err(got[k], ref[k]) < 1e-4, k


def test_gat_multihead_captured_partial_cache():
    """4-head GAT (C3's model) captured with a partial cache vs the per-head
    composition oracle, one step."""
    import torch

    import paper_2303_13775_b200 as sg
    from paper_2303_13775_b200.engine import CapturedStep, capacities_for
    graph = _graph(seed=7)
    pm = sg.range_partition(graph.num_vertices, 1)
    cache = sg.build_cache(graph, pm, 0.2)
    F, C, B, H = 100, 6, 64, 4
    Xh = sg.synthetic_features(graph.num_vertices, F, seed=1)
    feats = sg.FeatureStore.from_host(Xh, cache)
    labels = sg.synthetic_labels(graph.num_vertices, C, seed=2)
    rng = np.random.default_rng(11)
    samples = [sg.sample_minibatch(graph, rng.choice(graph.num_vertices, B, replace=False), [8, 6, 4], rng)
               for _ in range(2)]
    cap_nV, cap_nE = capacities_for(samples, slack=1.1)
    params = sg.init_params("gat", F, 16, C, 3, seed=4, heads=H)
    host0 = {k: np.asarray(v, dtype=np.float64).copy() for k, v in params.tensors().items()}
    dp = sg.DeviceParams.from_host(params)
    cs = CapturedStep(dp, pm, cache, feats, torch.from_numpy(labels).cuda(), cap_nV, cap_nE, 0.0)
    cs.capture(samples[0])
    cs.run(samples[1])
    loss = float(cs.out[dp.n].item())
    grads = dp.grads_to_dict(cs.out)
    smp = samples[1]
    V = [np.asarray(v, np.int64) for v in smp.layer_vertices]
    E = [(np.asarray(a, np.int64), np.asarray(b, np.int64)) for a, b in smp.layer_edges]
    rl, rg, _ = multihead_run(V, E, host0, Xh.astype(np.float64), labels, H)
    assert abs(loss - rl) <= 1e-4 * abs(rl), (loss, rl)
    scale = max(np.abs(v).max() for v in rg.values())
    for k in rg:
        err = np.abs(np.asarray(grads[k]) - rg[k]).max()
        assert err <= 1e-4 * max(np.abs(rg[k]).max(), 1e-3 * scale), k
