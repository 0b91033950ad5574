"""The CUDA-graph captured step (capacity layouts, sizes read from device
memory) trains exactly like the eager step and the oracle."""

import numpy as np
import pytest

from helpers import rel_err
from oracle.coop_oracle import CoopRun, reduce_and_sgd
from oracle.model_oracle import glorot_params
from oracle.split_oracle import split_sample

pytestmark = pytest.mark.gpu


def test_captured_step_matches_oracle_over_steps():
    import torch

    import paper_2303_13775_b200 as sg
    from paper_2303_13775_b200.engine import CapturedStep, capacities_for
    graph = sg.generate_powerlaw(20000, 200000, blocks=16, p_local=0.8, seed=9)
    pm = sg.range_partition(graph.num_vertices, 1)
    cache = sg.full_cache(pm)
    F, C, B = 32, 6, 96
    feats = sg.FeatureStore.synthetic(graph.num_vertices, F, seed=1)
    hostX = sg.synthetic_features(graph.num_vertices, F, seed=1).astype(np.float64)
    labels = sg.synthetic_labels(graph.num_vertices, C, seed=2)
    rng = np.random.default_rng(3)
    samples = [sg.sample_minibatch(graph, rng.choice(graph.num_vertices, B, replace=False), [8, 6, 4], rng)
               for _ in range(6)]
    cap_nV, cap_nE = capacities_for(samples, slack=1.1)
    params = sg.init_params("graphsage", F, 16, C, 3, seed=4)
    dp = sg.DeviceParams.from_host(params)
    lab = torch.from_numpy(labels).cuda()
    cs = CapturedStep(dp, pm, cache, feats, lab, cap_nV, cap_nE, 0.1 / B)
    cs.capture(samples[0])  # applies step 0 eagerly
    ref = glorot_params("graphsage", F, 16, C, 3, seed=4)
    losses = []
    for i, smp in enumerate(samples):
        if i > 0:
            cs.run(smp)
        losses.append(float(cs.out[dp.n].item()) if i > 0 else None)
        ws, wp = split_sample(smp.layer_vertices, smp.layer_edges, pm.assignment, 1, cache.cached)
        run = CoopRun(ref, ws, wp, hostX, labels)
        rl, rg = run.run()
        reduce_and_sgd(ref, rg, 0.1, B)
        if i > 0:
            assert abs(losses[-1] - rl) <= 1e-4 * abs(rl), (i, losses[-1], rl)
    got = dp.to_host().tensors()
    for k in ref:
        assert rel_err(got[k], ref[k]) < 1e-4, k


@pytest.mark.parametrize("kind", ["graphsage", "gat"])
def test_pipelined_run_matches_sequential(kind):
    """run_pipelined (double-buffered H2D on a copy stream, loss read one step
    behind) trains bit-identically to sequential run() calls."""
    import torch

    import paper_2303_13775_b200 as sg
    from paper_2303_13775_b200.engine import CapturedStep, PinnedSample, capacities_for
    graph = sg.generate_powerlaw(20000, 200000, blocks=16, p_local=0.8, seed=11)
    pm = sg.range_partition(graph.num_vertices, 1)
    cache = sg.full_cache(pm)
    F, C, B = 32, 6, 96
    feats = sg.FeatureStore.synthetic(graph.num_vertices, F, seed=1)
    labels = torch.from_numpy(sg.synthetic_labels(graph.num_vertices, C, seed=2)).cuda()
    rng = np.random.default_rng(5)
    samples = [sg.sample_minibatch(graph, rng.choice(graph.num_vertices, B, replace=False), [8, 6, 4], rng)
               for _ in range(7)]
    cap_nV, cap_nE = capacities_for(samples)
    heads = 2 if kind == "gat" else 1
    params = sg.init_params(kind, F, 8, C, 3, seed=4, heads=heads)
    runs = []
    for mode in ("seq", "pipe"):
        dp = sg.DeviceParams.from_host(params)
        cs = CapturedStep(dp, pm, cache, feats, labels, cap_nV, cap_nE, 0.1 / B)
        cs.capture(samples[0])
        if mode == "seq":
            losses = []
            for smp in samples[1:]:
                cs.run(smp)
                losses.append(float(cs.out[dp.n].item()) / len(smp.targets))
        else:
            pinned = [PinnedSample(smp, cs.inp) for smp in samples[1:]]
            losses, h2d, d2h = cs.run_pipelined(pinned)
            assert h2d == sum(p.h2d_bytes for p in pinned) and d2h == 4 * len(pinned)
        torch.cuda.synchronize()
        runs.append((losses, dp.flat.cpu().numpy().copy()))
    assert runs[0][0] == runs[1][0]
    assert np.array_equal(runs[0][1], runs[1][1])


@pytest.mark.parametrize("kind", ["graphsage", "gat"])
def test_back_to_back_runs_match_synchronized(kind):
    """CapturedStep.run() queues the sample's H2D copy behind the running
    step: calling it back to back (no host synchronisation) must train exactly
    like synchronising after every step (the pinned staging slot of a queued
    copy is never repacked)."""
    import torch

    import paper_2303_13775_b200 as sg
    from paper_2303_13775_b200.engine import CapturedStep, capacities_for
    graph = sg.generate_powerlaw(60000, 900000, blocks=16, p_local=0.8, seed=12)
    pm = sg.range_partition(graph.num_vertices, 1)
    cache = sg.full_cache(pm)
    F, C, B = 100, 6, 512
    feats = sg.FeatureStore.synthetic(graph.num_vertices, F, seed=1, pad_rows=kind == "graphsage")
    labels = torch.from_numpy(sg.synthetic_labels(graph.num_vertices, C, seed=2)).cuda()
    rng = np.random.default_rng(6)
    samples = [sg.sample_minibatch(graph, rng.choice(graph.num_vertices, B, replace=False), [15, 10, 5], rng)
               for _ in range(10)]
    cap_nV, cap_nE = capacities_for(samples)
    params = sg.init_params(kind, F, 16, C, 3, seed=4, heads=4 if kind == "gat" else 1)
    runs = []
    for mode in ("sync", "queued"):
        dp = sg.DeviceParams.from_host(params)
        cs = CapturedStep(dp, pm, cache, feats, labels, cap_nV, cap_nE, 0.1 / B)
        cs.capture(samples[0])
        torch.cuda.synchronize()
        losses = []
        for smp in samples[1:]:
            cs.run(smp)
            losses.append(cs.out[dp.n:dp.n + 1].clone() if mode == "queued" else float(cs.out[dp.n].item()))
        torch.cuda.synchronize()
        if mode == "queued":
            losses = [float(x.item()) for x in losses]
        runs.append((losses, dp.flat.cpu().numpy().copy()))
    assert runs[0][0] == runs[1][0]
    assert np.array_equal(runs[0][1], runs[1][1])
    assert np.isfinite(runs[1][1]).all()


def _reverse_groups(smp):
    """Same sample with each layer's destination groups listed in descending
    destination order (still grouped, no longer ascending)."""
    import paper_2303_13775_b200 as sg
    edges = []
    for a, b in smp.layer_edges:
        a, b = np.asarray(a), np.asarray(b)
        order = np.argsort(-b, kind="stable")
        edges.append((a[order], b[order]))
    return sg.MiniBatchSample(smp.num_layers, list(smp.layer_vertices), edges)


def test_pinned_compact_falls_back_for_unordered_groups():
    """PinnedSample(compact=True) rebuilds destinations from run starts, valid
    only for ascending destinations: a grouped-but-unordered sample must take
    the full layout and train exactly like run()."""
    import torch

    import paper_2303_13775_b200 as sg
    from paper_2303_13775_b200.engine import CapturedStep, PinnedSample, capacities_for
    graph = sg.generate_powerlaw(20000, 200000, blocks=16, p_local=0.8, seed=11)
    pm = sg.range_partition(graph.num_vertices, 1)
    cache = sg.full_cache(pm)
    F, C, B = 32, 6, 96
    feats = sg.FeatureStore.synthetic(graph.num_vertices, F, seed=1)
    labels = torch.from_numpy(sg.synthetic_labels(graph.num_vertices, C, seed=2)).cuda()
    rng = np.random.default_rng(5)
    samples = [_reverse_groups(sg.sample_minibatch(graph, rng.choice(graph.num_vertices, B, replace=False),
                                                   [8, 6, 4], rng)) for _ in range(4)]
    assert all(s.is_dst_grouped() for s in samples)
    cap_nV, cap_nE = capacities_for(samples)
    params = sg.init_params("graphsage", F, 8, C, 3, seed=4)
    runs = []
    for mode in ("seq", "pipe"):
        dp = sg.DeviceParams.from_host(params)
        cs = CapturedStep(dp, pm, cache, feats, labels, cap_nV, cap_nE, 0.1 / B)
        cs.capture(samples[0])
        if mode == "seq":
            losses = []
            for smp in samples[1:]:
                cs.run(smp)
                losses.append(float(cs.out[dp.n].item()) / len(smp.targets))
        else:
            pinned = [PinnedSample(smp, cs.inp, compact=True) for smp in samples[1:]]
            assert not any(p.compact for p in pinned)
            losses, _, _ = cs.run_pipelined(pinned)
        torch.cuda.synchronize()
        runs.append((losses, dp.flat.cpu().numpy().copy()))
    assert runs[0][0] == runs[1][0]
    assert np.array_equal(runs[0][1], runs[1][1])


def test_captured_step_normalises_by_each_samples_target_count():
    """allreduce_and_step divides by the sample's own num_targets: a short
    last batch replayed through the captured graph (captured at B = 96) gets
    lr / 40, read on the device from the sample's sizes."""
    import torch

    import paper_2303_13775_b200 as sg
    from paper_2303_13775_b200.engine import CapturedStep, capacities_for
    graph = sg.generate_powerlaw(20000, 200000, blocks=16, p_local=0.8, seed=9)
    pm = sg.range_partition(graph.num_vertices, 1)
    cache = sg.full_cache(pm)
    F, C = 32, 6
    feats = sg.FeatureStore.synthetic(graph.num_vertices, F, seed=1)
    hostX = sg.synthetic_features(graph.num_vertices, F, seed=1).astype(np.float64)
    labels = sg.synthetic_labels(graph.num_vertices, C, seed=2)
    rng = np.random.default_rng(3)
    samples = [sg.sample_minibatch(graph, rng.choice(graph.num_vertices, b, replace=False), [8, 6, 4], rng)
               for b in (96, 96, 40)]
    cap_nV, cap_nE = capacities_for(samples, slack=1.1)
    params = sg.init_params("graphsage", F, 16, C, 3, seed=4)
    dp = sg.DeviceParams.from_host(params)
    cs = CapturedStep(dp, pm, cache, feats, torch.from_numpy(labels).cuda(), cap_nV, cap_nE, 0.1 / 96)
    cs.capture(samples[0])
    for smp in samples[1:]:
        cs.run(smp)
    ref = glorot_params("graphsage", F, 16, C, 3, seed=4)
    for smp in samples:
        ws, wp = split_sample(smp.layer_vertices, smp.layer_edges, pm.assignment, 1, cache.cached)
        _, rg = CoopRun(ref, ws, wp, hostX, labels).run()
        reduce_and_sgd(ref, rg, 0.1, len(smp.targets))
    got = dp.to_host().tensors()
    for k in ref:
        assert rel_err(got[k], ref[k]) < 1e-4, k


@pytest.mark.parametrize("kind,g", [("graphsage", 4), ("graphsage", 8), ("gat", 3)])
def test_captured_multi_part_step_matches_oracle(kind, g):
    """g split parts on ONE GPU captured as one graph (bench --parts g, C1's
    2 partitions): every exchange round is a device copy, sizes never reach
    the host, and training equals the oracle's cooperative g-part run."""
    import torch

    import paper_2303_13775_b200 as sg
    from paper_2303_13775_b200.engine import CapturedStep, capacities_for
    graph = sg.generate_powerlaw(20000, 200000, blocks=16, p_local=0.8, seed=9)
    pm = sg.range_partition(graph.num_vertices, g)
    cache = sg.full_cache(pm)
    F, C, B = 64, 6, 96
    feats = sg.FeatureStore.synthetic(graph.num_vertices, F, seed=1)
    hostX = sg.synthetic_features(graph.num_vertices, F, seed=1).astype(np.float64)
    labels = sg.synthetic_labels(graph.num_vertices, C, seed=2)
    rng = np.random.default_rng(3)
    samples = [sg.sample_minibatch(graph, rng.choice(graph.num_vertices, B, replace=False), [8, 6, 4], rng)
               for _ in range(4)]
    cap_nV, cap_nE = capacities_for(samples, slack=1.1)
    params = sg.init_params(kind, F, 16, C, 3, seed=4)
    dp = sg.DeviceParams.from_host(params)
    cs = CapturedStep(dp, pm, cache, feats, torch.from_numpy(labels).cuda(), cap_nV, cap_nE, 0.1 / B)
    cs.capture(samples[0])
    losses = [None]
    for smp in samples[1:]:
        cs.run(smp)
        losses.append(float(cs.out[dp.n].item()))
    ref = glorot_params(kind, F, 16, C, 3, seed=4)
    for i, smp in enumerate(samples):
        ws, wp = split_sample(smp.layer_vertices, smp.layer_edges, pm.assignment, g, cache.cached)
        rl, rg = CoopRun(ref, ws, wp, hostX, labels).run()
        reduce_and_sgd(ref, rg, 0.1, B)
        if i > 0:
            assert abs(losses[i] - rl) <= 1e-4 * abs(rl), (i, losses[i], rl)
    got = dp.to_host().tensors()
    for k in ref:
        assert rel_err(got[k], ref[k]) < 1e-4, k
