"""GPU k-hop sampler (csrc/sampler.cu) vs the native host sampler: the same
seed gives the identical sample (every layer's vertices in first-seen order,
every edge in emission order), on power-law graphs with hub vertices
(partial Fisher-Yates path), small-degree vertices (take-all path), fanout 0,
and the C2 fanouts; samples pass the reference's validate() rules."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed,fanouts,batch", [(1, [15, 10, 5], 512), (2, [4, 3], 64), (3, [25, 0, 6], 300),
                                                 (4, [64, 2], 40)])
def test_gpu_sampler_matches_native(seed, fanouts, batch):
    import paper_2303_13775_b200 as sg
    graph = sg.generate_powerlaw(20000, 300000, blocks=8, p_local=0.7, seed=seed)
    rng = np.random.default_rng(seed)
    targets = rng.choice(graph.num_vertices, batch, replace=False)
    cpu = sg.NativeSampler(graph).sample(targets, fanouts, 12345 + seed)
    gpu = sg.GpuSampler(graph).sample(targets, fanouts, 12345 + seed)
    assert len(cpu.layer_vertices) == len(gpu.layer_vertices)
    for a, b in zip(cpu.layer_vertices, gpu.layer_vertices):
        assert np.array_equal(np.asarray(a, np.int64), np.asarray(b, np.int64))
    for (a0, a1), (b0, b1) in zip(cpu.layer_edges, gpu.layer_edges):
        assert np.array_equal(np.asarray(a0, np.int64), np.asarray(b0, np.int64))
        assert np.array_equal(np.asarray(a1, np.int64), np.asarray(b1, np.int64))
    gpu.validate(graph.num_vertices)


def test_gpu_sampler_repeated_calls_and_errors():
    import paper_2303_13775_b200 as sg
    graph = sg.generate_powerlaw(5000, 40000, blocks=4, p_local=0.5, seed=9)
    gs = sg.GpuSampler(graph)
    ns = sg.NativeSampler(graph)
    rng = np.random.default_rng(0)
    for i in range(6):  # generation stamps across calls
        t = rng.choice(graph.num_vertices, 100, replace=False)
        a, b = ns.sample(t, [5, 5], i), gs.sample(t, [5, 5], i)
        for x, y in zip(a.layer_vertices, b.layer_vertices):
            assert np.array_equal(np.asarray(x, np.int64), np.asarray(y, np.int64))
    with pytest.raises(ValueError):
        gs.sample([1, 1], [3], 0)
    with pytest.raises(ValueError):
        gs.sample([graph.num_vertices], [3], 0)


def test_sampled_captured_step_trains_like_oracle():
    """Sampler + split + step in ONE CUDA graph (SampledCapturedStep), fed only
    targets and a seed: the samples equal the native sampler's for the same
    seeds, and the parameters after several replays equal the oracle's."""
    import torch

    import paper_2303_13775_b200 as sg
    from helpers import rel_err
    from oracle.coop_oracle import CoopRun, reduce_and_sgd
    from oracle.model_oracle import glorot_params
    from oracle.split_oracle import split_sample
    from paper_2303_13775_b200.engine import SampledCapturedStep, capacities_for
    graph = sg.generate_powerlaw(20000, 200000, blocks=16, p_local=0.8, seed=9)
    pm = sg.range_partition(graph.num_vertices, 1)
    cache = sg.full_cache(pm)
    F, C, B, fan = 32, 6, 96, [8, 6, 4]
    feats = sg.FeatureStore.synthetic(graph.num_vertices, F, seed=1)
    hostX = sg.synthetic_features(graph.num_vertices, F, seed=1).astype(np.float64)
    labels = sg.synthetic_labels(graph.num_vertices, C, seed=2)
    rng = np.random.default_rng(3)
    plan = [(rng.choice(graph.num_vertices, B, replace=False), 1000 + i) for i in range(6)]
    ns = sg.NativeSampler(graph)
    samples = [ns.sample(t, fan, sd) for t, sd in plan]
    cap_nV, cap_nE = capacities_for(samples, slack=1.2)
    params = sg.init_params("graphsage", F, 16, C, 3, seed=4)
    dp = sg.DeviceParams.from_host(params)
    lab = torch.from_numpy(labels).cuda()
    cs = SampledCapturedStep(sg.GpuSampler(graph), fan, B, dp, pm, cache, feats, lab, cap_nV, cap_nE, 0.1 / B)
    ref = glorot_params("graphsage", F, 16, C, 3, seed=4)
    for i, ((t, sd), smp) in enumerate(zip(plan, samples)):
        if i == 0:
            cs.capture_targets(t, sd)      # applies step 0 eagerly
        else:
            cs.run_targets(t, sd)
        loss = float(cs.out[dp.n].item())
        ws, wp = split_sample(smp.layer_vertices, smp.layer_edges, pm.assignment, 1, cache.cached)
        rl, rg = CoopRun(ref, ws, wp, hostX, labels).run()
        reduce_and_sgd(ref, rg, 0.1, B)
        if i > 0:
            assert abs(loss - rl) <= 1e-4 * abs(rl), (i, loss, rl)
    cs.check()
    got = dp.to_host().tensors()
    for k in ref:
        assert rel_err(got[k], ref[k]) < 1e-4, k
