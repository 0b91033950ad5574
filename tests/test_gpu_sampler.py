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
