"""oracle/workload.py (the NumPy workload generators bench.py's reference arm
uses so that it never loads the product library) is bit-identical to the
product's native generators: graph, labels, features and samples."""

import numpy as np
import pytest

from oracle import workload as wl


@pytest.mark.parametrize("n,m,blocks,p_local,seed", [(5000, 60000, 8, 0.92, 0), (3001, 20000, 64, 0.5, 7)])
def test_powerlaw_graph_matches_native(n, m, blocks, p_local, seed):
    import paper_2303_13775_b200 as sg
    g = sg.generate_powerlaw(n, m, blocks=blocks, p_local=p_local, seed=seed, threads=2)
    ro, ci = wl.generate_powerlaw(n, m, blocks=blocks, p_local=p_local, seed=seed, chunk=7000)
    assert np.array_equal(ro, g.row_offsets)
    assert np.array_equal(ci, g.col_indices)


def test_labels_and_features_match_native():
    import paper_2303_13775_b200 as sg
    assert np.array_equal(wl.synthetic_labels(10000, 47, 2), sg.synthetic_labels(10000, 47, 2))
    ids = np.array([0, 5, 9999, 123456], dtype=np.int64)
    want = sg.synthetic_features(0, 100, 1, row_ids=ids)
    got = wl.synthetic_features(ids, 100, 1, dtype=np.float32)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("fan", [[15, 10, 5], [3, 3], [40]])
def test_sampler_matches_native(fan):
    import paper_2303_13775_b200 as sg
    g = sg.generate_powerlaw(20000, 300000, blocks=16, p_local=0.8, seed=3)
    ns = sg.NativeSampler(g, threads=2)
    rng = np.random.default_rng(1)
    for t in range(3):
        tg = rng.choice(g.num_vertices, 200, replace=False)
        a = ns.sample(tg, fan, 1234 + t)
        V, E = wl.sample(g.row_offsets, g.col_indices, tg, fan, 1234 + t)
        for x, y in zip(a.layer_vertices, V):
            assert np.array_equal(np.asarray(x, np.int64), y)
        for (s1, d1), (s2, d2) in zip(a.layer_edges, E):
            assert np.array_equal(np.asarray(s1, np.int64), s2)
            assert np.array_equal(np.asarray(d1, np.int64), d2)


def test_epoch_batches_match():
    import paper_2303_13775_b200 as sg
    tr = np.arange(1000)
    a = sg.epoch_batches(tr, 96, np.random.default_rng(5))
    b = wl.epoch_batches(tr, 96, np.random.default_rng(5))
    assert len(a) == len(b) and all(np.array_equal(x, y) for x, y in zip(a, b))
