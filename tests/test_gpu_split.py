"""GPU splitter parity: every LocalSplit / PlanEntry field bit-exact with the
reference (golden fixtures from the real reference) and with the oracle on
random cases (scheduler.py:164-254)."""

import glob
import os

import numpy as np
import pytest

from golden_io import unpack_sample, unpack_splits
from helpers import (GOLD, assert_split_equal, cached_lists, load_golden, plan_as_dict, random_partition_case,
                     splits_as_dicts)
from oracle.split_oracle import split_sample

pytestmark = pytest.mark.gpu


def _golden_split_files():
    out = []
    for p in sorted(glob.glob(os.path.join(GOLD, "*.npz"))):
        z = np.load(p)
        if "S_g" in z:
            out.append(p)
    return out


@pytest.mark.parametrize("path", _golden_split_files(), ids=lambda p: os.path.basename(p)[:-4])
def test_split_matches_reference_golden(path):
    import paper_2303_13775_b200 as sg
    z = np.load(path)
    V, E = unpack_sample(z)
    want_s, want_p = unpack_splits(z, len(E))
    pm = sg.PartitionMap(z["assignment"], int(z["g"]), 100.0)
    cl = cached_lists(z)
    cache = sg.CacheState(cl, 1.0) if cl is not None else None
    sample = sg.MiniBatchSample(len(E), V, E)
    splits, plan = sg.split_minibatch(sample, pm, cache)
    assert_split_equal(splits_as_dicts(splits), plan_as_dict(plan), want_s, want_p)
    assert [plan.pair_count(l) for l in range(1, len(E) + 1)] == z["pair_count"].tolist()


@pytest.mark.parametrize("g", [1, 2, 3, 4, 8, 16])
@pytest.mark.parametrize("seed", [0, 1])
def test_split_matches_oracle_random(g, seed):
    import paper_2303_13775_b200 as sg
    graph, pm, sample, cache = random_partition_case(seed, g=g, idle=(seed == 1),
                                                     cache_frac=0.3 if seed == 0 else None)
    splits, plan = sg.split_minibatch(sample, pm, cache)
    want_s, want_p = split_sample(sample.layer_vertices, sample.layer_edges, pm.assignment, g,
                                  cache.cached if cache is not None else None)
    assert_split_equal(splits_as_dicts(splits), plan_as_dict(plan), want_s, want_p)


def test_split_three_layers_large_batch():
    import paper_2303_13775_b200 as sg
    graph, pm, sample, cache = random_partition_case(7, n=50000, m=600000, g=8, batch=2048,
                                                     fanouts=(10, 8, 5), cache_frac=0.1)
    splits, plan = sg.split_minibatch(sample, pm, cache)
    want_s, want_p = split_sample(sample.layer_vertices, sample.layer_edges, pm.assignment, 8,
                                  cache.cached)
    assert_split_equal(splits_as_dicts(splits), plan_as_dict(plan), want_s, want_p)


def test_split_unordered_edges():
    """Edges not grouped by destination (test_models.py:102-117 shuffles them):
    the split lists must still follow the sample's edge order exactly."""
    import paper_2303_13775_b200 as sg
    graph, pm, sample, _ = random_partition_case(3, g=3)
    rng = np.random.default_rng(0)
    edges = []
    for s, d in sample.layer_edges:
        perm = rng.permutation(len(s))
        edges.append((np.asarray(s)[perm], np.asarray(d)[perm]))
    shuffled = sg.MiniBatchSample(sample.num_layers, sample.layer_vertices, edges)
    assert not shuffled.is_dst_grouped()
    splits, plan = sg.split_minibatch(shuffled, pm)
    want_s, want_p = split_sample(shuffled.layer_vertices, edges, pm.assignment, 3)
    assert_split_equal(splits_as_dicts(splits), plan_as_dict(plan), want_s, want_p)


def test_split_missing_vertex_raises():
    import paper_2303_13775_b200 as sg
    V = [np.array([2, 1]), np.array([2])]
    E = [(np.array([0, 1]), np.array([0, 0]))]
    pm = sg.PartitionMap(np.array([0, 1]), 2, 1.0)
    with pytest.raises(ValueError, match="missing from partition map"):
        sg.split_minibatch(sg.MiniBatchSample(1, V, E), pm)


def test_split_is_pure_and_deterministic():
    import paper_2303_13775_b200 as sg
    graph, pm, sample, cache = random_partition_case(5, g=4, cache_frac=0.2)
    a = sg.split_minibatch(sample, pm, cache)
    b = sg.split_minibatch(sample, pm, cache)
    assert_split_equal(splits_as_dicts(a[0]), plan_as_dict(a[1]), splits_as_dicts(b[0]),
                       plan_as_dict(b[1]))


@pytest.mark.parametrize("name", ["split_random_0", "split_random_1", "split_random_2", "split_random_3",
                                  "split_random_4", "split_random_5", "edge_single_cross", "edge_all_on_one",
                                  "workload3_graphsage"])
def test_split_cost_matches_reference_golden(name):
    """split_cost (scheduler.py:257-309) on the GPU: cost per layer, per-device
    edge counts bit-exact; skew and locality equal to the reference's."""
    import paper_2303_13775_b200 as sg
    z = load_golden(name)
    V, E = unpack_sample(z)
    g = int(z["g"])
    pm = sg.PartitionMap(z["assignment"], g, float(g))
    rep = sg.split_cost(sg.MiniBatchSample(len(E), V, E), pm, g)
    assert rep.cost_per_layer == [int(x) for x in z["cost_per_layer"]]
    assert np.array_equal(rep.edges_per_device, z["edges_per_device"])
    assert abs(rep.local_edge_fraction - float(z["local_edge_fraction"])) < 1e-12
    assert abs(rep.edge_skew - float(z["edge_skew"])) < 1e-12
    assert rep.cost_per_layer == [int(x) for x in z["pair_count"]]  # C[v^l] summed == pair_count(l)
    for l, c in enumerate(rep.per_layer_cost):
        assert len(c) == len(V[l + 1]) and c.sum() == rep.cost_per_layer[l]
