"""The load-balanced transposed SpMM (tspmm.cu: row pieces, continuation
pieces, chunk-ordered combine) against the oracle. Production routes only
layers with >= TSPMM_MIN_EDGES edges through it; here the threshold is
forced to 0 so every backward scatter / GAT source pass takes it, and a hub
graph makes rows span many 32-edge chunks."""

import numpy as np
import pytest

from helpers import assert_grads_close, random_partition_case
from oracle.coop_oracle import CoopRun
from oracle.model_oracle import glorot_params
from oracle.multihead_oracle import multihead_run
from oracle.split_oracle import split_sample
from test_gpu_sage import TOL

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def force_tspmm(monkeypatch):
    from paper_2303_13775_b200 import engine
    monkeypatch.setattr(engine, "TSPMM_MIN_EDGES", 0)


def hub_case(seed, g, n=4000, hubs=3, batch=256, fanouts=(12, 8, 4)):
    """Every vertex has the hubs among its in-neighbours, so a sample's hub
    rows have hundreds of out-edges at layer 0 (and span many chunks)."""
    import paper_2303_13775_b200 as sg
    rng = np.random.default_rng(seed)
    src = [rng.integers(0, n, 6 * n)]
    dst = [rng.integers(0, n, 6 * n)]
    for h in range(hubs):
        src.append(np.full(n, h))
        dst.append(np.arange(n))
    src, dst = np.concatenate(src), np.concatenate(dst)
    keep = src != dst
    graph = sg.from_edges(n, src[keep], dst[keep])
    pm = sg.PartitionMap(rng.integers(0, g, n), g, float(g))
    targets = rng.choice(n, size=batch, replace=False)
    sample = sg.sample_minibatch(graph, targets, list(fanouts), rng)
    return graph, pm, sample


def _check(kind, graph, pm, sample, cache=None, heads=1, F=20, hid=16, C=7):
    import paper_2303_13775_b200 as sg
    g = pm.num_devices
    feats = sg.synthetic_features(graph.num_vertices, F, seed=3)
    labels = sg.synthetic_labels(graph.num_vertices, C, seed=4)
    params = sg.init_params(kind, F, hid, C, 3, seed=5, heads=heads)
    splits, plan = sg.split_minibatch(sample, pm, cache)
    ex = sg.SplitExecutor(params, splits, plan, feats, labels)
    loss, grads = ex.run()
    cached = cache.cached if cache is not None else None
    if heads == 1:
        ws, wp = split_sample(sample.layer_vertices, sample.layer_edges, pm.assignment, g, cached)
        ref = CoopRun(glorot_params(kind, F, hid, C, 3, seed=5), ws, wp, feats.astype(np.float64), labels)
        rloss, rgrads = ref.run()
        assert abs(loss - rloss) <= TOL * abs(rloss)
        for d in range(g):
            assert_grads_close(grads[d], rgrads[d], TOL, d)
    else:
        rloss, rgrad, _ = multihead_run(sample.layer_vertices, sample.layer_edges,
                                        {k: np.asarray(v, dtype=np.float64) for k, v in params.tensors().items()},
                                        feats.astype(np.float64), labels, heads)
        assert abs(loss - rloss) <= TOL * abs(rloss)
        tot = {k: sum(np.asarray(gd[k], dtype=np.float64) for gd in grads) for k in rgrad}
        assert_grads_close(tot, rgrad, TOL)
    return loss, grads


def _max_src_degree(sample):
    return int(np.bincount(np.asarray(sample.layer_edges[0][0])).max())


@pytest.mark.parametrize("kind", ["graphsage", "gat"])
@pytest.mark.parametrize("g", [1, 2, 4])
def test_tspmm_hub_rows_match_oracle(kind, g):
    graph, pm, sample = hub_case(11 + g, g)
    assert _max_src_degree(sample) > 96  # rows span >= 3 chunks
    _check(kind, graph, pm, sample)


@pytest.mark.parametrize("kind", ["graphsage", "gat"])
@pytest.mark.parametrize("g", [1, 3])
def test_tspmm_random_with_cache_match_oracle(kind, g):
    graph, pm, sample, cache = random_partition_case(70 + g, n=5000, m=60000, g=g, batch=128,
                                                     fanouts=(6, 5, 4), cache_frac=0.2)
    _check(kind, graph, pm, sample, cache)


@pytest.mark.parametrize("g", [1, 2])
def test_tspmm_multihead_gat_matches_oracle(g):
    graph, pm, sample = hub_case(21 + g, g)
    _check("gat", graph, pm, sample, heads=4, hid=16)


@pytest.mark.parametrize("F,hid", [(12, 5), (16, 8), (24, 32), (64, 16)])
def test_tspmm_widths(F, hid):
    """Unaligned (scalar lanes) and 4/8/16-column lanes."""
    graph, pm, sample = hub_case(31, 2, batch=128)
    _check("graphsage", graph, pm, sample, F=F, hid=hid)
    _check("gat", graph, pm, sample, F=F, hid=hid)


def test_tspmm_is_deterministic():
    graph, pm, sample = hub_case(41, 2)
    a = _check("gat", graph, pm, sample)[1]
    b = _check("gat", graph, pm, sample)[1]
    for d in range(len(a)):
        for k in a[d]:
            assert np.array_equal(np.asarray(a[d][k]), np.asarray(b[d][k])), (d, k)
