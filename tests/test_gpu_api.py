"""The reference-facing API as a user drives it (reference engine.py:655-826
run_epoch's split branch): split_minibatch -> SplitExecutor.run ->
allreduce_and_step, step after step, with host ModelParams updated in place.

The executor runs destination-grouped samples as a replay of a cached CUDA
graph (engine._ApiGraphStep) and leaves gradients on the device; these tests
pin that path to the eager kernels (SG_API_EAGER=1) and to the float64 oracle,
and check the lazy host views."""

import os

import numpy as np
import pytest

from helpers import rel_err

pytestmark = pytest.mark.gpu


def _workload(kind, g, F=24, C=5, B=64, steps=5, seed=0, cache_frac=None):
    import paper_2303_13775_b200 as sg
    graph = sg.generate_powerlaw(6000, 60000, blocks=8, p_local=0.8, seed=seed)
    pm = sg.range_partition(graph.num_vertices, g)
    cache = sg.full_cache(pm) if cache_frac is None else sg.build_cache(graph, pm, cache_frac)
    feats = sg.synthetic_features(graph.num_vertices, F, seed=seed + 1)
    labels = sg.synthetic_labels(graph.num_vertices, C, seed=seed + 2)
    rng = np.random.default_rng(seed + 3)
    samples = [sg.sample_minibatch(graph, rng.choice(graph.num_vertices, B - 7 * (i % 2), replace=False),
                                   [6, 4, 3], rng) for i in range(steps)]
    params = sg.init_params(kind, F, 8, C, 3, seed=seed + 4)
    return graph, pm, cache, feats, labels, samples, params


def _train(sg, params, samples, pm, cache, feats, labels, lr=0.1):
    losses = []
    for smp in samples:
        splits, plan = sg.split_minibatch(smp, pm, cache)
        ex = sg.SplitExecutor(params, splits, plan, feats, labels)
        loss, grads = ex.run()
        sg.allreduce_and_step(params, grads, lr, len(smp.targets))
        losses.append(loss)
    return losses


@pytest.mark.parametrize("kind,g", [("graphsage", 1), ("graphsage", 3), ("gat", 2)])
def test_api_loop_graph_path_matches_eager_and_oracle(kind, g, monkeypatch):
    import copy
    import paper_2303_13775_b200 as sg
    from paper_2303_13775_b200 import engine
    from oracle.coop_oracle import CoopRun, reduce_and_sgd
    from oracle.split_oracle import split_sample
    graph, pm, cache, feats, labels, samples, params = _workload(kind, g)
    p_graph, p_eager = copy.deepcopy(params), copy.deepcopy(params)
    engine._API_GRAPHS.clear()
    l_graph = _train(sg, p_graph, samples, pm, cache, feats, labels)
    assert len(engine._API_GRAPHS) >= 1  # the captured path ran
    monkeypatch.setenv("SG_API_EAGER", "1")
    l_eager = _train(sg, p_eager, samples, pm, cache, feats, labels)
    np.testing.assert_allclose(l_graph, l_eager, rtol=1e-5)
    for k, v in p_graph.tensors().items():
        assert rel_err(v, p_eager.tensors()[k]) < 1e-5, k
    # float64 oracle replaying the same samples from the same init
    from oracle.model_oracle import glorot_params
    rp = glorot_params(kind, feats.shape[1], 8, 5, 3, seed=4)
    for i, smp in enumerate(samples):
        ws, wp = split_sample(smp.layer_vertices, smp.layer_edges, pm.assignment, g, cache.cached)
        rloss, rgrads = CoopRun(rp, ws, wp, feats.astype(np.float64), labels).run()
        reduce_and_sgd(rp, rgrads, 0.1, len(smp.targets))
        assert abs(l_graph[i] - rloss) <= 1e-4 * abs(rloss), (i, l_graph[i], rloss)
    for k, v in p_graph.tensors().items():
        assert rel_err(v, rp[k]) < 1e-4, k


def test_api_lazy_views_and_states():
    """split_minibatch's host views are built on first access and equal the
    oracle split; states after a captured run() equal the eager executor's."""
    import paper_2303_13775_b200 as sg
    from oracle.split_oracle import split_sample
    graph, pm, cache, feats, labels, samples, params = _workload("graphsage", 2, steps=1)
    smp = samples[0]
    splits, plan = sg.split_minibatch(smp, pm, cache)
    assert splits._fill_fn is not None and len(splits) == 2  # not built yet
    ex = sg.SplitExecutor(params, splits, plan, feats, labels)
    loss, grads = ex.run()
    assert splits._fill_fn is not None  # run() did not need the host views
    assert grads[0]._lazy
    ws, wp = split_sample(smp.layer_vertices, smp.layer_edges, pm.assignment, 2, cache.cached)
    for d in range(2):
        for l in range(4):
            assert np.array_equal(splits[d].owned_gids[l], ws[d]["owned_gids"][l])
    assert plan.pair_count(1) == sum(e.count for (l, _, _), e in plan.entries.items() if l == 1)
    ex2 = sg.SplitExecutor(params, *sg.split_minibatch(smp, pm, cache), feats, labels)
    ex2.forward()
    for d in range(2):
        for l in range(4):
            np.testing.assert_array_equal(ex.states[d].h[l], ex2.states[d].h[l])
    assert set(grads[0].keys()) == set(params.tensors().keys())


def test_api_partial_cache():
    """Cache misses staged from host memory on the captured API path."""
    import copy
    import paper_2303_13775_b200 as sg
    graph, pm, cache, feats, labels, samples, params = _workload("graphsage", 2, cache_frac=0.2, steps=3)
    p1, p2 = copy.deepcopy(params), copy.deepcopy(params)
    l1 = _train(sg, p1, samples, pm, cache, feats, labels)
    os.environ["SG_API_EAGER"] = "1"
    try:
        l2 = _train(sg, p2, samples, pm, cache, feats, labels)
    finally:
        del os.environ["SG_API_EAGER"]
    np.testing.assert_allclose(l1, l2, rtol=1e-5)


def test_split_from_pinned_sample_matches_packed(monkeypatch):
    """A native-sampler sample lives in one pinned buffer and reaches the
    device with one H2D + sg_relayout_sample_compact (no host pack): the device layout,
    the split's host views and the plan equal those of the packing path; a
    sample whose arrays were replaced falls back to packing."""
    import torch
    import paper_2303_13775_b200 as sg
    from paper_2303_13775_b200 import scheduler
    graph, pm, cache, feats, labels, samples, params = _workload("graphsage", 3, cache_frac=0.3)
    smp = samples[1]
    assert smp.pinned is not None and smp.pinned.intact(smp)
    # compact form: only [header | V | es | run starts] crosses PCIe; the
    # destination lists are rebuilt on the device, so they are read-only here
    assert smp.pinned.RS > 0 and smp.pinned.dma_words < smp.pinned.S + smp.pinned.VS + 2 * smp.pinned.ES
    with pytest.raises(ValueError):
        smp.layer_edges[0][1][0] = 0

    def layout(splits):
        buf, used, geo = splits.device_split.packed
        h = buf[:used].cpu().numpy()
        nV, nE = smp.sizes()
        segs = [h[:geo.S]] + [h[geo.o_V + geo.voff[l]:][:nV[l]] for l in range(geo.L + 1)] + \
               [h[geo.o_es + geo.eoff[l]:][:nE[l]] for l in range(geo.L)] + \
               [h[geo.o_ed + geo.eoff[l]:][:nE[l]] for l in range(geo.L)]
        return np.concatenate(segs)

    s1, p1 = sg.split_minibatch(smp, pm, cache)
    monkeypatch.setattr(scheduler, "_DIRECT", False)
    s2, p2 = sg.split_minibatch(smp, pm, cache)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(layout(s1), layout(s2))
    for a, b in zip(s1, s2):
        for l in range(len(a.owned_gids)):
            np.testing.assert_array_equal(a.owned_gids[l], b.owned_gids[l])
            np.testing.assert_array_equal(a.ref_gids[l], b.ref_gids[l])
        np.testing.assert_array_equal(a.load_gids, b.load_gids)
    assert sorted(p1.entries.keys()) == sorted(p2.entries.keys())
    for k in p1.entries.keys():
        for f in ("gids", "holder_idx", "owner_idx"):
            np.testing.assert_array_equal(getattr(p1.entries[k], f), getattr(p2.entries[k], f))
    monkeypatch.setattr(scheduler, "_DIRECT", True)
    # an array replaced by the caller: the pinned buffer no longer describes the sample
    other = sg.MiniBatchSample(smp.num_layers, [v.copy() for v in smp.layer_vertices], list(smp.layer_edges),
                               dst_grouped=True, pinned=smp.pinned)
    assert not other.pinned.intact(other)
    # a destination list made writable again (and so possibly edited) is packed too
    d = smp.layer_edges[1][1]
    d.flags.writeable = True
    assert not smp.pinned.intact(smp)
    d.flags.writeable = False
    assert smp.pinned.intact(smp)
    s3, _ = sg.split_minibatch(other, pm, cache)
    np.testing.assert_array_equal(layout(s3), layout(s2))
    # vertices beyond the partition map still raise (packing path checks them)
    small = sg.range_partition(graph.num_vertices // 2, 3)
    with pytest.raises(ValueError, match="missing from partition map"):
        sg.split_minibatch(smp, small)


@pytest.mark.parametrize("g", [1, 3])
def test_host_sgd_matches_device_sgd(g):
    """allreduce_and_step on gradients a captured run brought to the host (the
    host SGD) equals the device kernel (sg_sum_sgd: device-order fp32 sum,
    fused multiply-add) on the same gradients: at most 1 ulp apart, almost
    always equal."""
    import copy
    import torch
    import paper_2303_13775_b200 as sg
    from paper_2303_13775_b200 import engine
    graph, pm, cache, feats, labels, samples, params = _workload("graphsage", g)
    p_host, p_dev = copy.deepcopy(params), copy.deepcopy(params)
    splits, plan = sg.split_minibatch(samples[0], pm, cache)
    ex = sg.SplitExecutor(p_host, splits, plan, feats, labels)
    _, grads = ex.run()
    assert ex.graph is not None and all(gd.host_flat is not None for gd in grads)
    dev_grads = [engine.GradDict(dparams=gd.dparams, device_flat=torch.from_numpy(gd.host_flat).cuda())
                 for gd in grads]
    nt = len(samples[0].targets)
    s_host = sg.allreduce_and_step(p_host, grads, 0.37, nt)
    s_dev = sg.allreduce_and_step(p_dev, dev_grads, 0.37, nt)
    for k in s_host.keys():
        np.testing.assert_array_equal(s_host[k], s_dev[k])  # the device-order sum, bit-exact
    a = engine._host_flat(p_host)
    b = engine._host_flat(p_dev)
    ulp = np.abs(a.view(np.int32).astype(np.int64) - b.view(np.int32).astype(np.int64))
    assert ulp.max() <= 1 and np.count_nonzero(ulp) <= max(1, a.size // 1000), (ulp.max(), np.count_nonzero(ulp))


def test_split_from_pinned_full_form_matches_packed(monkeypatch):
    """The non-compact pinned form ([header | V | es | ed], no run starts:
    sg_relayout_sample_hdr) gives the same device layout as packing."""
    import torch
    import paper_2303_13775_b200 as sg
    from paper_2303_13775_b200 import scheduler
    from paper_2303_13775_b200.sampling import PinnedArrays
    graph, pm, cache, feats, labels, samples, params = _workload("graphsage", 2)
    src = samples[2]
    nV, nE = src.sizes()
    L = len(nE)
    S, VS, ES = 2 * (2 * L + 1), sum(nV), sum(nE)
    t = torch.empty(S + VS + 2 * ES, dtype=torch.int32, pin_memory=True)
    buf = t.numpy()
    buf[:S].view(np.int64)[:] = nV + nE
    o = S
    lv = []
    for v in src.layer_vertices:
        buf[o:o + len(v)] = v
        lv.append(buf[o:o + len(v)])
        o += len(v)
    es, ed = [], []
    for a, _ in src.layer_edges:
        buf[o:o + len(a)] = a
        es.append(buf[o:o + len(a)])
        o += len(a)
    for _, b in src.layer_edges:
        buf[o:o + len(b)] = b
        ed.append(buf[o:o + len(b)])
        o += len(b)
    le = list(zip(es, ed))
    smp = sg.MiniBatchSample(L, lv, le, dst_grouped=True)
    smp.pinned = PinnedArrays(t, buf.ctypes.data, S, VS, ES, graph.num_vertices, tuple(lv) + tuple(le))
    assert smp.pinned.intact(smp) and smp.pinned.RS == 0
    s1, _ = sg.split_minibatch(smp, pm, cache)
    monkeypatch.setattr(scheduler, "_DIRECT", False)
    s2, _ = sg.split_minibatch(smp, pm, cache)
    torch.cuda.synchronize()
    b1, u1, geo = s1.device_split.packed
    b2, u2, _ = s2.device_split.packed
    assert u1 == u2 and s1.device_split.h2d_bytes == 4 * (S + VS + 2 * ES)
    h1, h2 = b1[:u1].cpu().numpy(), b2[:u2].cpu().numpy()
    for a, n in [(0, geo.S)] + [(geo.o_V + geo.voff[l], nV[l]) for l in range(L + 1)] + \
            [(geo.o_es + geo.eoff[l], nE[l]) for l in range(L)] + [(geo.o_ed + geo.eoff[l], nE[l]) for l in range(L)]:
        np.testing.assert_array_equal(h1[a:a + n], h2[a:a + n])
    for a, b in zip(s1, s2):
        np.testing.assert_array_equal(a.load_gids, b.load_gids)
        for l in range(len(a.owned_gids)):
            np.testing.assert_array_equal(a.owned_gids[l], b.owned_gids[l])
