"""GAT split-parallel step on the GPU vs the reference (golden) and the oracle
(engine.py:280-552): alpha, activations and gradients within rel 1e-4,
alpha sums to 1 across devices, 50-step loss curve within 1e-3."""

import numpy as np
import pytest

from golden_io import unpack_dict, unpack_sample
from helpers import assert_grads_close, cached_lists, load_golden, random_partition_case, rel_err
from oracle.coop_oracle import CoopRun
from oracle.model_oracle import glorot_params
from oracle.split_oracle import split_sample
from test_gpu_sage import LOSS_TOL, TOL, _run_fixture

pytestmark = pytest.mark.gpu

GAT_FIXTURES = ["exec_gat_0", "exec_gat_1", "exec_gat_2", "exec_gat_3", "edge_all_on_one",
                "edge_idle_device_gat", "workload3_gat"]


@pytest.mark.parametrize("name", GAT_FIXTURES)
def test_gat_matches_reference_golden(name):
    z, ex, loss, grads, rec = _run_fixture(name)
    assert abs(loss - float(z["loss_split"])) <= TOL * max(1.0, abs(float(z["loss_split"])))
    L = int(z["L"])
    for d in range(int(z["g"])):
        assert_grads_close(grads[d], unpack_dict(z, f"G{d}"), TOL, d)
        for l in range(L + 1):
            assert rel_err(ex.states[d].h[l], z[f"h_{d}_{l}"]) < TOL, (d, l)
        for l in range(1, L + 1):
            assert rel_err(ex.states[d].layer[l]["alpha"], z[f"alpha_{d}_{l}"]) < TOL, (d, l)
    assert rec.peer_bytes == int(z["peer_bytes"])  # reference metering formula


@pytest.mark.parametrize("g", [1, 2, 4, 8])
def test_gat_matches_oracle_random(g):
    import paper_2303_13775_b200 as sg
    graph, pm, sample, cache = random_partition_case(40 + g, n=5000, m=60000, g=g, batch=128,
                                                     fanouts=(6, 5, 4), cache_frac=0.2)
    F = 20
    feats = sg.synthetic_features(graph.num_vertices, F, seed=3)
    labels = sg.synthetic_labels(graph.num_vertices, 7, seed=4)
    params = sg.init_params("gat", F, 16, 7, 3, seed=5)
    splits, plan = sg.split_minibatch(sample, pm, cache)
    ex = sg.SplitExecutor(params, splits, plan, feats, labels)
    loss, grads = ex.run()
    ws, wp = split_sample(sample.layer_vertices, sample.layer_edges, pm.assignment, g, cache.cached)
    ref = CoopRun(glorot_params("gat", F, 16, 7, 3, seed=5), ws, wp, feats.astype(np.float64), labels)
    rloss, rgrads = ref.run()
    assert abs(loss - rloss) <= TOL * abs(rloss)
    for d in range(g):
        assert_grads_close(grads[d], rgrads[d], TOL, d)
        for l in range(1, 4):
            assert rel_err(ex.states[d].h[l], ref.h[d][l]) < TOL, (d, l)
            assert rel_err(ex.states[d].layer[l]["alpha"], ref.keep[d][l]["alpha"]) < TOL, (d, l)


def test_gat_alpha_sums_to_one_across_devices():  # test_engine.py:136-159
    import paper_2303_13775_b200 as sg
    for seed in range(3):
        graph, pm, sample, _ = random_partition_case(60 + seed, g=3)
        F = 5
        feats = sg.synthetic_features(graph.num_vertices, F, seed=seed)
        labels = sg.synthetic_labels(graph.num_vertices, 3, seed=seed)
        params = sg.init_params("gat", F, 4, 3, 2, seed=seed)
        splits, plan = sg.split_minibatch(sample, pm)
        ex = sg.SplitExecutor(params, splits, plan, feats, labels)
        ex.forward()
        crossers = 0
        for l in (1, 2):
            tot = {}
            for d, st in enumerate(ex.states):
                _, dst_gid = splits[d].edge_gids(l)
                for gid, a in zip(dst_gid.tolist(), st.layer[l]["alpha"].tolist()):
                    tot[gid] = tot.get(gid, 0.0) + a
                crossers += splits[d].num_ref(l)
            assert max(abs(v - 1.0) for v in tot.values()) < 1e-5
        assert crossers > 0


def test_gat_loss_curve_50_steps():
    import paper_2303_13775_b200 as sg
    z = load_golden("losscurve_gat")
    P0 = unpack_dict(z, "P0")
    params = sg.ModelParams("gat", [sg.GatLayer(P0[f"layer{i}.w"].copy(), P0[f"layer{i}.a_src"].copy(),
                                                P0[f"layer{i}.a_dst"].copy()) for i in range(2)],
                            P0["cls.w"].copy(), P0["cls.b"].copy())
    pm = sg.PartitionMap(z["assignment"], int(z["g"]), 100.0)
    cache = sg.CacheState(cached_lists(z), 1.0)
    losses = []
    for it in range(int(z["steps"])):
        sub = {k[len(f"it{it}_"):]: z[k] for k in z.files if k.startswith(f"it{it}_")}
        V, E = unpack_sample(sub)
        splits, plan = sg.split_minibatch(sg.MiniBatchSample(len(E), V, E), pm, cache)
        loss, grads = sg.SplitExecutor(params, splits, plan, z["features"], z["labels"]).run()
        sg.allreduce_and_step(params, grads, float(z["lr"]), len(V[-1]))
        losses.append(loss / len(V[-1]))
    diff = np.abs(np.asarray(losses) - z["losses"])
    assert diff.max() < LOSS_TOL, diff.max()


@pytest.mark.parametrize("g,F", [(1, 24), (2, 24), (4, 24), (1, 100), (2, 100)])
def test_gat_multihead_matches_composed_oracle(g, F):
    """C3's 4-head GAT: parity by per-head composition of the reference layer
    (SURVEY §8(a) row 11): split run summed over devices == composed single-
    device oracle."""
    import paper_2303_13775_b200 as sg
    from oracle.multihead_oracle import multihead_run
    graph, pm, sample, cache = random_partition_case(80 + g, n=5000, m=60000, g=g, batch=96,
                                                     fanouts=(6, 5, 4), cache_frac=0.3)
    H, dh, C = 4, 16, 7  # F = 100: the C3 layer-1 shape (tensor-core projection / weight gradient)
    feats = sg.synthetic_features(graph.num_vertices, F, seed=3)
    labels = sg.synthetic_labels(graph.num_vertices, C, seed=4)
    params = sg.init_params("gat", F, dh, C, 3, seed=5, heads=H)
    splits, plan = sg.split_minibatch(sample, pm, cache)
    ex = sg.SplitExecutor(params, splits, plan, feats, labels)
    loss, grads = ex.run()
    rloss, rgrads, rh = multihead_run(sample.layer_vertices, sample.layer_edges,
                                      {k: np.asarray(v, dtype=np.float64) for k, v in params.tensors().items()},
                                      feats.astype(np.float64), labels, H)
    assert abs(loss - rloss) <= TOL * abs(rloss), (loss, rloss)
    tot = {k: sum(gd[k] for gd in grads) for k in rgrads}
    assert_grads_close(tot, rgrads, TOL, "sum")
    for d in range(g):
        for l in range(1, 4):
            want = rh[l][splits[d].owned_pos[l]]
            assert rel_err(ex.states[d].h[l], want) < TOL, (d, l)


def test_multihead_init_is_reference_for_one_head():
    import paper_2303_13775_b200 as sg
    a = sg.init_params("gat", 10, 8, 3, 2, seed=1).tensors()
    b = sg.init_params("gat", 10, 8, 3, 2, seed=1, heads=1).tensors()
    assert all(np.array_equal(a[k], b[k]) for k in a)


@pytest.mark.parametrize("F,H", [(36, 2), (64, 8), (100, 4)])
def test_gat_tcgen05_projection_shapes(F, H):
    """The tcgen05 projection (D = 64, w <= 104, head width 32 / 8 / 16; K
    padded to 8) over enough rows that every CTA runs several 128-row tiles
    (pipelined gathers, partial last tile) against the composed float64
    oracle."""
    import paper_2303_13775_b200 as sg
    from oracle.multihead_oracle import multihead_run
    graph, pm, sample, cache = random_partition_case(300 + F, n=120000, m=1500000, g=1, batch=2048,
                                                     fanouts=(10, 8), cache_frac=1.0)
    assert len(sample.layer_vertices[0]) > 148 * 128  # several tiles on some CTAs
    dh, C = 64 // H, 5
    feats = sg.synthetic_features(graph.num_vertices, F, seed=3)
    labels = sg.synthetic_labels(graph.num_vertices, C, seed=4)
    params = sg.init_params("gat", F, dh, C, 2, seed=5, heads=H)
    splits, plan = sg.split_minibatch(sample, pm, cache)
    ex = sg.SplitExecutor(params, splits, plan, feats, labels)
    loss, grads = ex.run()
    rloss, rgrads, rh = multihead_run(sample.layer_vertices, sample.layer_edges,
                                      {k: np.asarray(v, dtype=np.float64) for k, v in params.tensors().items()},
                                      feats.astype(np.float64), labels, H)
    assert abs(loss - rloss) <= TOL * abs(rloss), (loss, rloss)
    assert_grads_close(grads[0], rgrads, TOL, "tc")
    for l in range(1, 3):
        assert rel_err(ex.states[0].h[l], rh[l][splits[0].owned_pos[l]]) < TOL, l


@pytest.mark.parametrize("H,dh,g", [(1, 64, 1), (2, 32, 3), (4, 16, 2), (4, 16, 1)])
def test_gat_wgrad_dst_matches_source_path(H, dh, g, monkeypatch):
    """The destination-centric layer-1 weight gradient (sg_gat_wgrad_dst,
    heads 1 / 2 / 4, with holders' dt combined at g > 1) against the
    source-row path it replaces (k_gat_bwd_src + the weight-gradient kernel,
    SG_GAT_WGRAD_DST=0): same loss, every gradient within fp32 roundoff."""
    import paper_2303_13775_b200 as sg
    from helpers import assert_grads_close
    graph, pm, sample, cache = random_partition_case(400 + H * 10 + g, n=6000, m=70000, g=g, batch=128,
                                                     fanouts=(7, 5), cache_frac=0.5)
    F, C = 24, 5
    feats = sg.synthetic_features(graph.num_vertices, F, seed=3)
    labels = sg.synthetic_labels(graph.num_vertices, C, seed=4)
    params = sg.init_params("gat", F, dh, C, 2, seed=5, heads=H)
    out = {}
    monkeypatch.setenv("SG_API_EAGER", "1")  # the flag is read per step, not per cached graph
    for flag in ("1", "0"):
        monkeypatch.setenv("SG_GAT_WGRAD_DST", flag)
        splits, plan = sg.split_minibatch(sample, pm, cache)
        ex = sg.SplitExecutor(params, splits, plan, feats, labels)
        loss, grads = ex.run()
        tot = {k: sum(np.asarray(gd[k], dtype=np.float64) for gd in grads) for k in grads[0]}
        out[flag] = (loss, tot)
    assert abs(out["1"][0] - out["0"][0]) <= 1e-6 * abs(out["0"][0])
    assert_grads_close(out["1"][1], out["0"][1], 1e-5)
