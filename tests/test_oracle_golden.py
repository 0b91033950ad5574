"""Pin the CPU oracle (oracle/) against the real reference's outputs.

Golden .npz files were produced by tests/golden/make_golden.py running the
unmodified reference package; the hand goldens below restate the reference's
own known-answer tests (file:line cited per test).
"""

import glob
import os

import numpy as np
import pytest

from golden_io import unpack_dict, unpack_sample, unpack_splits
from oracle.coop_oracle import CoopRun, reduce_and_sgd, shuffle_forward
from oracle.model_oracle import glorot_params, seg_max, seg_sum, single_device_run, softmax_xent
from oracle.split_oracle import pair_count, split_cost_report, split_sample, transfer_bytes

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return np.load(os.path.join(GOLD, name + ".npz"), allow_pickle=False)


def cached_lists(z):
    n = int(z["cache_ndev"])
    return None if n < 0 else [z[f"cache_{d}"] for d in range(n)]


def assert_split_equal(got_splits, got_plan, want_splits, want_plan):
    assert len(got_splits) == len(want_splits)
    for gs, ws in zip(got_splits, want_splits):
        for f in ("owned_gids", "owned_pos", "ref_gids", "ref_owner", "edges_src",
                  "edges_dst", "self_rows"):
            for a, b in zip(gs[f], ws[f]):
                assert np.array_equal(np.asarray(a, np.int64), np.asarray(b, np.int64)), f
        assert np.array_equal(gs["load_gids"], ws["load_gids"])
    assert sorted(got_plan) == sorted(want_plan)
    for k in want_plan:
        for a, b in zip(got_plan[k], want_plan[k]):
            assert np.array_equal(a, b), k


def split_files():
    return sorted(glob.glob(os.path.join(GOLD, "*.npz")))


@pytest.mark.parametrize("path", split_files(), ids=lambda p: os.path.basename(p)[:-4])
def test_oracle_splitter_matches_reference_goldens(path):
    z = np.load(path)
    if "S_g" not in z:
        pytest.skip("loss-curve fixture has no split section")
    V, E = unpack_sample(z)
    want_s, want_p = unpack_splits(z, len(E))
    got_s, got_p = split_sample(V, E, z["assignment"], int(z["g"]), cached_lists(z))
    assert_split_equal(got_s, got_p, want_s, want_p)
    assert [pair_count(got_p, l) for l in range(1, len(E) + 1)] == z["pair_count"].tolist()
    rep = split_cost_report(V, E, z["assignment"], int(z["g"]))
    assert rep["cost_per_layer"] == z["cost_per_layer"].tolist()
    assert rep["cost_per_layer"] == z["pair_count"].tolist()  # C[v^l] == pair_count
    assert np.array_equal(rep["edges_per_device"], z["edges_per_device"])
    assert rep["local_edge_fraction"] == float(z["local_edge_fraction"])
    assert rep["edge_skew"] == float(z["edge_skew"])


def exec_files():
    return sorted(p for p in split_files() if "features" in np.load(p) and "S_g" in np.load(p))


def rel_err(a, b):
    scale = max(np.abs(b).max(initial=0.0), 1e-9)
    return np.abs(np.asarray(a) - b).max(initial=0.0) / scale


@pytest.mark.parametrize("path", exec_files(), ids=lambda p: os.path.basename(p)[:-4])
def test_oracle_executor_matches_reference_goldens(path):
    z = np.load(path)
    V, E = unpack_sample(z)
    splits, plan = unpack_splits(z, len(E))
    params = unpack_dict(z, "P")
    X = z["features"].astype(np.float64)
    run = CoopRun(params, splits, plan, X, z["labels"])
    loss, grads = run.run()
    assert abs(loss - float(z["loss_split"])) <= 1e-12 * max(1.0, abs(loss))
    assert run.peer_bytes == int(z["peer_bytes"])
    for d in range(len(splits)):
        want = unpack_dict(z, f"G{d}")
        for k in want:
            assert rel_err(grads[d][k], want[k]) < 1e-12, (d, k)
        for l in range(len(E) + 1):
            assert rel_err(run.h[d][l], z[f"h_{d}_{l}"]) < 1e-12
        if str(z["kind"]) == "gat":
            for l in range(1, len(E) + 1):
                assert rel_err(run.keep[d][l]["alpha"], z[f"alpha_{d}_{l}"]) < 1e-12
    # single-device oracle
    loss_r, grads_r = single_device_run(V, E, params, X, z["labels"])
    assert abs(loss_r - float(z["loss_ref"])) <= 1e-12 * max(1.0, abs(loss_r))
    want = unpack_dict(z, "Gref")
    for k in want:
        assert rel_err(grads_r[k], want[k]) < 1e-12, k


@pytest.mark.parametrize("kind", ["graphsage", "gat"])
def test_oracle_loss_curve_matches_reference(kind):
    z = load(f"losscurve_{kind}")
    params = unpack_dict(z, "P0")
    p0 = glorot_params(kind, 8, 16, 4, 2, seed=12)
    for k in p0:
        assert np.array_equal(p0[k], params[k]), k          # init draw order pinned
    X = z["features"].astype(np.float64)
    cache = cached_lists(z)
    for it in range(int(z["steps"])):
        sub = {k[len(f"it{it}_"):]: z[k] for k in z.files if k.startswith(f"it{it}_")}
        V, E = unpack_sample(sub)
        splits, plan = split_sample(V, E, z["assignment"], int(z["g"]), cache)
        run = CoopRun(params, splits, plan, X, z["labels"])
        loss, grads = run.run()
        reduce_and_sgd(params, grads, float(z["lr"]), len(V[-1]))
        assert abs(loss / len(V[-1]) - z["losses"][it]) < 1e-10
    final = unpack_dict(z, "Pfinal")
    for k in final:
        assert rel_err(params[k], final[k]) < 1e-9, k


# -- the reference's own hand goldens, restated -------------------------------

def test_segment_sum_golden():  # test_models.py:27-31
    assert np.array_equal(seg_sum(np.array([[1.0, 2.0], [3.0, 4.0]]), np.array([0, 0]), 1), [[4.0, 6.0]])


def test_segment_empty_slots():  # test_models.py:34-39
    out = seg_sum(np.ones((2, 3)), np.array([2, 2]), 4)
    assert np.array_equal(out[2], [2, 2, 2]) and np.all(out[[0, 1, 3]] == 0)
    m = seg_max(np.array([5.0, 1.0]), np.array([1, 1]), 3)
    assert m[1] == 5.0 and np.isneginf(m[0]) and np.isneginf(m[2])


def test_single_cross_edge_golden():  # test_scheduler.py:38-52
    V = [np.array([1, 0]), np.array([1])]
    E = [(np.array([0, 1]), np.array([0, 0]))]
    splits, plan = split_sample(V, E, np.array([0, 1]), 2)
    assert len(splits[0]["edges_src"][0]) == 1
    assert splits[0]["ref_gids"][1].tolist() == [1] and splits[0]["ref_owner"][1].tolist() == [1]
    assert plan[(1, 0, 1)][0].tolist() == [1]
    assert len(splits[1]["edges_src"][0]) == 1


def test_split_cost_golden():  # test_scheduler.py:123-144
    V = [np.arange(5), np.array([0])]
    E = [(np.arange(5), np.zeros(5, dtype=np.int64))]
    rep = split_cost_report(V, E, np.array([0, 1, 1, 2, 0]), 3)
    assert rep["per_layer_cost"][0][0] == 2 and rep["cost_total"] == 2
    assert rep["edges_per_device"].tolist() == [2, 2, 1]
    assert rep["edges_local"] == 2 and rep["local_edge_fraction"] == 2 / 5


def test_missing_vertex_raises():  # test_scheduler.py:115-120
    V = [np.array([2, 1]), np.array([2])]
    E = [(np.array([0, 1]), np.array([0, 0]))]
    with pytest.raises(ValueError, match="missing from partition map"):
        split_sample(V, E, np.array([0, 1]), 2)


def test_shuffle_forward_byte_count():  # test_engine.py:104-114
    V = [np.array([1, 0]), np.array([1])]
    E = [(np.array([0, 1]), np.array([0, 0]))]
    splits, plan = split_sample(V, E, np.array([0, 1]), 2)
    owned = [np.full((len(s["owned_gids"][1]), 4), float(d)) for d, s in enumerate(splits)]
    bufs, nbytes = shuffle_forward(splits, plan, 1, owned)
    assert nbytes == 32 and np.allclose(bufs[0], 1.0)


def test_classifier_loss_manual():  # test_models.py:120-129
    p = glorot_params("graphsage", 3, 4, 3, 1, seed=11)
    h = np.random.default_rng(12).random((5, 4))
    y = np.array([0, 2, 1, 1, 0])
    loss, _, _, d_b = softmax_xent(p, h, y)
    logits = h @ p["cls.w"] + p["cls.b"]
    pr = np.exp(logits) / np.exp(logits).sum(axis=1, keepdims=True)
    assert abs(loss - (-np.log(pr[np.arange(5), y]).sum())) < 1e-12
    assert np.allclose(d_b, (pr - np.eye(3)[y]).sum(axis=0), atol=1e-12)


def test_transfer_manifest_full_cache():  # test_scheduler.py:195-216 (property form)
    z = load("workload3_graphsage")
    V, E = unpack_sample(z)
    cache = cached_lists(z)
    splits, _ = split_sample(V, E, z["assignment"], int(z["g"]), cache)
    host = transfer_bytes(splits, 16, cache)
    v0 = set(V[0].tolist())
    cached = set(np.concatenate(cache).tolist())
    assert int(host.sum()) == (len(v0) - len(v0 & cached)) * 16 * 8
