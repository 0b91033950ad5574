"""Shared test helpers: fixture loading and comparison utilities."""

from __future__ import annotations

import os

import numpy as np

from golden_io import unpack_dict, unpack_sample, unpack_splits

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load_golden(name):
    return np.load(os.path.join(GOLD, name + ".npz"), allow_pickle=False)


def cached_lists(z):
    n = int(z["cache_ndev"])
    return None if n < 0 else [z[f"cache_{d}"] for d in range(n)]


def rel_err(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = max(np.abs(b).max(initial=0.0), 1e-9)
    return float(np.abs(a - b).max(initial=0.0) / scale)


def splits_as_dicts(splits):
    out = []
    for s in splits:
        out.append(dict(owned_gids=s.owned_gids, owned_pos=s.owned_pos, ref_gids=s.ref_gids,
                        ref_owner=s.ref_owner, edges_src=s.edges_src, edges_dst=s.edges_dst,
                        self_rows=s.self_rows, load_gids=s.load_gids))
    return out


def plan_as_dict(plan):
    return {k: (e.gids, e.holder_idx, e.owner_idx) for k, e in plan.entries.items()}


def assert_split_equal(got_splits, got_plan, want_splits, want_plan):
    """Bit-exact equality of every LocalSplit field and every PlanEntry."""
    assert len(got_splits) == len(want_splits)
    for d, (gs, ws) in enumerate(zip(got_splits, want_splits)):
        for f in ("owned_gids", "owned_pos", "ref_gids", "ref_owner", "edges_src", "edges_dst",
                  "self_rows"):
            assert len(gs[f]) == len(ws[f]), (d, f)
            for l, (a, b) in enumerate(zip(gs[f], ws[f])):
                a = np.asarray(a, np.int64)
                b = np.asarray(b, np.int64)
                assert a.shape == b.shape and np.array_equal(a, b), (d, f, l, a[:10], b[:10])
        assert np.array_equal(np.asarray(gs["load_gids"], np.int64),
                              np.asarray(ws["load_gids"], np.int64)), (d, "load_gids")
    assert sorted(got_plan) == sorted(want_plan), (sorted(got_plan), sorted(want_plan))
    for k in want_plan:
        for a, b in zip(got_plan[k], want_plan[k]):
            assert np.array_equal(np.asarray(a, np.int64), np.asarray(b, np.int64)), k


def random_partition_case(seed, n=3000, m=30000, g=4, batch=64, fanouts=(5, 5), idle=False,
                          cache_frac=None):
    """Native power-law graph + random partition + native sample."""
    import paper_2303_13775_b200 as sg
    graph = sg.generate_powerlaw(n, m, blocks=8, p_local=0.5, seed=seed)
    rng = np.random.default_rng(seed)
    asn = rng.integers(0, g, n)
    if idle and g > 2:
        asn[asn == g - 1] = 0  # device g-1 owns nothing
    pm = sg.PartitionMap(asn, g, float(g))
    targets = rng.choice(n, size=batch, replace=False)
    sample = sg.sample_minibatch(graph, targets, list(fanouts), rng)
    cache = None
    if cache_frac is not None:
        cache = sg.build_cache(graph, pm, cache_frac)
    return graph, pm, sample, cache


def assert_grads_close(got, want, tol, where=""):
    """Per-tensor relative error; a tensor whose true gradient is numerically
    zero (e.g. GAT a_dst where every pre-activation is positive, so the softmax
    is invariant to t_v) is compared against 1e-3 x the largest gradient of the
    model instead of a 1e-9 floor (float32 arithmetic, float64 reference)."""
    gmax = max(float(np.abs(np.asarray(v)).max(initial=0.0)) for v in want.values())
    bad = []
    for k, w in want.items():
        w = np.asarray(w, dtype=np.float64)
        g = np.asarray(got[k], dtype=np.float64)
        scale = max(float(np.abs(w).max(initial=0.0)), 1e-3 * gmax, 1e-12)
        err = float(np.abs(g - w).max(initial=0.0)) / scale
        if err >= tol:
            bad.append((k, err))
    assert not bad, (where, bad)
