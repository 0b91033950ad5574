"""CPU restatement of the reference online splitter — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module (as the checker / timed CPU baseline). Product code never
does.

Restates /root/reference/pkg/src/splitgnn/scheduler.py:
  * _group_by                        scheduler.py:157-161
  * split_minibatch                  scheduler.py:164-254
  * split_cost                       scheduler.py:257-309
  * transfer_manifest                scheduler.py:324-347
The outputs are plain dicts so the GPU splitter can be compared field by
field (bit-exact, int64).

Inputs are the raw sample arrays:
  layer_vertices[l]  int64 global ids of V^l, l = 0..L   (sampling.py:18-32)
  layer_edges[l-1]   (src_pos in V^(l-1), dst_pos in V^l) for l = 1..L
"""

from __future__ import annotations

import numpy as np

__all__ = [
    "stable_groups",
    "split_sample",
    "pair_count",
    "transfer_bytes",
    "split_cost_report",
]


def stable_groups(keys: np.ndarray, g: int):
    """Stable counting sort of indices by key in [0, g) (scheduler.py:157-161).

    Returns a list of g index arrays, each in ascending original order.
    """
    keys = np.asarray(keys, dtype=np.int64)
    order = np.argsort(keys, kind="stable")
    edges = np.searchsorted(keys[order], np.arange(g + 1))
    return [order[edges[k]:edges[k + 1]] for k in range(g)]


def split_sample(layer_vertices, layer_edges, assignment, num_devices,
                 cached_lists=None):
    """Split one sample into per-device work (scheduler.py:164-254).

    Returns (splits, plan):
      splits[d] = dict(owned_gids, owned_pos, ref_gids, ref_owner  [per layer 0..L],
                       edges_src, edges_dst, self_rows             [per layer 1..L],
                       load_gids)
      plan[(l, holder, owner)] = (gids, holder_idx, owner_idx)
    Raises ValueError when a sampled vertex is outside the map (:175-178).
    """
    asn = np.asarray(assignment, dtype=np.int64)
    g = int(num_devices)
    L = len(layer_edges)
    V = [np.asarray(v, dtype=np.int64) for v in layer_vertices]
    for ids in V:
        if len(ids) and ids.max() >= len(asn):
            raise ValueError("sample vertex missing from partition map")

    owner = [asn[ids] for ids in V]                      # :180
    pos_by_dev = []                                      # owned_pos per layer/device
    rank_in_dev = []                                     # local_of_pos (:184-190)
    for l in range(L + 1):
        groups = stable_groups(owner[l], g)
        rank = np.empty(len(V[l]), dtype=np.int64)
        for grp in groups:
            rank[grp] = np.arange(len(grp), dtype=np.int64)
        pos_by_dev.append(groups)
        rank_in_dev.append(rank)

    in_cache = None
    if cached_lists is not None:                         # global mask (:193-195)
        in_cache = np.zeros(len(asn), dtype=bool)
        for ids in cached_lists:
            in_cache[np.asarray(ids, dtype=np.int64)] = True

    empty = np.empty(0, dtype=np.int64)
    splits = []
    for d in range(g):
        owned_gids = [V[l][pos_by_dev[l][d]] for l in range(L + 1)]
        load = owned_gids[0]
        if in_cache is not None and len(load):
            load = load[~in_cache[load]]                 # :197-203
        splits.append(dict(
            owned_gids=owned_gids,
            owned_pos=[pos_by_dev[l][d] for l in range(L + 1)],
            ref_gids=[empty.copy() for _ in range(L + 1)],
            ref_owner=[empty.copy() for _ in range(L + 1)],
            edges_src=[None] * L,
            edges_dst=[None] * L,
            self_rows=[None] * L,
            load_gids=load,
        ))

    plan = {}
    for l in range(1, L + 1):
        src, dst = (np.asarray(a, dtype=np.int64) for a in layer_edges[l - 1])
        src_owner = owner[l - 1][src]
        routed = 0
        for d, eidx in enumerate(stable_groups(src_owner, g)):   # :224-227
            sp = splits[d]
            es, ed = src[eidx], dst[eidx]
            routed += len(eidx)
            foreign = owner[l][ed] != d
            rpos = np.unique(ed[foreign])                          # :228-232
            rgid = V[l][rpos]
            by_gid = np.argsort(rgid)
            rpos, rgid = rpos[by_gid], rgid[by_gid]
            ref_row = np.full(len(V[l]), -1, dtype=np.int64)
            ref_row[rpos] = np.arange(len(rpos), dtype=np.int64)
            n_own = len(pos_by_dev[l][d])
            local_dst = np.where(foreign, n_own + ref_row[ed],
                                 rank_in_dev[l][ed])              # :233-238
            sp["ref_gids"][l] = rgid
            sp["ref_owner"][l] = asn[rgid]
            sp["edges_src"][l - 1] = rank_in_dev[l - 1][es]        # :241
            sp["edges_dst"][l - 1] = local_dst
            sp["self_rows"][l - 1] = rank_in_dev[l - 1][sp["owned_pos"][l]]  # :243
            for o, ridx in enumerate(stable_groups(sp["ref_owner"][l], g)):  # :244-252
                if len(ridx) == 0:
                    continue
                assert o != d, "a device cannot be its own peer"
                plan[(l, d, o)] = (rgid[ridx], ridx.astype(np.int64),
                                   rank_in_dev[l][rpos[ridx]])
        assert routed == len(src), "edge routing dropped or duplicated edges"
    return splits, plan


def pair_count(plan, l):
    """ShufflePlan.pair_count (scheduler.py:120-122)."""
    return int(sum(len(v[0]) for k, v in plan.items() if k[0] == l))


def transfer_bytes(splits, feat_dim, cached_lists=None):
    """Host bytes per device of transfer_manifest (scheduler.py:324-347)."""
    host = np.array([len(s["load_gids"]) * feat_dim * 8 for s in splits],
                    dtype=np.int64)
    loads = (np.concatenate([s["load_gids"] for s in splits])
             if splits else np.empty(0, dtype=np.int64))
    assert len(np.unique(loads)) == len(loads), "a feature vector loaded twice"
    if cached_lists is not None and len(loads):
        cached = np.concatenate([np.asarray(c, dtype=np.int64) for c in cached_lists])
        assert not np.intersect1d(loads, cached).size, "splits predate this cache"
    return host


def _spread(counts):
    """Edge skew (max-min)/mean (scheduler.py:150-154)."""
    counts = np.asarray(counts)
    mean = counts.mean() if len(counts) else 0.0
    return 0.0 if mean == 0 else float((counts.max() - counts.min()) / mean)


def split_cost_report(layer_vertices, layer_edges, assignment, g):
    """Per-vertex shuffle cost C[v^l], edge skew, locality (scheduler.py:257-309)."""
    asn = np.asarray(assignment, dtype=np.int64)
    cost_per_layer, per_dev, local, total, per_layer_cost = [], [], 0, 0, []
    for l in range(1, len(layer_edges) + 1):
        src, dst = (np.asarray(a, dtype=np.int64) for a in layer_edges[l - 1])
        so = asn[np.asarray(layer_vertices[l - 1])[src]]
        do = asn[np.asarray(layer_vertices[l])[dst]]
        per_dev.append(np.bincount(so, minlength=g))
        local += int(np.count_nonzero(so == do))
        total += len(src)
        x = so != do
        keys = np.unique(dst[x] * g + so[x])
        c = np.bincount(keys // g, minlength=len(layer_vertices[l])).astype(np.int64)
        per_layer_cost.append(c)
        cost_per_layer.append(int(c.sum()))
    edges_per_device = np.sum(per_dev, axis=0) if per_dev else np.zeros(g, np.int64)
    return dict(
        per_layer_cost=per_layer_cost,
        cost_per_layer=cost_per_layer,
        cost_total=int(sum(cost_per_layer)),
        edges_per_device_per_layer=per_dev,
        edges_per_device=edges_per_device,
        skew_per_layer=[_spread(c) for c in per_dev],
        edge_skew=_spread(edges_per_device),
        local_edge_fraction=(local / total) if total else 1.0,
        edges_total=total,
        edges_local=local,
    )
