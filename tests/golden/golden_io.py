"""Flat .npz (de)serialisation of golden cases (samples, splits, plans, grads).

Shared by make_golden.py (which runs in the build container with the real
reference importable) and the tests (which run anywhere).
"""

from __future__ import annotations

import numpy as np


def pack_sample(out, layer_vertices, layer_edges):
    out["L"] = np.int64(len(layer_edges))
    for l, v in enumerate(layer_vertices):
        out[f"V{l}"] = np.asarray(v, dtype=np.int64)
    for l, (s, d) in enumerate(layer_edges, start=1):
        out[f"E{l}_src"] = np.asarray(s, dtype=np.int64)
        out[f"E{l}_dst"] = np.asarray(d, dtype=np.int64)


def unpack_sample(z):
    L = int(z["L"])
    V = [z[f"V{l}"] for l in range(L + 1)]
    E = [(z[f"E{l}_src"], z[f"E{l}_dst"]) for l in range(1, L + 1)]
    return V, E


SPLIT_LAYER_FIELDS = ("owned_gids", "owned_pos", "ref_gids", "ref_owner")
SPLIT_EDGE_FIELDS = ("edges_src", "edges_dst", "self_rows")


def pack_splits(out, splits, plan, prefix="S"):
    """splits: list of dicts with the LocalSplit fields; plan: {(l,h,o): (gids,hidx,oidx)}."""
    out[f"{prefix}_g"] = np.int64(len(splits))
    for d, s in enumerate(splits):
        for f in SPLIT_LAYER_FIELDS:
            for l, arr in enumerate(s[f]):
                out[f"{prefix}{d}_{f}_{l}"] = np.asarray(arr, dtype=np.int64)
        for f in SPLIT_EDGE_FIELDS:
            for l, arr in enumerate(s[f], start=1):
                out[f"{prefix}{d}_{f}_{l}"] = np.asarray(arr, dtype=np.int64)
        out[f"{prefix}{d}_load_gids"] = np.asarray(s["load_gids"], dtype=np.int64)
    keys = sorted(plan)
    out[f"{prefix}_plan_keys"] = np.asarray(keys, dtype=np.int64).reshape(-1, 3)
    for (l, h, o) in keys:
        gids, hidx, oidx = plan[(l, h, o)]
        out[f"{prefix}_plan_{l}_{h}_{o}_gids"] = np.asarray(gids, dtype=np.int64)
        out[f"{prefix}_plan_{l}_{h}_{o}_hidx"] = np.asarray(hidx, dtype=np.int64)
        out[f"{prefix}_plan_{l}_{h}_{o}_oidx"] = np.asarray(oidx, dtype=np.int64)


def unpack_splits(z, L, prefix="S"):
    g = int(z[f"{prefix}_g"])
    splits = []
    for d in range(g):
        s = {}
        for f in SPLIT_LAYER_FIELDS:
            s[f] = [z[f"{prefix}{d}_{f}_{l}"] for l in range(L + 1)]
        for f in SPLIT_EDGE_FIELDS:
            s[f] = [z[f"{prefix}{d}_{f}_{l}"] for l in range(1, L + 1)]
        s["load_gids"] = z[f"{prefix}{d}_load_gids"]
        splits.append(s)
    plan = {}
    for l, h, o in z[f"{prefix}_plan_keys"].reshape(-1, 3).tolist():
        plan[(l, h, o)] = (z[f"{prefix}_plan_{l}_{h}_{o}_gids"],
                           z[f"{prefix}_plan_{l}_{h}_{o}_hidx"],
                           z[f"{prefix}_plan_{l}_{h}_{o}_oidx"])
    return splits, plan


def pack_dict(out, d, prefix):
    out[f"{prefix}__keys"] = np.array(list(d.keys()))
    for k, v in d.items():
        out[f"{prefix}__{k}"] = np.asarray(v)


def unpack_dict(z, prefix):
    return {str(k): z[f"{prefix}__{k}"] for k in z[f"{prefix}__keys"]}
