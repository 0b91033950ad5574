"""Multi-head GAT by COMPOSITION of the reference single-head layer —
TEST INFRASTRUCTURE ONLY (tests/, smoke(), bench CPU legs).

The reference is single-head (multi-head a non-goal at :392).
C3's 4-head GAT is pinned the only way SURVEY §8(a) row 11 allows: each head
is the reference layer (models.py:217-261, restated in model_oracle.gat_fwd /
gat_bwd) applied to the same input with its own (W_h, a_src_h, a_dst_h);
outputs are concatenated, input gradients summed.
"""

from __future__ import annotations

import numpy as np

from oracle.model_oracle import SLOPE, gat_bwd, gat_fwd, softmax_xent


def multihead_init(feat_dim, hidden, num_classes, num_layers, seed, heads):
    """Glorot draws of an H-head GAT in the product's order (each head drawn
    as a reference single-head layer, models.py:107-142, heads concatenated):
    per layer, per head (w, a_src, a_dst); then cls.w; biases zero."""
    rng = np.random.default_rng(seed)

    def draw(fi, fo, shape):
        lim = np.sqrt(6.0 / (fi + fo))
        return rng.uniform(-lim, lim, size=shape)

    p = {}
    width = hidden * heads
    for i in range(num_layers):
        d_in = feat_dim if i == 0 else width
        ws, as_, ad = [], [], []
        for _ in range(heads):
            ws.append(draw(d_in, hidden, (d_in, hidden)))
            as_.append(draw(hidden, 1, (hidden,)))
            ad.append(draw(hidden, 1, (hidden,)))
        p[f"layer{i}.w"] = np.concatenate(ws, axis=1)
        p[f"layer{i}.a_src"] = np.stack(as_)
        p[f"layer{i}.a_dst"] = np.stack(ad)
    p["cls.w"] = draw(width, num_classes, (width, num_classes))
    p["cls.b"] = np.zeros(num_classes)
    return p


def _head_params(p, i, h, dh):
    return {f"layer{i}.w": p[f"layer{i}.w"][:, h * dh:(h + 1) * dh],
            f"layer{i}.a_src": np.asarray(p[f"layer{i}.a_src"])[h],
            f"layer{i}.a_dst": np.asarray(p[f"layer{i}.a_dst"])[h]}


def multihead_run(layer_vertices, layer_edges, params, features, labels, heads, slope=SLOPE):
    """Single-device forward/backward of an L-layer H-head GAT (concat)."""
    L = len(layer_edges)
    h = [np.asarray(features, dtype=np.float64)[np.asarray(layer_vertices[0], dtype=np.int64)]]
    keeps = []
    for l in range(1, L + 1):
        src, dst = (np.asarray(a, dtype=np.int64) for a in layer_edges[l - 1])
        n_out = len(layer_vertices[l])
        D = params[f"layer{l-1}.w"].shape[1]
        dh = D // heads
        outs, kl = [], []
        for hh in range(heads):
            ph = _head_params(params, l - 1, hh, dh)
            o, kp = gat_fwd(ph, l - 1, h[-1], src, dst, n_out, l == L, slope)
            outs.append(o)
            kl.append((ph, kp))
        h.append(np.concatenate(outs, axis=1))
        keeps.append(kl)
    y = np.asarray(labels, dtype=np.int64)[np.asarray(layer_vertices[L], dtype=np.int64)]
    loss, d_h, dwc, dbc = softmax_xent(params, h[-1], y)
    grads = {k: np.zeros_like(np.asarray(v, dtype=np.float64)) for k, v in params.items()}
    for l in range(L, 0, -1):
        src, dst = (np.asarray(a, dtype=np.int64) for a in layer_edges[l - 1])
        D = params[f"layer{l-1}.w"].shape[1]
        dh = D // heads
        d_prev = np.zeros_like(h[l - 1])
        for hh, (ph, kp) in enumerate(keeps[l - 1]):
            gh = {k: np.zeros_like(np.asarray(v, dtype=np.float64)) for k, v in ph.items()}
            d_prev += gat_bwd(ph, l - 1, h[l - 1], kp, src, dst, d_h[:, hh * dh:(hh + 1) * dh],
                              l == L, gh, slope)
            grads[f"layer{l-1}.w"][:, hh * dh:(hh + 1) * dh] += gh[f"layer{l-1}.w"]
            if heads > 1:
                grads[f"layer{l-1}.a_src"][hh] += gh[f"layer{l-1}.a_src"]
                grads[f"layer{l-1}.a_dst"][hh] += gh[f"layer{l-1}.a_dst"]
            else:
                grads[f"layer{l-1}.a_src"] += gh[f"layer{l-1}.a_src"]
                grads[f"layer{l-1}.a_dst"] += gh[f"layer{l-1}.a_dst"]
        d_h = d_prev
    grads["cls.w"] += dwc
    grads["cls.b"] += dbc
    return loss, grads, h
