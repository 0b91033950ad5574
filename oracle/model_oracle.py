"""CPU restatement of the reference numeric core — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module. Restates /root/reference/pkg/src/splitgnn/models.py:
  * segment_sum / segment_max / segment_count   models.py:150-175
  * init_params (Glorot, draw order)            models.py:102-142
  * GraphSAGE layer fwd/bwd                     models.py:195-214
  * GAT layer fwd/bwd (one head)                models.py:217-261
  * classifier_loss                             models.py:287-302
  * forward/backward/run_reference              models.py:264-345
  * ModelParams.sgd_step                        models.py:95-99
Parameters are an ordered dict name -> float64 array using the reference's
names (models.py:61-75): layer{i}.w_self / .w_neigh / .bias (graphsage),
layer{i}.w / .a_src / .a_dst (gat), cls.w, cls.b.
"""

from __future__ import annotations

import numpy as np

SLOPE = 0.2


# -- segment primitives (models.py:150-175) ----------------------------------

def seg_sum(vals, keys, n_out):
    vals = np.asarray(vals, dtype=np.float64)
    out = np.zeros((n_out,) + vals.shape[1:])
    if len(keys) == 0:
        return out
    order = np.argsort(keys, kind="stable")
    k = np.asarray(keys)[order]
    heads = np.flatnonzero(np.r_[True, k[1:] != k[:-1]])
    out[k[heads]] = np.add.reduceat(vals[order], heads, axis=0)
    return out


def seg_max(vals, keys, n_out, fill=-np.inf):
    vals = np.asarray(vals, dtype=np.float64)
    out = np.full((n_out,) + vals.shape[1:], fill)
    if len(keys) == 0:
        return out
    order = np.argsort(keys, kind="stable")
    k = np.asarray(keys)[order]
    heads = np.flatnonzero(np.r_[True, k[1:] != k[:-1]])
    out[k[heads]] = np.maximum.reduceat(vals[order], heads, axis=0)
    return out


def seg_count(keys, n_out):
    return np.bincount(np.asarray(keys, dtype=np.int64), minlength=n_out).astype(np.float64)


# -- parameters (models.py:102-142) -------------------------------------------

def glorot_params(kind, feat_dim, hidden, num_classes, num_layers, seed=0):
    """Same draws, same order as init_params: per layer (w_self, w_neigh) or
    (w, a_src, a_dst), then cls.w; biases zero."""
    if kind not in ("graphsage", "gat"):
        raise ValueError(f"unknown model kind {kind!r}")
    if num_layers < 1:
        raise ValueError("num_layers must be >= 1")
    rng = np.random.default_rng(seed)

    def draw(fi, fo, shape):
        lim = np.sqrt(6.0 / (fi + fo))
        return rng.uniform(-lim, lim, size=shape)

    p = {}
    for i in range(num_layers):
        din = feat_dim if i == 0 else hidden
        if kind == "graphsage":
            p[f"layer{i}.w_self"] = draw(din, hidden, (din, hidden))
            p[f"layer{i}.w_neigh"] = draw(din, hidden, (din, hidden))
            p[f"layer{i}.bias"] = np.zeros(hidden)
        else:
            p[f"layer{i}.w"] = draw(din, hidden, (din, hidden))
            p[f"layer{i}.a_src"] = draw(hidden, 1, (hidden,))
            p[f"layer{i}.a_dst"] = draw(hidden, 1, (hidden,))
    p["cls.w"] = draw(hidden, num_classes, (hidden, num_classes))
    p["cls.b"] = np.zeros(num_classes)
    return p


def num_layers_of(params):
    return sum(1 for k in params if k.endswith((".w_self", ".w")) and k.startswith("layer"))


def kind_of(params):
    return "graphsage" if "layer0.w_self" in params else "gat"


def sgd(params, grads, lr, num_targets):
    """ModelParams.sgd_step (models.py:95-99), in place."""
    scale = lr / float(num_targets)
    for k in params:
        params[k] -= scale * grads[k]


# -- layer math ---------------------------------------------------------------

def sage_fwd(p, i, h_prev, src, dst, n_out, last):
    """models.py:195-203."""
    s = seg_sum(h_prev[src], dst, n_out)
    c = seg_count(dst, n_out)
    mean = s / c[:, None]
    pre = h_prev[:n_out] @ p[f"layer{i}.w_self"] + mean @ p[f"layer{i}.w_neigh"] + p[f"layer{i}.bias"]
    return (pre if last else np.maximum(pre, 0.0)), dict(mean=mean, counts=c, pre=pre)


def sage_bwd(p, i, h_prev, keep, src, dst, d_h, last, grads):
    """models.py:206-214."""
    d_pre = d_h if last else d_h * (keep["pre"] > 0)
    n_out = len(d_pre)
    grads[f"layer{i}.w_self"] += h_prev[:n_out].T @ d_pre
    grads[f"layer{i}.w_neigh"] += keep["mean"].T @ d_pre
    grads[f"layer{i}.bias"] += d_pre.sum(axis=0)
    d_prev = np.zeros_like(h_prev)
    d_prev[:n_out] += d_pre @ p[f"layer{i}.w_self"].T
    g_sum = (d_pre @ p[f"layer{i}.w_neigh"].T) / keep["counts"][:, None]
    d_prev += seg_sum(g_sum[dst], src, len(h_prev))
    return d_prev


def leaky(x, slope=SLOPE):
    return np.where(x > 0, x, slope * x)


def gat_fwd(p, i, h_prev, src, dst, n_out, last, slope=SLOPE):
    """models.py:217-237 (one head)."""
    z = h_prev @ p[f"layer{i}.w"]
    s = z @ p[f"layer{i}.a_src"]
    t = z[:n_out] @ p[f"layer{i}.a_dst"]
    pre_e = s[src] + t[dst]
    e = leaky(pre_e, slope)
    m = seg_max(e, dst, n_out)
    w_e = np.exp(e - m[dst])
    den = seg_sum(w_e, dst, n_out)
    alpha = w_e / den[dst]
    num = seg_sum(alpha[:, None] * z[src], dst, n_out)
    keep = dict(z=z, pre_e=pre_e, w_e=w_e, denom=den, alpha=alpha, num=num, m=m)
    return (num if last else np.maximum(num, 0.0)), keep


def gat_bwd(p, i, h_prev, keep, src, dst, d_h, last, grads, slope=SLOPE):
    """models.py:240-261 (max is a detached stabilizer, :250-252)."""
    z, alpha, w_e, den, pre_e = (keep[k] for k in ("z", "alpha", "w_e", "denom", "pre_e"))
    n_out, n_prev = len(d_h), len(h_prev)
    d_num = d_h if last else d_h * (keep["num"] > 0)
    d_alpha = (d_num[dst] * z[src]).sum(axis=1)
    d_z = seg_sum(alpha[:, None] * d_num[dst], src, n_prev)
    d_den = seg_sum(-d_alpha * w_e / den[dst] ** 2, dst, n_out)
    d_w = d_alpha / den[dst] + d_den[dst]
    d_pre = d_w * w_e * np.where(pre_e > 0, 1.0, slope)
    d_s = seg_sum(d_pre, src, n_prev)
    d_t = seg_sum(d_pre, dst, n_out)
    a_src, a_dst = p[f"layer{i}.a_src"], p[f"layer{i}.a_dst"]
    d_z += d_s[:, None] * a_src
    grads[f"layer{i}.a_src"] += z.T @ d_s
    d_z[:n_out] += d_t[:, None] * a_dst
    grads[f"layer{i}.a_dst"] += z[:n_out].T @ d_t
    grads[f"layer{i}.w"] += h_prev.T @ d_z
    return d_z @ p[f"layer{i}.w"].T


def softmax_xent(p, h, y):
    """classifier_loss (models.py:287-302): summed loss and its gradients."""
    y = np.asarray(y, dtype=np.int64)
    logits = h @ p["cls.w"] + p["cls.b"]
    mx = logits.max(axis=1, keepdims=True) if len(h) else np.zeros((0, 1))
    ex = np.exp(logits - mx)
    tot = ex.sum(axis=1, keepdims=True)
    rows = np.arange(len(y))
    loss = float((mx[:, 0] + np.log(tot[:, 0]) - logits[rows, y]).sum())
    d_log = ex / tot
    d_log[rows, y] -= 1.0
    return loss, d_log @ p["cls.w"].T, h.T @ d_log, d_log.sum(0)


# -- single-device reference (models.py:264-345) -------------------------------

def single_device_run(layer_vertices, layer_edges, params, features, labels,
                      slope=SLOPE, keep_trace=False):
    """run_reference: (loss_sum, grads) [, trace dict(h, keep)]."""
    kind = kind_of(params)
    L = len(layer_edges)
    feats = np.asarray(features, dtype=np.float64)
    h = [feats[np.asarray(layer_vertices[0], dtype=np.int64)]]
    keeps = []
    for l in range(1, L + 1):
        src, dst = (np.asarray(a, dtype=np.int64) for a in layer_edges[l - 1])
        n_out = len(layer_vertices[l])
        if kind == "graphsage":
            out, kp = sage_fwd(params, l - 1, h[-1], src, dst, n_out, l == L)
        else:
            out, kp = gat_fwd(params, l - 1, h[-1], src, dst, n_out, l == L, slope)
        h.append(out)
        keeps.append(kp)
    y = np.asarray(labels, dtype=np.int64)[np.asarray(layer_vertices[L], dtype=np.int64)]
    loss, d_h, dwc, dbc = softmax_xent(params, h[-1], y)
    grads = {k: np.zeros_like(v) for k, v in params.items()}
    for l in range(L, 0, -1):
        src, dst = (np.asarray(a, dtype=np.int64) for a in layer_edges[l - 1])
        if kind == "graphsage":
            d_h = sage_bwd(params, l - 1, h[l - 1], keeps[l - 1], src, dst, d_h, l == L, grads)
        else:
            d_h = gat_bwd(params, l - 1, h[l - 1], keeps[l - 1], src, dst, d_h, l == L, grads, slope)
    grads["cls.w"] += dwc
    grads["cls.b"] += dbc
    if keep_trace:
        return loss, grads, dict(h=h, keep=keeps)
    return loss, grads
