"""GraphSAGE / GAT model constructors and parameter stores.

Host side mirrors splitgnn.models (models.py:33-142): SageLayer, GatLayer,
ModelParams (float64 numpy, reference names and tensor order) and init_params
with the SAME Glorot draws in the same order, so a reference checkpoint and a
B200 run start from identical weights. DeviceParams is the flat fp32 copy the
kernels read; its layout follows ModelParams.tensors() order, which makes
each layer's gradient block [W_self | W_neigh | bias] (or [W | a_src | a_dst])
contiguous — the kernels' per-block partials land on it directly.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

MODEL_KINDS = ("graphsage", "gat")


@dataclass
class SageLayer:
    w_self: np.ndarray
    w_neigh: np.ndarray
    bias: np.ndarray


@dataclass
class GatLayer:
    w: np.ndarray
    a_src: np.ndarray
    a_dst: np.ndarray
    heads: int = 1


@dataclass
class ModelParams:
    kind: str
    layers: list
    w_cls: np.ndarray
    b_cls: np.ndarray
    leaky_slope: float = 0.2

    @property
    def num_layers(self):
        return len(self.layers)

    def tensors(self) -> dict:
        out = {}
        for i, layer in enumerate(self.layers):
            if self.kind == "graphsage":
                out[f"layer{i}.w_self"] = layer.w_self
                out[f"layer{i}.w_neigh"] = layer.w_neigh
                out[f"layer{i}.bias"] = layer.bias
            else:
                out[f"layer{i}.w"] = layer.w
                out[f"layer{i}.a_src"] = layer.a_src
                out[f"layer{i}.a_dst"] = layer.a_dst
        out["cls.w"] = self.w_cls
        out["cls.b"] = self.b_cls
        return out

    def zero_grads(self):
        return {k: np.zeros_like(v) for k, v in self.tensors().items()}

    def copy(self):
        if self.kind == "graphsage":
            layers = [SageLayer(l.w_self.copy(), l.w_neigh.copy(), l.bias.copy()) for l in self.layers]
        else:
            layers = [GatLayer(l.w.copy(), l.a_src.copy(), l.a_dst.copy(), l.heads) for l in self.layers]
        return ModelParams(self.kind, layers, self.w_cls.copy(), self.b_cls.copy(), self.leaky_slope)

    def sgd_step(self, grads, lr, num_targets):
        """models.py:95-99."""
        scale = lr / float(num_targets)
        for name, t in self.tensors().items():
            t -= scale * grads[name]

    def layer_dims(self, i):
        layer = self.layers[i]
        w = layer.w_self if self.kind == "graphsage" else layer.w
        return int(w.shape[0]), int(w.shape[1])

    @classmethod
    def from_reference(cls, params):
        """Adopt a reference splitgnn ModelParams (duck-typed)."""
        if params.kind == "graphsage":
            layers = [SageLayer(np.array(l.w_self, dtype=np.float64), np.array(l.w_neigh, dtype=np.float64),
                                np.array(l.bias, dtype=np.float64)) for l in params.layers]
        else:
            layers = [GatLayer(np.array(l.w, dtype=np.float64), np.array(l.a_src, dtype=np.float64),
                               np.array(l.a_dst, dtype=np.float64)) for l in params.layers]
        return cls(params.kind, layers, np.array(params.w_cls, dtype=np.float64),
                   np.array(params.b_cls, dtype=np.float64), float(params.leaky_slope))


def init_params(kind, feat_dim, hidden, num_classes, num_layers, seed=0, leaky_slope=0.2, heads=1):
    """Glorot-uniform weights, zero biases, reference draw order
    (models.py:107-142). GAT with heads > 1 (not in the reference)
    draws each head as a reference single-head layer, in head order, and
    concatenates: W = [W_1 | ... | W_H] (d_in x H*hidden), a_src / a_dst
    (H x hidden); the next layer's input width is H*hidden."""
    if kind not in MODEL_KINDS:
        raise ValueError(f"unknown model kind {kind!r}")
    if num_layers < 1:
        raise ValueError("num_layers must be >= 1")
    rng = np.random.default_rng(seed)

    def glorot(fi, fo, shape):
        lim = np.sqrt(6.0 / (fi + fo))
        return rng.uniform(-lim, lim, size=shape)

    if heads < 1 or (heads > 1 and kind != "gat"):
        raise ValueError("heads > 1 is only defined for GAT")
    layers = []
    width = hidden * heads
    for i in range(num_layers):
        d_in = feat_dim if i == 0 else width
        if kind == "graphsage":
            layers.append(SageLayer(glorot(d_in, hidden, (d_in, hidden)),
                                    glorot(d_in, hidden, (d_in, hidden)), np.zeros(hidden)))
        elif heads == 1:
            layers.append(GatLayer(glorot(d_in, hidden, (d_in, hidden)),
                                   glorot(hidden, 1, (hidden,)), glorot(hidden, 1, (hidden,))))
        else:
            ws, as_, ad = [], [], []
            for _ in range(heads):
                ws.append(glorot(d_in, hidden, (d_in, hidden)))
                as_.append(glorot(hidden, 1, (hidden,)))
                ad.append(glorot(hidden, 1, (hidden,)))
            layers.append(GatLayer(np.concatenate(ws, axis=1), np.stack(as_), np.stack(ad), heads))
    w_cls = glorot(width, num_classes, (width, num_classes))
    return ModelParams(kind, layers, w_cls, np.zeros(num_classes), leaky_slope)


class DeviceParams:
    """Flat fp32 parameter buffer on the GPU (+ name -> view)."""

    def __init__(self, kind, names, shapes, flat, leaky_slope=0.2):
        self.kind = kind
        self.names = list(names)
        self.shapes = [tuple(s) for s in shapes]
        self.sizes = [int(np.prod(s)) if len(s) else 1 for s in self.shapes]
        self.offsets = np.r_[0, np.cumsum(self.sizes)].astype(np.int64)
        self.n = int(self.offsets[-1])
        self.flat = flat
        self.leaky_slope = float(leaky_slope)
        self.num_layers = sum(1 for k in self.names if k.endswith((".w_self", ".w")) and k.startswith("layer"))

    @classmethod
    def from_host(cls, params: ModelParams, device="cuda"):
        t = params.tensors()
        host = np.concatenate([np.asarray(v, dtype=np.float32).reshape(-1) for v in t.values()])
        flat = torch.from_numpy(host).to(device)
        return cls(params.kind, t.keys(), [np.shape(v) for v in t.values()], flat, params.leaky_slope)

    def offset(self, name):
        return int(self.offsets[self.names.index(name)])

    def view(self, name):
        i = self.names.index(name)
        return self.flat[self.offsets[i]:self.offsets[i + 1]].view(self.shapes[i])

    def layer_dims(self, i):
        s = self.shapes[self.names.index(f"layer{i}.w_self" if self.kind == "graphsage" else f"layer{i}.w")]
        return int(s[0]), int(s[1])

    def heads_of(self, i):
        """GAT heads of layer i (a_src is (heads, d_head) for heads > 1)."""
        if self.kind != "gat":
            return 1
        s = self.shapes[self.names.index(f"layer{i}.a_src")]
        return int(s[0]) if len(s) == 2 else 1

    @property
    def num_classes(self):
        return int(self.shapes[self.names.index("cls.w")][1])

    @property
    def hidden(self):
        return int(self.shapes[self.names.index("cls.w")][0])

    def grads_to_dict(self, flat_grads) -> dict:
        g = flat_grads[: self.n].double().cpu().numpy()
        return {k: g[self.offsets[i]:self.offsets[i + 1]].reshape(self.shapes[i]).copy()
                for i, k in enumerate(self.names)}

    def to_host(self) -> ModelParams:
        d = self.grads_to_dict(self.flat)
        L = self.num_layers
        if self.kind == "graphsage":
            layers = [SageLayer(d[f"layer{i}.w_self"], d[f"layer{i}.w_neigh"], d[f"layer{i}.bias"])
                      for i in range(L)]
        else:
            layers = [GatLayer(d[f"layer{i}.w"], d[f"layer{i}.a_src"], d[f"layer{i}.a_dst"],
                               self.heads_of(i)) for i in range(L)]
        return ModelParams(self.kind, layers, d["cls.w"], d["cls.b"], self.leaky_slope)
