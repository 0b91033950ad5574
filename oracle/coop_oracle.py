"""CPU restatement of the cooperative split executor — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module. Restates /root/reference/pkg/src/splitgnn/engine.py:
  * exchange rounds _to_owner / _from_owner + metering     engine.py:121-156
  * _load_inputs                                           engine.py:160-167
  * GraphSAGE forward / backward                           engine.py:176-276
  * GAT forward / backward (10 exchange rounds per layer)  engine.py:280-552
  * seed_loss / run                                        engine.py:556-588
  * scatter_shuffle_forward                                engine.py:591-630
  * allreduce_and_step                                     engine.py:633-647
Devices run sequentially in ascending order (PhaseRunner workers=1,
engine.py:70-75); the owner combines holder rows in ascending sender order.

`splits` / `plan` are the dicts produced by oracle.split_oracle.split_sample.
"""

from __future__ import annotations

import numpy as np

from oracle.model_oracle import SLOPE, kind_of, leaky, seg_count, seg_max, seg_sum, softmax_xent


class CoopRun:
    """One cooperative forward/backward over prepared splits.

    After run(): .loss_sum, .grads[d], .h[d][l] (owned rows), .keep[d][l]
    (per-layer retained tensors, e.g. 'alpha' per local edge), .peer_bytes.
    """

    def __init__(self, params, splits, plan, features, labels, slope=SLOPE):
        self.p = params
        self.sp = splits
        self.plan = plan
        self.X = np.asarray(features, dtype=np.float64)
        self.y = np.asarray(labels, dtype=np.int64)
        self.g = len(splits)
        self.kind = kind_of(params)
        self.L = len(splits[0]["edges_src"]) if splits else 0
        self.slope = slope
        self.peer_bytes = 0
        self.h = [[] for _ in range(self.g)]
        self.keep = [[None] for _ in range(self.g)]
        self.grads = [{k: np.zeros_like(v) for k, v in params.items()} for _ in range(self.g)]
        self.d_h = [None] * self.g
        self.loss_parts = [0.0] * self.g

    # -- helpers -------------------------------------------------------------
    def _pairs(self, l):
        return sum(len(v[0]) for k, v in self.plan.items() if k[0] == l)

    def _push_to_owner(self, l, width, send, combine):
        """Owner d combines holder rows, holders in ascending order (engine.py:125-140)."""
        self.peer_bytes += self._pairs(l) * width * 8
        for d in range(self.g):
            for s in range(self.g):
                ent = self.plan.get((l, s, d)) if s != d else None
                if ent is not None:
                    combine(d, ent[2], send(s, ent[1]))

    def _push_from_owner(self, l, width, send, store):
        """Holder d overwrites its ref rows from each owner (engine.py:142-156)."""
        self.peer_bytes += self._pairs(l) * width * 8
        for d in range(self.g):
            for o in range(self.g):
                ent = self.plan.get((l, d, o)) if o != d else None
                if ent is not None:
                    store(d, ent[1], send(o, ent[2]))

    def _edges(self, d, l):
        s = self.sp[d]
        return s["edges_src"][l - 1], s["edges_dst"][l - 1]

    def _n(self, d, l):
        s = self.sp[d]
        return len(s["owned_gids"][l]), len(s["ref_gids"][l])

    # -- GraphSAGE (engine.py:176-276) ----------------------------------------
    def _sage_fwd(self, l, last):
        i = l - 1
        Ws, Wn, b = self.p[f"layer{i}.w_self"], self.p[f"layer{i}.w_neigh"], self.p[f"layer{i}.bias"]
        din = Ws.shape[0]
        part = []
        for d in range(self.g):
            src, dst = self._edges(d, l)
            no, nr = self._n(d, l)
            sums = seg_sum(self.h[d][l - 1][src], dst, no + nr).reshape(no + nr, din)
            cnt = seg_count(dst, no + nr)
            part.append([sums, cnt])

        def send(s, hidx):
            no, _ = self._n(s, l)
            return np.concatenate([part[s][0][no + hidx], part[s][1][no + hidx, None]], axis=1)

        def combine(d, oidx, rows):
            part[d][0][oidx] += rows[:, :din]
            part[d][1][oidx] += rows[:, din]

        self._push_to_owner(l, din + 1, send, combine)
        for d in range(self.g):
            no, _ = self._n(d, l)
            cnt = part[d][1][:no]
            mean = part[d][0][:no] / cnt[:, None]
            hs = self.h[d][l - 1][self.sp[d]["self_rows"][l - 1]]
            pre = hs @ Ws + mean @ Wn + b
            self.h[d].append(pre if last else np.maximum(pre, 0.0))
            self.keep[d].append(dict(mean=mean, counts=cnt, pre=pre))

    def _sage_bwd(self, l, last):
        i = l - 1
        Ws, Wn = self.p[f"layer{i}.w_self"], self.p[f"layer{i}.w_neigh"]
        din = Ws.shape[0]
        gown, gref, dprev = [], [], []
        for d in range(self.g):
            kp = self.keep[d][l]
            d_pre = self.d_h[d] if last else self.d_h[d] * (kp["pre"] > 0)
            selfr = self.sp[d]["self_rows"][l - 1]
            hs = self.h[d][l - 1][selfr]
            G = self.grads[d]
            G[f"layer{i}.w_self"] += hs.T @ d_pre
            G[f"layer{i}.w_neigh"] += kp["mean"].T @ d_pre
            G[f"layer{i}.bias"] += d_pre.sum(axis=0)
            dp = np.zeros_like(self.h[d][l - 1])
            dp[selfr] += d_pre @ Ws.T
            dprev.append(dp)
            gown.append((d_pre @ Wn.T) / kp["counts"][:, None])
            gref.append(np.zeros((self._n(d, l)[1], din)))

        def send(o, oidx):
            return gown[o][oidx]

        def store(d, hidx, rows):
            gref[d][hidx] = rows

        self._push_from_owner(l, din, send, store)
        for d in range(self.g):
            src, dst = self._edges(d, l)
            allg = np.concatenate([gown[d], gref[d]], axis=0)
            dprev[d] += seg_sum(allg[dst], src, len(self.h[d][l - 1])).reshape(dprev[d].shape)
            self.d_h[d] = dprev[d]

    # -- GAT (engine.py:280-552) ----------------------------------------------
    def _gat_fwd(self, l, last):
        i = l - 1
        W, a_s, a_d = self.p[f"layer{i}.w"], self.p[f"layer{i}.a_src"], self.p[f"layer{i}.a_dst"]
        dout = W.shape[1]
        st = []
        for d in range(self.g):
            z = self.h[d][l - 1] @ W
            no, nr = self._n(d, l)
            st.append(dict(z=z, s=z @ a_s, t_own=z[self.sp[d]["self_rows"][l - 1]] @ a_d,
                           t_ref=np.zeros(nr)))

        def put(key):
            def store(d, hidx, rows):
                st[d][key][hidx] = rows
            return store

        def get(key):
            return lambda o, oidx: st[o][key][oidx]

        self._push_from_owner(l, 1, get("t_own"), put("t_ref"))
        for d in range(self.g):
            src, dst = self._edges(d, l)
            no, nr = self._n(d, l)
            S = st[d]
            t_all = np.concatenate([S["t_own"], S["t_ref"]])
            S["pre_e"] = S["s"][src] + t_all[dst]
            S["e"] = leaky(S["pre_e"], self.slope)
            lm = seg_max(S["e"], dst, no + nr)
            S["m_own"], S["m_loc_ref"], S["m_ref"] = lm[:no].copy(), lm[no:], np.zeros(nr)

        def max_in(d, oidx, rows):
            st[d]["m_own"][oidx] = np.maximum(st[d]["m_own"][oidx], rows)

        def add_in(key):
            def combine(d, oidx, rows):
                st[d][key][oidx] += rows
            return combine

        self._push_to_owner(l, 1, lambda s, h: st[s]["m_loc_ref"][h], max_in)
        self._push_from_owner(l, 1, get("m_own"), put("m_ref"))
        for d in range(self.g):
            src, dst = self._edges(d, l)
            no, nr = self._n(d, l)
            S = st[d]
            m_all = np.concatenate([S["m_own"], S["m_ref"]])
            S["w_e"] = np.exp(S["e"] - m_all[dst])
            ld = seg_sum(S["w_e"], dst, no + nr)
            S["den_own"], S["den_loc_ref"], S["den_ref"] = ld[:no].copy(), ld[no:], np.zeros(nr)
        self._push_to_owner(l, 1, lambda s, h: st[s]["den_loc_ref"][h], add_in("den_own"))
        self._push_from_owner(l, 1, get("den_own"), put("den_ref"))
        for d in range(self.g):
            src, dst = self._edges(d, l)
            no, nr = self._n(d, l)
            S = st[d]
            S["den_all"] = np.concatenate([S["den_own"], S["den_ref"]])
            S["alpha"] = S["w_e"] / S["den_all"][dst]
            ln = seg_sum(S["alpha"][:, None] * S["z"][src], dst, no + nr).reshape(no + nr, dout)
            S["num_own"], S["num_loc_ref"] = ln[:no].copy(), ln[no:]
        self._push_to_owner(l, dout, lambda s, h: st[s]["num_loc_ref"][h], add_in("num_own"))
        for d in range(self.g):
            S = st[d]
            num = S["num_own"]
            self.h[d].append(num if last else np.maximum(num, 0.0))
            self.keep[d].append(dict(z=S["z"], pre_e=S["pre_e"], w_e=S["w_e"],
                                     denom_all=S["den_all"], alpha=S["alpha"], num=num,
                                     m_own=S["m_own"]))

    def _gat_bwd(self, l, last):
        i = l - 1
        W, a_s, a_d = self.p[f"layer{i}.w"], self.p[f"layer{i}.a_src"], self.p[f"layer{i}.a_dst"]
        dout = W.shape[1]
        st = []
        for d in range(self.g):
            kp = self.keep[d][l]
            no, nr = self._n(d, l)
            st.append(dict(dn_own=self.d_h[d] if last else self.d_h[d] * (kp["num"] > 0),
                           dn_ref=np.zeros((nr, dout))))

        def put(key):
            def store(d, hidx, rows):
                st[d][key][hidx] = rows
            return store

        def add_in(key):
            def combine(d, oidx, rows):
                st[d][key][oidx] += rows
            return combine

        self._push_from_owner(l, dout, lambda o, oi: st[o]["dn_own"][oi], put("dn_ref"))
        for d in range(self.g):
            src, dst = self._edges(d, l)
            no, nr = self._n(d, l)
            kp, S = self.keep[d][l], st[d]
            dn_all = np.concatenate([S["dn_own"], S["dn_ref"]], axis=0)
            z, alpha, w_e = kp["z"], kp["alpha"], kp["w_e"]
            den_e = kp["denom_all"][dst]
            d_alpha = (dn_all[dst] * z[src]).sum(axis=1)
            S["d_z"] = seg_sum(alpha[:, None] * dn_all[dst], src, len(z)).reshape(z.shape)
            pdd = seg_sum(-d_alpha * w_e / den_e ** 2, dst, no + nr)
            S["d_direct"] = d_alpha / den_e
            S["dd_own"], S["dd_loc_ref"], S["dd_ref"] = pdd[:no].copy(), pdd[no:], np.zeros(nr)
        self._push_to_owner(l, 1, lambda s, h: st[s]["dd_loc_ref"][h], add_in("dd_own"))
        self._push_from_owner(l, 1, lambda o, oi: st[o]["dd_own"][oi], put("dd_ref"))
        for d in range(self.g):
            src, dst = self._edges(d, l)
            no, nr = self._n(d, l)
            kp, S = self.keep[d][l], st[d]
            dd_all = np.concatenate([S["dd_own"], S["dd_ref"]])
            d_e = (S["d_direct"] + dd_all[dst]) * kp["w_e"]
            d_pre = d_e * np.where(kp["pre_e"] > 0, 1.0, self.slope)
            S["ds"] = seg_sum(d_pre, src, len(kp["z"]))
            pdt = seg_sum(d_pre, dst, no + nr)
            S["dt_own"], S["dt_loc_ref"] = pdt[:no].copy(), pdt[no:]
        self._push_to_owner(l, 1, lambda s, h: st[s]["dt_loc_ref"][h], add_in("dt_own"))
        for d in range(self.g):
            kp, S = self.keep[d][l], st[d]
            z = kp["z"]
            d_z = S["d_z"] + S["ds"][:, None] * a_s
            G = self.grads[d]
            G[f"layer{i}.a_src"] += z.T @ S["ds"]
            selfr = self.sp[d]["self_rows"][l - 1]
            d_z[selfr] += S["dt_own"][:, None] * a_d
            G[f"layer{i}.a_dst"] += z[selfr].T @ S["dt_own"]
            G[f"layer{i}.w"] += self.h[d][l - 1].T @ d_z
            self.d_h[d] = d_z @ W.T

    # -- driver (engine.py:556-588) -----------------------------------------------
    def forward(self):
        for d in range(self.g):
            self.h[d] = [self.X[self.sp[d]["owned_gids"][0]]]
        for l in range(1, self.L + 1):
            (self._sage_fwd if self.kind == "graphsage" else self._gat_fwd)(l, l == self.L)

    def backward(self):
        for d in range(self.g):
            yd = self.y[self.sp[d]["owned_gids"][self.L]]
            loss, d_h, dwc, dbc = softmax_xent(self.p, self.h[d][self.L], yd)
            self.loss_parts[d] = loss
            self.d_h[d] = d_h
            self.grads[d]["cls.w"] += dwc
            self.grads[d]["cls.b"] += dbc
        for l in range(self.L, 0, -1):
            (self._sage_bwd if self.kind == "graphsage" else self._gat_bwd)(l, l == self.L)

    def run(self):
        self.forward()
        self.backward()
        self.loss_sum = float(sum(self.loss_parts))
        return self.loss_sum, self.grads


def shuffle_forward(splits, plan, l, owned_rows):
    """scatter_shuffle_forward (engine.py:591-630): returns (buffers, peer_bytes)."""
    width = next((r.shape[1] for r in owned_rows if r.ndim == 2), 0)
    bufs = [np.zeros((len(s["ref_gids"][l]), width)) for s in splits]
    g = len(splits)
    for d in range(g):
        for o in range(g):
            ent = plan.get((l, d, o)) if o != d else None
            if ent is not None:
                bufs[d][ent[1]] = owned_rows[o][ent[2]]
    nbytes = sum(len(v[0]) for k, v in plan.items() if k[0] == l) * width * 8
    return bufs, nbytes


def reduce_and_sgd(params, per_device_grads, lr, num_targets):
    """allreduce_and_step (engine.py:633-647): device-order sum, then SGD."""
    tot = {k: v.copy() for k, v in per_device_grads[0].items()}
    for gd in per_device_grads[1:]:
        for k in tot:
            tot[k] += gd[k]
    scale = lr / float(num_targets)
    for k in params:
        params[k] -= scale * tot[k]
    return tot
