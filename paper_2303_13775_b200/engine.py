"""Cooperative split-parallel forward/backward on B200 (engine.py of the reference).

SplitStep is the device-resident hot path: for every local device it launches
the sm_100a kernels layer by layer, with the push-to-owner / push-from-owner
rounds handed to a transport (one copy kernel when all devices share this
GPU, NCCL all-to-all-v when each device is its own process/GPU). No host
synchronisation happens inside a step except the transports' use of the
count descriptor, which is fetched once per iteration.

The reference-facing API keeps the reference's names and signatures:
SplitExecutor (engine.py:95-588), PhaseRunner (:58-79),
scatter_shuffle_forward (:591-630), allreduce_and_step (:633-647) and
Trainer / train_model (:655-870).
"""

from __future__ import annotations

import contextlib
import ctypes
import gc
import os

import time

import numpy as np
import torch

from paper_2303_13775_b200 import _lib
from paper_2303_13775_b200.exchange import LocalTransport
from paper_2303_13775_b200.features import FeatureStore
from paper_2303_13775_b200.metrics import EpochMetrics, IterationMetrics, account_transfer, union_edge_count
from paper_2303_13775_b200.models import DeviceParams, ModelParams, init_params
from paper_2303_13775_b200.partition import CacheState, PartitionMap, full_cache
from paper_2303_13775_b200.sampling import epoch_batches, sample_microbatches, sample_minibatch
from paper_2303_13775_b200.scheduler import DeviceSplit, pinned_from, split_cost_packed, split_minibatch

DEBUG_CHECK_FINITE = False
NB_PARTIAL = 2 * 148  # max blocks of the deterministic partial reductions (measured best vs 592, 888)
# layers with at least this many edges (capacity) take the load-balanced
# transposed SpMM (tspmm.cu); below it hub rows are short (max out-degree
# ~25-125 at C2 layers 2-3) and the single-kernel row-per-warp path is faster
TSPMM_MIN_EDGES = int(os.environ.get("SG_TSPMM_MIN_EDGES", "65536"))  # load-balanced transposed SpMM from this many edges


def _pipe_direct():
    """run_pipelined with one captured graph per staging slot (SG_PIPE_DIRECT=0:
    one graph and a device-to-device copy of each staged sample)."""
    return os.environ.get("SG_PIPE_DIRECT", "1") == "1"


@contextlib.contextmanager
def _capturing(graph):
    """CUDA-graph capture that other threads' CUDA calls cannot invalidate
    (thread-local capture mode) and that no garbage collection interrupts: a
    collected step object's destructor frees pinned memory (cudaFreeHost), which
    is illegal while a capture is open (seen as an intermittent
    cudaErrorStreamCaptureInvalidated in back-to-back tests)."""
    was = gc.isenabled()
    gc.collect()
    gc.disable()
    try:
        with torch.cuda.graph(graph, capture_error_mode="thread_local"):
            yield
    finally:
        if was:
            gc.enable()


def _nblocks(rows, tile=32):
    return int(max(1, min(NB_PARTIAL, (int(rows) + tile - 1) // tile)))


def _r4(x):
    return (int(x) + 3) // 4 * 4


def _f32(n, *shape, device):
    return torch.empty((max(int(n), 1),) + tuple(shape), dtype=torch.float32, device=device)


class SplitStep:
    """One iteration's forward + backward for `devices` of a DeviceSplit."""

    def __init__(self, dparams: DeviceParams, dsplit: DeviceSplit, feats: FeatureStore,
                 labels_dev, devices=None, transport=None, exact=True, record_events=False):
        self.p = dparams
        self.ds = dsplit
        self.f = feats
        self.labels = labels_dev
        self.g, self.L = dsplit.g, dsplit.L
        self.devices = list(range(self.g)) if devices is None else list(devices)
        self.transport = transport or LocalTransport()
        self.meta = dsplit.host_meta() if exact else None
        self.dev = dsplit.device
        self.kind = dparams.kind
        if self.kind != "graphsage":
            from paper_2303_13775_b200 import gat  # noqa: F401  (GAT path)
        self.h = [None] * (self.L + 1)
        self.keep = [None] * (self.L + 1)
        self.grads = None
        # record_events: False | True/"all" (every phase) | "agg" (layer-1 SpMM, and
        # the GAT layer-1 projection: the bench's roofline kernels, only)
        self.events = {} if record_events else None
        self.ev_mode = "agg" if record_events == "agg" else "all"
        self.wire_bytes = 0
        self.host_bytes = 0

    # -- size bounds (exact when the count descriptor was fetched) ------------
    def n_own(self, l, d):
        return int(self.meta.n_own[l][d]) if self.meta is not None else self.ds.nV[l]

    def n_rows(self, l, d):
        if self.meta is not None:
            return int(self.meta.n_own[l][d] + self.meta.n_ref[l][d])
        return self.ds.nV[l] + self.ds.pair_bound(l)

    def n_recv(self, l, d):
        if self.meta is not None:
            return int(self.meta.recv_off[l][d + 1] - self.meta.recv_off[l][d])
        return self.ds.pair_bound(l)

    def _ev(self, name):
        if self.events is None:
            return None
        if self.ev_mode == "agg" and not name.startswith(("agg1", "roof1", "wgd1")):
            return None
        try:  # external=True: a real event-record node when captured in a CUDA graph
            e = torch.cuda.Event(enable_timing=True, external=True)
        except TypeError:
            e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.events.setdefault(name, []).append(e)
        return e

    # -- forward ----------------------------------------------------------------
    def layer0(self):
        ds, st = self.ds, _lib.stream_ptr()
        if self.g == 1 and self.f.identity:
            # one device, whole table cached in id order: the layer-0 owned rows
            # are the sample positions and their table rows are the gids
            self.src_row0 = ds.V
            return
        self.src_row0 = torch.empty(max(ds.nV[0], 1), dtype=torch.int32, device=self.dev)
        if not ds.all_cached:
            # the sample may hold uncached layer-0 rows: stage this step's load
            # lists on the device (exact or captured alike)
            if self.meta is not None:
                self.host_bytes += 4 * self.f.feat_dim * sum(int(self.meta.n_load[d]) for d in self.devices)
                if sum(int(self.meta.n_load[d]) for d in self.devices):
                    self.f.stage_misses(ds, self.devices)
            else:
                self.f.stage_misses(ds, self.devices)
        for d in self.devices:
            _lib.call("sg_layer0_rows", _lib.ptr(ds.ws), ds.lay, d, _lib.ptr(ds.V),
                      _lib.ptr(self.f.cache_slot), int(self.f.n_cached), _lib.ptr(self.src_row0), st)

    def _fused_ok(self, w, dout, dperm):
        """Single-device split: the update can run inside the aggregation."""
        return (self.g == 1 and dperm is None and w % 4 == 0 and w <= 128 and dout in (4, 8, 16, 32)
                and not getattr(self, "no_fuse", False))

    def _xbuf(self, P, *shape):
        """A round's exchange buffer: the peer-mapped one of a PeerTransport
        (same request order on every rank), else a plain device tensor."""
        shared = getattr(self.transport, "shared", None)
        if shared is None or self.g == 1 or P <= 0:
            return _f32(P, *shape, device=self.dev)
        width = int(np.prod(shape)) if shape else 1
        return shared(P, width).view(P, *shape)

    def _final_fused_ok(self, w, dout, dperm, any_g=False):
        """The last layer, the loss and the last layer's row-local backward run
        as one kernel (sg_sage_final_fused at g = 1; sg_sage_final_combine after
        the push-to-owner round otherwise)."""
        return ((self.g == 1 and dperm is None or any_g) and w % 4 == 0 and w <= 128 and dout <= 64
                and self.p.num_classes <= 1024 and not getattr(self, "no_fuse", False)
                and not getattr(self, "no_fuse_final", False))

    def _begin_grads(self):
        """Flat per-device gradient buffers (+ loss slot) and the partial-sum jobs."""
        if self.grads is None:
            self.grads = {d: torch.empty(self.p.n + 1, dtype=torch.float32, device=self.dev)
                          for d in self.devices}
            self.jobs = []
            self._partials = []

    def _final_fused(self, l, w, dout, h_prev, src_row, comb=None):
        """Last layer + loss + the layer's row-local backward, one kernel per
        device: aggregating itself (g = 1) or combining the local partial with
        the holders' partials after the push-to-owner round (comb = (sums,
        counts, recv, stride))."""
        ds, p, st = self.ds, self.p, _lib.stream_ptr()
        self._begin_grads()
        C = p.num_classes
        nV = ds.nV[l]
        mean = _f32(nV, w, device=self.dev)
        counts = comb[1] if comb is not None else _f32(nV, device=self.dev)
        h = _f32(nV, dout, device=self.dev)
        need_prev = l > 1
        d_self = _f32(nV, w, device=self.dev) if need_prev else None
        d_sums = _f32(nV, w, device=self.dev) if need_prev else None
        ncls, nlay = dout * C + C + 1, 2 * w * dout + dout
        W = [_lib.ptr(p.view(f"layer{l-1}.w_self")), _lib.ptr(p.view(f"layer{l-1}.w_neigh")),
             _lib.ptr(p.view(f"layer{l-1}.bias")), _lib.ptr(p.view("cls.w")), _lib.ptr(p.view("cls.b"))]
        self._ev(f"ph:final{l}:s")
        for d in self.devices:
            n = self.n_own(l, d)
            nb = max(1, min(_nblocks(n, tile=8), 2 * 148))
            part_c = _f32(nb * ncls, device=self.dev)
            part_l = _f32(nb * nlay, device=self.dev)
            if comb is None:
                _lib.call("sg_sage_final_fused", _lib.ptr(ds.ws), ds.lay, d, _lib.ptr(h_prev), _lib.ptr(src_row),
                          w, dout, C, *W, _lib.ptr(ds.V), _lib.ptr(self.labels), _lib.ptr(mean),
                          _lib.ptr(counts), _lib.ptr(h), _lib.ptr(d_self), _lib.ptr(d_sums), _lib.ptr(part_c),
                          _lib.ptr(part_l), nb, n, st)
            else:
                sums, _, recv, SW = comb
                _lib.call("sg_sage_final_combine", _lib.ptr(ds.ws), ds.lay, d, _lib.ptr(h_prev),
                          _lib.ptr(src_row), w, dout, C, *W, _lib.ptr(ds.V), _lib.ptr(self.labels),
                          _lib.ptr(sums), _lib.ptr(recv), SW, _lib.ptr(mean), _lib.ptr(counts), _lib.ptr(h),
                          _lib.ptr(d_self), _lib.ptr(d_sums), _lib.ptr(part_c), _lib.ptr(part_l), nb, n, st)
            self.jobs.append((part_c, nb, ncls, self.grads[d], p.offset("cls.w")))
            self.jobs.append((part_l, nb, nlay, self.grads[d], p.offset(f"layer{l-1}.w_self")))
            self._partials += [part_c, part_l]
        self._ev(f"ph:final{l}:e")
        self.h[l] = h
        self.keep[l] = dict(mean=mean, counts=counts)
        self._final_rows = (d_self, d_sums)

    def _padded_ok(self, l, w, dout, dperm):
        """Layer 1 reads a padded feature table only through the kernels that
        take a row stride: the one-kernel layer (g = 1) or the g > 1
        aggregation + combine; never as the last layer."""
        if l != 1 or self.L < 2 or w <= 64:
            return False
        return self._fused_ok(w, dout, dperm) or self._combine_ok(w, dout, _r4(w + 1))

    def _combine_ok(self, w, dout, SW):
        return (w % 4 == 0 and w <= 128 and dout in (4, 8, 16, 32) and SW % 4 == 0
                and not getattr(self, "no_fuse", False))

    def _dst_perm(self):
        """CSR-by-destination for samples whose edges are not grouped by dst."""
        if self.ds.dst_grouped:
            return None
        if getattr(self, "_dperm", None) is None:
            ds, st = self.ds, _lib.stream_ptr()
            n_max = max(int(ds.lay.nEtot), 1)
            self._dperm = {}
            for d in self.devices:
                ws = torch.empty(int(_lib.load().sg_sort_ws_bytes(n_max)), dtype=torch.uint8, device=self.dev)
                keys = torch.empty(n_max, dtype=torch.int32, device=self.dev)
                perm = torch.empty(n_max, dtype=torch.int32, device=self.dev)
                ndev = torch.empty(1, dtype=torch.int32, device=self.dev)
                _lib.call("sg_dst_csr", _lib.ptr(ds.ws), ds.lay, d, _lib.ptr(ws), n_max, _lib.ptr(ndev),
                          _lib.ptr(keys), _lib.ptr(perm), st)
                self._dperm[d] = (perm, ws, keys, ndev)
        return self._dperm

    def phase(self, name):
        """Context manager recording start/end events of a phase (profiling)."""
        step = self

        class _P:
            def __enter__(self_):
                if step.events is not None:
                    step._ev(f"ph:{name}:s")

            def __exit__(self_, *a):
                if step.events is not None:
                    step._ev(f"ph:{name}:e")
        return _P()

    def phase_ms(self):
        """{phase: ms} from the most recent recording (after synchronisation)."""
        out = {}
        if not self.events:
            return out
        for k, v in self.events.items():
            if k.startswith("ph:") and k.endswith(":s"):
                name = k[3:-2]
                e = self.events.get(f"ph:{name}:e")
                if e:
                    out[name] = out.get(name, 0.0) + sum(a.elapsed_time(b) for a, b in zip(v, e))
        return out

    def forward(self):
        if hasattr(self.transport, "begin_step"):
            self.transport.begin_step()
        if self.kind != "graphsage":
            from paper_2303_13775_b200.gat import gat_forward
            gat_forward(self)
            self._check_finite()
            return
        ds, p, st = self.ds, self.p, _lib.stream_ptr()
        self.grads, self._final_rows = None, None
        with self.phase("layer0"):
            self.layer0()
        dperm = self._dst_perm()
        self._launch_src_csr_async(2)
        self.h[0] = self.f.table
        for l in range(1, self.L + 1):
            w, dout = p.layer_dims(l - 1)
            final = int(l == self.L)
            h_prev, src_row = (self.f.table, self.src_row0) if l == 1 else (self.h[l - 1], None)
            hst = self.f.row_stride if l == 1 else w
            nV = ds.nV[l]
            if hst != w and not self._padded_ok(l, w, dout, dperm):
                raise ValueError("padded feature rows are read only by the wide SAGE layer-1 kernels "
                                 "(build the FeatureStore with pad_rows=False for this model)")
            if l == self.L and self._final_fused_ok(w, dout, dperm):
                self._final_fused(l, w, dout, h_prev, src_row)
                continue
            if self._fused_ok(w, dout, dperm):
                mean = _f32(nV, w, device=self.dev)
                counts = _f32(nV, device=self.dev)
                hs = _f32(nV, w, device=self.dev)
                h = _f32(nV, dout, device=self.dev)
                self._ev(f"agg{l}_start")
                self._ev(f"ph:agg+update{l}:s")
                _lib.call("sg_sage_fused_fwd", _lib.ptr(ds.ws), ds.lay, l, 0, _lib.ptr(h_prev),
                          _lib.ptr(src_row), w, hst, dout, _lib.ptr(p.view(f"layer{l-1}.w_self")),
                          _lib.ptr(p.view(f"layer{l-1}.w_neigh")), _lib.ptr(p.view(f"layer{l-1}.bias")),
                          final, _lib.ptr(mean), _lib.ptr(counts), _lib.ptr(hs), _lib.ptr(h),
                          self.n_own(l, 0), st)
                self._ev(f"agg{l}_end")
                self._ev(f"ph:agg+update{l}:e")
                self.h[l] = h
                self.keep[l] = dict(mean=mean, counts=counts, hs=hs)
                continue
            sums = _f32(nV, w, device=self.dev)
            counts = _f32(nV, device=self.dev)
            SW = _r4(w + 1)
            P = ds.pair_bound(l)
            recv = self._xbuf(P, SW)
            peer_push = hasattr(self.transport, "peers_of") and self.g > 1 and P > 0
            send = None if peer_push else _f32(P, SW, device=self.dev)
            self._ev(f"agg{l}_start")
            self._ev(f"ph:agg{l}:s")
            for d in self.devices:
                if peer_push:  # push-to-owner fused into the aggregation epilogue
                    _lib.call("sg_sage_agg_fwd_peer", _lib.ptr(ds.ws), ds.lay, l, d, _lib.ptr(h_prev),
                              _lib.ptr(src_row), w, hst, _lib.ptr(sums), _lib.ptr(counts),
                              _lib.ptr(self.transport.peers_of(recv)), SW,
                              _lib.ptr(dperm[d][0]) if dperm is not None else None, self.n_rows(l, d), st)
                elif dperm is None:
                    _lib.call("sg_sage_agg_fwd", _lib.ptr(ds.ws), ds.lay, l, d, _lib.ptr(h_prev),
                              _lib.ptr(src_row), w, hst, _lib.ptr(sums), _lib.ptr(counts), _lib.ptr(send),
                              SW, self.n_rows(l, d), st)
                else:
                    _lib.call("sg_sage_agg_fwd_perm", _lib.ptr(ds.ws), ds.lay, l, d, _lib.ptr(h_prev),
                              _lib.ptr(src_row), w, hst, _lib.ptr(sums), _lib.ptr(counts), _lib.ptr(send),
                              SW, _lib.ptr(dperm[d][0]), self.n_rows(l, d), st)
            self._ev(f"agg{l}_end")
            self._ev(f"ph:agg{l}:e")
            if self.g > 1 and P > 0:
                if peer_push:
                    self.transport.to_owner(ds, l, None, recv, SW, pushed=True)
                else:
                    self.transport.to_owner(ds, l, send, recv, SW)
                if self.meta is not None:
                    self.wire_bytes += int(self.meta.npairs[l]) * SW * 4
            if self._combine_ok(w, dout, SW):
                if l == self.L and self._final_fused_ok(w, dout, None, any_g=True):
                    self._final_fused(l, w, dout, h_prev, src_row, comb=(sums, counts, recv, SW))
                    continue
                mean = _f32(nV, w, device=self.dev)
                h = _f32(nV, dout, device=self.dev)
                hs = _f32(nV, w, device=self.dev)
                self._ev(f"ph:update{l}:s")
                for d in self.devices:
                    _lib.call("sg_sage_combine_fwd", _lib.ptr(ds.ws), ds.lay, l, d, _lib.ptr(h_prev),
                              _lib.ptr(src_row), w, hst, dout, _lib.ptr(p.view(f"layer{l-1}.w_self")),
                              _lib.ptr(p.view(f"layer{l-1}.w_neigh")), _lib.ptr(p.view(f"layer{l-1}.bias")),
                              final, _lib.ptr(sums), _lib.ptr(counts), _lib.ptr(recv), SW, _lib.ptr(mean),
                              _lib.ptr(hs), _lib.ptr(h), self.n_own(l, d), st)
                self._ev(f"ph:update{l}:e")
                self.h[l] = h
                self.keep[l] = dict(mean=mean, counts=counts, hs=hs)
                continue
            mean = _f32(nV, w, device=self.dev)
            h = _f32(nV, dout, device=self.dev)
            tiled = w % 4 == 0 and dout in (4, 8, 16, 32)
            hs = _f32(nV, w, device=self.dev) if tiled else None
            self._ev(f"ph:update{l}:s")
            for d in self.devices:
                _lib.call("sg_sage_update", _lib.ptr(ds.ws), ds.lay, l, d, _lib.ptr(h_prev),
                          _lib.ptr(src_row), w, dout, _lib.ptr(sums), _lib.ptr(counts), _lib.ptr(recv),
                          SW, _lib.ptr(p.view(f"layer{l-1}.w_self")), _lib.ptr(p.view(f"layer{l-1}.w_neigh")),
                          _lib.ptr(p.view(f"layer{l-1}.bias")), final, _lib.ptr(mean), _lib.ptr(h),
                          _lib.ptr(hs), self.n_own(l, d), st)
            self._ev(f"ph:update{l}:e")
            self.h[l] = h
            self.keep[l] = dict(mean=mean, counts=counts)
            if hs is not None:
                self.keep[l]["hs"] = hs

        self._check_finite()

    def _check_finite(self):
        """engine.py:49-55 (DEBUG_CHECK_FINITE): scan every layer's owned output
        rows of every local device; FloatingPointError names the first layer
        with a NaN / Inf. Covers every forward kernel path (one-kernel layers,
        the fused last layer, owner combine, GAT). Eager steps only: a
        captured graph cannot branch on device values."""
        if not DEBUG_CHECK_FINITE or self.meta is None or torch.cuda.is_current_stream_capturing():
            return
        for l in range(1, self.L + 1):
            h = self.h[l]
            for d in self.devices:
                b, n = int(self.meta.own_off[l][d]), int(self.meta.n_own[l][d])
                if n and not bool(torch.isfinite(h[b:b + n]).all()):
                    raise FloatingPointError(f"non-finite values in {self.kind} layer {l} output")

    # -- loss + backward -----------------------------------------------------------
    def _src_csr(self, lmin, val_mode=1):
        ds, st = self.ds, _lib.stream_ptr()
        n_max = max(int(ds.lay.nEtot - ds.lay.eoff[lmin - 1]), 1)
        rows = max(sum(ds.nV[l - 1] for l in range(lmin, self.L + 1)), 1)
        out = {}
        for d in self.devices:
            ws = torch.empty(int(_lib.load().sg_sort_ws_bytes(n_max)), dtype=torch.uint8, device=self.dev)
            keys = torch.empty(n_max, dtype=torch.int32, device=self.dev)
            perm = torch.empty(n_max, dtype=torch.int32, device=self.dev)
            ndev = torch.empty(1, dtype=torch.int32, device=self.dev)
            beg = torch.empty(rows, dtype=torch.int32, device=self.dev)
            end = torch.empty(rows, dtype=torch.int32, device=self.dev)
            _lib.call("sg_src_csr", _lib.ptr(ds.ws), ds.lay, d, lmin, val_mode, _lib.ptr(ws), n_max,
                      _lib.ptr(ndev), _lib.ptr(keys), _lib.ptr(perm), _lib.ptr(beg), _lib.ptr(end), rows, st)
            out[d] = (perm, beg, end, ws, keys, ndev)
        kb, acc = {}, 0
        for l in range(lmin, self.L + 1):
            kb[l] = acc
            acc += ds.nV[l - 1]
        return out, kb

    def _launch_src_csr_async(self, lmin):
        """The CSR-by-source build depends only on the split: run it on a side
        stream so it overlaps the forward pass (also inside a captured graph)."""
        self._csr_async = None
        if self.L < lmin or self.events is not None and self.ev_mode == "all":
            return  # phase-profiling runs keep it serial so its time is visible
        main = torch.cuda.current_stream()
        side = getattr(self, "_side", None)
        if side is None:
            side = torch.cuda.Stream(device=self.dev)
            self._side = side
        side.wait_stream(main)
        with torch.cuda.stream(side):
            out = self._src_csr(lmin, val_mode=1 if self.kind == "graphsage" else 0)
        self._csr_async = (lmin, out, side)

    def _join_src_csr(self, lmin):
        pending = getattr(self, "_csr_async", None)
        if pending is not None and pending[0] == lmin:
            torch.cuda.current_stream().wait_stream(pending[2])
            self._csr_async = None
            return pending[1]
        if self.L < lmin:
            return {}, {}
        return self._src_csr(lmin, val_mode=1 if self.kind == "graphsage" else 0)

    def loss(self):
        ds, p, st = self.ds, self.p, _lib.stream_ptr()
        L = self.L
        hid, C = p.hidden, p.num_classes
        # every parameter block (and the loss slot) is written by a reduction job
        self._begin_grads()
        self.d_h = _f32(ds.nV[L], hid, device=self.dev)
        ncls = hid * C + C + 1
        for d in self.devices:
            nb = _nblocks(self.n_own(L, d), tile=8)
            part = _f32(nb * ncls, device=self.dev)
            _lib.call("sg_cls_loss", _lib.ptr(ds.ws), ds.lay, d, _lib.ptr(ds.V), _lib.ptr(self.labels),
                      _lib.ptr(self.h[L]), hid, C, _lib.ptr(p.view("cls.w")), _lib.ptr(p.view("cls.b")),
                      _lib.ptr(self.d_h), _lib.ptr(part), nb, self.n_own(L, d), st)
            self.jobs.append((part, nb, ncls, self.grads[d], p.offset("cls.w")))
            self._partials.append(part)

    def backward(self):
        if self.kind != "graphsage":
            from paper_2303_13775_b200.gat import gat_backward
            self.loss()
            gat_backward(self)
            self.reduce()
            return
        ds, p, st = self.ds, self.p, _lib.stream_ptr()
        fused_final = getattr(self, "_final_rows", None) is not None
        if not fused_final:
            with self.phase("loss"):
                self.loss()
        with self.phase("src_csr_join"):
            csr, kb = self._join_src_csr(2)
        d_h = None if fused_final else self.d_h
        rows_done = None  # (d_self, d_sums) of a layer whose row backward ran inside the scatter
        for l in range(self.L, 0, -1):
            w, dout = p.layer_dims(l - 1)
            final = int(l == self.L)
            need_prev = l > 1  # d(loss)/d(features) is never used
            h_prev, src_row = (self.f.table, self.src_row0) if l == 1 else (self.h[l - 1], None)
            nV = ds.nV[l]
            if l == self.L and fused_final:
                d_self, d_sums = self._final_rows
                devs = []
            elif rows_done is not None:
                d_self, d_sums = rows_done
                rows_done = None
                devs = []
            else:
                d_self = _f32(nV, w, device=self.dev) if need_prev else None
                d_sums = _f32(nV, w, device=self.dev) if need_prev else None
                devs = self.devices
            npart = 2 * w * dout + dout
            self._ev(f"ph:bwd_rows{l}:s")
            hs = self.keep[l].get("hs")
            if hs is not None:
                h_prev, src_row = hs, None
            for d in devs:
                nb = _nblocks(self.n_own(l, d))
                part = _f32(nb * npart, device=self.dev)
                _lib.call("sg_sage_bwd_rows", _lib.ptr(ds.ws), ds.lay, l, d, _lib.ptr(h_prev),
                          _lib.ptr(src_row), w, dout, _lib.ptr(d_h), _lib.ptr(self.h[l]), final,
                          _lib.ptr(self.keep[l]["mean"]), _lib.ptr(self.keep[l]["counts"]),
                          _lib.ptr(p.view(f"layer{l-1}.w_self")), _lib.ptr(p.view(f"layer{l-1}.w_neigh")),
                          _lib.ptr(part), nb, _lib.ptr(d_self), _lib.ptr(d_sums),
                          int(hs is not None), self.n_own(l, d), st)
                self.jobs.append((part, nb, npart, self.grads[d], p.offset(f"layer{l-1}.w_self")))
                self._partials.append(part)
            self._ev(f"ph:bwd_rows{l}:e")
            if not need_prev:
                break
            SWb = _r4(w)
            P = ds.pair_bound(l)
            bsend = self._xbuf(P, SWb)
            brecv = _f32(P, SWb, device=self.dev)
            if self.g > 1 and P > 0:
                for d in self.devices:
                    _lib.call("sg_pack_from_owner", _lib.ptr(ds.ws), ds.lay, l, d, _lib.ptr(d_sums), w,
                              _lib.ptr(bsend), SWb, self.n_recv(l, d), st)
                self.transport.from_owner(ds, l, bsend, brecv, SWb)
                if self.meta is not None:
                    self.wire_bytes += int(self.meta.npairs[l]) * SWb * 4
            w_in, _ = p.layer_dims(l - 2)
            hs_prev = self.keep[l - 1].get("hs")
            # (measured: a win for narrow rows; for the wide layer-1 rows the tile's
            # scatter latency and hub rows stall the weight-gradient pipeline)
            if (w in (4, 8, 16, 32) and w_in % 4 == 0 and w_in <= 64 and hs_prev is not None
                    and ds.nE[l - 1] < TSPMM_MIN_EDGES and not getattr(self, "no_fuse", False)):
                # transposed SpMM of layer l fused with layer l-1's row backward
                need2 = l - 1 > 1
                d_self2 = _f32(ds.nV[l - 1], w_in, device=self.dev) if need2 else None
                d_sums2 = _f32(ds.nV[l - 1], w_in, device=self.dev) if need2 else None
                npart2 = 2 * w_in * w + w
                self._ev(f"ph:scatter_rows{l}:s")
                for d in self.devices:
                    perm, beg, end, _, keys = csr[d][:5]
                    nb = _nblocks(self.n_own(l - 1, d))
                    part = _f32(nb * npart2, device=self.dev)
                    _lib.call("sg_sage_scatter_bwd_rows", _lib.ptr(ds.ws), ds.lay, l, d, _lib.ptr(d_self),
                              _lib.ptr(d_sums), _lib.ptr(brecv), SWb, _lib.ptr(perm), _lib.ptr(beg), _lib.ptr(end),
                              kb[l], _lib.ptr(hs_prev), w_in, w, _lib.ptr(self.h[l - 1]),
                              _lib.ptr(self.keep[l - 1]["mean"]), _lib.ptr(self.keep[l - 1]["counts"]),
                              _lib.ptr(p.view(f"layer{l-2}.w_self")), _lib.ptr(p.view(f"layer{l-2}.w_neigh")),
                              _lib.ptr(part), nb, _lib.ptr(d_self2), _lib.ptr(d_sums2), self.n_own(l - 1, d), st)
                    self.jobs.append((part, nb, npart2, self.grads[d], p.offset(f"layer{l-2}.w_self")))
                    self._partials.append(part)
                self._ev(f"ph:scatter_rows{l}:e")
                rows_done = (d_self2, d_sums2)
                d_h = None
                continue
            d_prev = _f32(ds.nV[l - 1], w, device=self.dev)
            self._ev(f"ph:scatter{l}:s")
            for d in self.devices:
                perm, beg, end, _, keys = csr[d][:5]
                if (w + 3) // 4 * 4 <= 192 and ds.nE[l - 1] >= TSPMM_MIN_EDGES:  # load-balanced pieces
                    nf = int(_lib.load().sg_tspmm_part_floats(ds.nE[l - 1], w, 0))
                    part = _f32(nf, device=self.dev)
                    _lib.call("sg_sage_scatter_bwd_lb", _lib.ptr(ds.ws), ds.lay, l, d, w, _lib.ptr(d_self),
                              _lib.ptr(d_sums), _lib.ptr(brecv), SWb, _lib.ptr(keys), _lib.ptr(perm),
                              _lib.ptr(beg), _lib.ptr(end), kb[l], 2, _lib.ptr(part), ds.nE[l - 1],
                              _lib.ptr(d_prev), self.n_own(l - 1, d), st)
                else:
                    _lib.call("sg_sage_scatter_bwd", _lib.ptr(ds.ws), ds.lay, l, d, w, _lib.ptr(d_self),
                              _lib.ptr(d_sums), _lib.ptr(brecv), SWb, _lib.ptr(perm), _lib.ptr(beg),
                              _lib.ptr(end), kb[l], _lib.ptr(d_prev), self.n_own(l - 1, d), st)
            self._ev(f"ph:scatter{l}:e")
            d_h = d_prev
        with self.phase("reduce"):
            self.reduce()

    def reduce(self):
        """Per-block partials -> per-device flat gradients (+ loss slot)."""
        jobs = []
        max_n = 1
        # (flat params, scale) or (flat params, lr, device num_targets): g = 1,
        # SGD fused into the reduction
        sgd = getattr(self, "sgd", None)
        for part, nb, n, gbuf, off in self.jobs:
            jobs += [part.data_ptr(), nb, n, gbuf.data_ptr() + 4 * off]
            if sgd is not None:
                jobs += [sgd[0].data_ptr() + 4 * off, max(0, min(n, self.p.n - off))]
            max_n = max(max_n, n)
        table = np.asarray(jobs, dtype=np.int64)
        if sgd is not None and len(sgd) == 3:
            _lib.call("sg_reduce_partials_sgd_nt", _lib.ptr(table), len(self.jobs), max_n, float(sgd[1]),
                      sgd[2].data_ptr(), _lib.stream_ptr())
        elif sgd is not None:
            _lib.call("sg_reduce_partials_sgd", _lib.ptr(table), len(self.jobs), max_n, float(sgd[1]),
                      _lib.stream_ptr())
        else:
            _lib.call("sg_reduce_partials", _lib.ptr(table), len(self.jobs), max_n, _lib.stream_ptr())

    def loss_sum_dev(self):
        return sum(self.grads[d][self.p.n] for d in self.devices)

    def run(self):
        with _pdl_for(self.kind):
            self.forward()
            self.backward()
        return self


class _pdl_for:
    """Programmatic dependent launch for the GAT step (SG_GAT_PDL=0 turns it
    off). Round 1 measured the GAT step faster without it (0.69-0.70 vs 0.73
    ms); on the round-2 kernels, with the tcgen05 projection's setup moved
    before its griddepcontrol.wait, it is slightly faster with it (C3 0.4554
    vs 0.4571 ms) and bit-identical."""

    def __init__(self, kind):
        self.off = kind != "graphsage" and os.environ.get("SG_GAT_PDL", "1") != "1"

    def __enter__(self):
        if self.off:
            lib = _lib.load()
            self.prev = lib.sg_get_pdl()
            lib.sg_set_pdl(0)

    def __exit__(self, *a):
        if self.off:
            _lib.load().sg_set_pdl(self.prev)


class PhaseRunner:
    """Signature-compatible with the reference (engine.py:58-79). Device work
    is stream-ordered, so phases need no threads; `workers` is accepted and
    results are identical for any value."""

    def __init__(self, num_devices, workers=1):
        self.num_devices = num_devices
        self.workers = max(1, int(workers))

    def each(self, fn):
        for d in range(self.num_devices):
            fn(d)

    def close(self):
        pass


# ---- reference-compatible executor --------------------------------------------

_FEATS = {}
_LABELS = {}


def _feature_store(features, cache, device, pad_rows=False):
    if isinstance(features, FeatureStore):
        return features
    key = (id(features), id(cache), bool(pad_rows))
    hit = _FEATS.get(key)
    if hit is not None and hit[0] is features:
        return hit[1]
    fs = FeatureStore.from_host(np.asarray(features), cache, device=device, pad_rows=pad_rows)
    _FEATS.clear()
    _FEATS[key] = (features, fs)
    return fs


def _labels_dev(labels, device):
    if isinstance(labels, torch.Tensor):
        return labels.to(device=device, dtype=torch.int32)
    hit = _LABELS.get(id(labels))
    if hit is not None and hit[0] is labels:
        return hit[1]
    t = torch.from_numpy(np.asarray(labels, dtype=np.int32)).to(device)
    _LABELS.clear()
    _LABELS[id(labels)] = (labels, t)
    return t


class GradDict(dict):
    """dict name -> float64 ndarray (reference type) that also carries the
    device-resident fp32 flat gradient for allreduce_and_step. Built from the
    device on first access (a caller that only hands it to
    allreduce_and_step never pays the D2H)."""

    device_flat = None
    host_flat = None
    dparams = None

    def __init__(self, data=None, dparams=None, device_flat=None, host_flat=None):
        super().__init__(data or {})
        self.dparams, self.device_flat, self.host_flat = dparams, device_flat, host_flat
        self._lazy = data is None and (device_flat is not None or host_flat is not None)

    def _fill(self):
        if self._lazy:
            self._lazy = False
            src = torch.from_numpy(self.host_flat) if self.host_flat is not None else self.device_flat
            dict.update(self, self.dparams.grads_to_dict(src))

    for _m in ("__getitem__", "__iter__", "__len__", "__contains__", "__repr__", "__eq__", "keys", "values",
               "items", "get", "copy"):
        def _wrap(self, *a, _name=_m, **k):
            self._fill()
            return getattr(dict, _name)(self, *a, **k)
        locals()[_m] = _wrap
    del _m, _wrap


class _StateView:
    def __init__(self, split):
        self.split = split
        self.h = []
        self.layer = []
        self.loss_sum = 0.0


class _PinnedFlat:
    """A pinned host copy of a flat parameter buffer with the event of its
    last async copy (a buffer is rewritten only after that copy completed)."""

    def __init__(self, n):
        self.t = torch.empty(n, dtype=torch.float32, pin_memory=True)
        self.np = self.t.numpy()
        self.ev = None

    def wait(self):
        if self.ev is not None:
            self.ev.synchronize()

    def record(self):
        # one event per buffer, re-recorded: every rewrite of the buffer waits
        # for the latest copy first, so only the latest record matters
        if self.ev is None:
            self.ev = torch.cuda.Event()
        self.ev.record(_lib.current_stream())


def _pinned_of(dp, which, shape=None):
    key = "_pin_" + which
    pf = getattr(dp, key, None)
    if pf is None:
        pf = _PinnedFlat(dp.n if shape is None else shape)
        setattr(dp, key, pf)
    return pf


class _ParamTable:
    """Pointers / sizes / element sizes of a host ModelParams' arrays for the
    native host helpers (sg_host_params_gather, sg_host_sum_sgd), kept on the
    ModelParams and rebuilt when one of its arrays is replaced."""

    __slots__ = ("arrs", "ptrs", "sizes", "eb", "n", "k", "a_ptrs", "a_sizes", "a_eb", "applied", "a_applied")

    def __init__(self, arrs):
        self.arrs = arrs
        self.k = len(arrs)
        self.ptrs = np.array([a.ctypes.data for a in arrs], dtype=np.uint64)
        self.sizes = np.array([a.size for a in arrs], dtype=np.int64)
        self.eb = np.array([a.itemsize for a in arrs], dtype=np.int32)
        self.n = int(self.sizes.sum())
        self.applied = np.zeros(1, dtype=np.int32)
        # addresses as ints: a numpy .ctypes.data costs ~1 us per access
        self.a_ptrs, self.a_sizes, self.a_eb, self.a_applied = (
            x.ctypes.data for x in (self.ptrs, self.sizes, self.eb, self.applied))


def _param_arrays(params):
    """params.tensors().values() in the same order, without building the names."""
    out = []
    if params.kind == "graphsage":
        for l in params.layers:
            out += (l.w_self, l.w_neigh, l.bias)
    else:
        for l in params.layers:
            out += (l.w, l.a_src, l.a_dst)
    out += (params.w_cls, params.b_cls)
    return out


def _param_table(params):
    """The native pointer table of `params` (host ModelParams), or None when an
    array is not a C-contiguous fp32 / fp64 ndarray (numpy paths then)."""
    arrs = _param_arrays(params)
    tab = getattr(params, "_sg_table", None)
    if tab is not None and len(tab.arrs) == len(arrs) and all(a is b for a, b in zip(tab.arrs, arrs)):
        return tab
    for a in arrs:
        if not (isinstance(a, np.ndarray) and a.dtype in (np.float32, np.float64) and a.flags.c_contiguous
                and a.flags.writeable):
            return None
    tab = _ParamTable(arrs)
    try:
        params._sg_table = tab
    except AttributeError:
        pass
    return tab


def _host_flat(params):
    tab = _param_table(params) if isinstance(params, ModelParams) else None
    if tab is not None:
        out = np.empty(tab.n, dtype=np.float32)
        _lib.call("sg_host_params_gather", tab.k, tab.a_ptrs, tab.a_sizes, tab.a_eb, out.ctypes.data)
        return out
    return np.concatenate([np.ravel(v) for v in params.tensors().values()], dtype=np.float32,
                          casting="same_kind")


class SplitExecutor:
    """engine.py:95-588: SplitExecutor(params, splits, plan, features, labels,
    runner, record).run() -> (loss_sum, per-device gradient dicts).

    Samples from split_minibatch (destination-grouped, i.e. every sampler's
    output) run as a replay of a cached CUDA graph of the whole step (split
    included; SG_API_EAGER=1 forces the eager kernels); the per-device
    gradients and the loss return in one pinned D2H, and allreduce_and_step
    applies the device-order sum + SGD to the host parameters."""

    def __init__(self, params, splits, plan, features, labels, runner=None, record=None):
        ds = getattr(splits, "device_split", None) or getattr(plan, "device_split", None)
        if ds is None:
            raise TypeError("splits/plan must come from paper_2303_13775_b200.split_minibatch "
                            "(they carry the device-resident split)")
        if not isinstance(params, ModelParams):
            params = ModelParams.from_reference(params)
        self.params = params
        self.splits = splits
        self.plan = plan
        self.ds = ds
        self.record = record
        self.runner = runner
        self.g = ds.g
        self.L = params.num_layers
        F = int(np.asarray(features).shape[1]) if not isinstance(features, FeatureStore) else 0
        hid = int(np.shape(_param_arrays(params)[0])[1]) if self.L else 0  # layer0.w_self / layer0.w
        pad = (params.kind == "graphsage" and self.L >= 2 and 64 < F <= 128 and F % 4 == 0
               and hid in (4, 8, 16, 32))  # wide layer 1 read in whole 128 B lines
        self.feats = _feature_store(features, ds.cache, ds.device, pad_rows=pad)
        self.labels = _labels_dev(labels, ds.device)
        self._states = None
        self.graph = None
        if (getattr(ds, "packed", None) is not None and os.environ.get("SG_API_EAGER") != "1"
                and not DEBUG_CHECK_FINITE):  # the per-layer finite scan runs on the eager kernels
            self.graph = _api_graph(params, ds, self.feats, self.labels)
            self.dparams = self.graph.p
            self.step = None
        else:
            self.dparams = DeviceParams.from_host(params, ds.device)
            self.step = SplitStep(self.dparams, ds, self.feats, self.labels)

    def _to_eager(self):
        """forward() / backward() called separately (reference engine.py:556-
        588): run this executor on the eager kernels."""
        if self.step is None:
            self.graph = None
            self.dparams = DeviceParams.from_host(self.params, self.ds.device)
            self.step = SplitStep(self.dparams, self.ds, self.feats, self.labels)

    def forward(self):
        self._to_eager()
        with _pdl_for(self.step.kind):
            self.step.forward()
        self._states = None

    def backward(self):
        self._to_eager()
        with _pdl_for(self.step.kind):
            self.step.backward()

    def _meter(self):
        if self.record is None:
            return
        for l in range(1, self.L + 1):
            d_in, d_out = self.params.layer_dims(l - 1)
            width = (2 * d_in + 1) if self.params.kind == "graphsage" else (2 * d_out + 8)
            account_transfer(self.record, "peer", self.ds.pair_count(l) * width * 8)
        if self.step is not None:
            self.record.wire_bytes += self.step.wire_bytes

    def run(self):
        if self.graph is not None:
            return self._run_graph()
        self.forward()
        self.backward()
        self._meter()
        loss = float(self.step.loss_sum_dev().item())
        out = [GradDict(dparams=self.dparams, device_flat=self.step.grads[d]) for d in range(self.g)]
        self._loss_slots = [float(gd.device_flat[self.dparams.n].item()) for gd in out]
        return loss, out

    def _run_graph(self):
        gs = self.graph
        host = _host_flat(self.params)
        self._snapshot = host
        st = _lib.stream_ptr()
        up = _pinned_of(gs.p, "up")
        up.wait()
        up.np[:] = host
        _lib.call("sg_copy_async", _lib.ptr(gs.p.flat), _lib.ptr(up.t), 4 * gs.p.n, st)
        up.record()
        buf, used, _ = self.ds.packed  # the sample into the graph's input buffer
        _lib.call("sg_copy_async", _lib.ptr(gs.inp.buf), _lib.ptr(buf), 4 * int(used), st)
        gs.replay()
        n = gs.p.n
        # every device's flat gradient (+ loss slot) comes back in one pinned
        # D2H: the loss needs a host sync anyway, and allreduce_and_step then
        # applies the device-order sum + SGD to the host parameters directly
        g = len(gs.out)
        dn = _pinned_of(gs.p, f"grads{g}", (g, n + 1))
        dn.wait()
        for d, f in enumerate(gs.out):
            _lib.call("sg_copy_async", _lib.ptr(dn.t) + 4 * d * (n + 1), _lib.ptr(f), 4 * (n + 1), st)
        dn.record()
        dn.wait()
        hg = dn.np.copy()  # the graph's buffers (and this slot) are reused by the next run
        self._meter()
        out = []
        for d in range(g):
            gd = GradDict(dparams=gs.p, host_flat=hg[d])
            gd.param_snapshot = host
            out.append(gd)
        self._loss_slots = [float(hg[d, n]) for d in range(g)]
        loss = hg[0, n]
        for d in range(1, g):
            loss = np.float32(loss + hg[d, n])
        return float(loss), out

    @property
    def states(self):
        """Per-device owned-row activations (reference DeviceState.h / .layer),
        materialised on demand from the device. On the captured path they are
        recomputed by one eager forward of the same split and parameters
        (the graph's activation buffers are shared across replays)."""
        if self._states is None:
            if self.step is None:
                snap = getattr(self, "_snapshot", None)
                if snap is not None:  # the parameters run() used, even if updated since
                    gp = self.graph.p
                    dp = DeviceParams(gp.kind, gp.names, gp.shapes, torch.from_numpy(snap).to(self.ds.device),
                                      gp.leaky_slope)
                else:
                    dp = DeviceParams.from_host(self.params, self.ds.device)
                self.step = SplitStep(dp, self.ds, self.feats, self.labels)
                with _pdl_for(self.step.kind):
                    self.step.forward()
            self._states = _materialise_states(self)
            slots = getattr(self, "_loss_slots", None)
            for d, st in enumerate(self._states):
                st.loss_sum = float(slots[d]) if slots is not None else 0.0
        return self._states


def _materialise_states(ex):
    ds, st = ex.ds, ex.step
    m = ds.host_meta()
    states = []
    table = ex.feats.table
    for d in range(ds.g):
        sv = _StateView(ex.splits[d] if d < len(ex.splits) else None)
        b0, n0 = int(m.own_off[0][d]), int(m.n_own[0][d])
        F = table.shape[1]
        h0 = torch.empty((max(n0, 1), F), dtype=torch.float32, device=ds.device)
        _lib.call("sg_gather_rows", _lib.ptr(table), _lib.ptr(st.src_row0[b0:]), n0, F, _lib.ptr(h0),
                  _lib.stream_ptr())
        sv.h.append(h0[:n0, :ex.feats.feat_dim].double().cpu().numpy())
        sv.layer.append(None)
        for l in range(1, ds.L + 1):
            b, n = int(m.own_off[l][d]), int(m.n_own[l][d])
            sv.h.append(st.h[l][b:b + n].double().cpu().numpy())
            keep = {}
            for k, v in (st.keep[l] or {}).items():
                if k in ("alpha", "pre_e", "w_e"):
                    eb = int(ds.lay.eoff[l - 1]) + int(m.edge_off[l - 1][d])
                    keep[k] = v[eb:eb + int(m.n_edge[l - 1][d])].double().cpu().numpy()
                elif k in ("z", "s"):  # rows at layer l-1
                    b1, n1 = int(m.own_off[l - 1][d]), int(m.n_own[l - 1][d])
                    keep[k] = v[b1:b1 + n1].double().cpu().numpy()
                else:
                    keep[k] = v[b:b + n].double().cpu().numpy()
            sv.layer.append(keep)
        states.append(sv)
    return states


def scatter_shuffle_forward(splits, plan, l, owned_rows, runner=None, record=None, transport=None):
    """engine.py:591-630: fill every device's reference rows at layer l from
    the owners' rows (one push-from-owner round on the GPU).

    transport=None moves all g devices' rows in this process (LocalTransport:
    one copy kernel). With a rank transport (NcclTransport / PeerTransport)
    this process is device `transport.rank`: only owned_rows[rank] is read
    (the other entries may be None), its rows are packed into the round's
    buffer, the round runs over NCCL / peer memory, and the returned list holds
    this device's reference rows at index `rank` (other entries empty).
    Meters pair_count(l) * width * 8 bytes like the reference (:620-627)."""
    ds = getattr(splits, "device_split", None) or getattr(plan, "device_split", None)
    if ds is None:
        raise TypeError("splits must come from paper_2303_13775_b200.split_minibatch")
    m = ds.host_meta()
    devices = list(range(ds.g)) if transport is None else [int(transport.rank)]
    if transport is not None and int(getattr(transport, "world", ds.g)) != ds.g:
        raise ValueError("transport world size differs from the split's device count")
    width = 0
    for d in devices:
        r = owned_rows[d]
        if r is not None and np.ndim(r) == 2:
            width = int(np.shape(r)[1])
            break
    if transport is not None and width == 0 and ds.pair_bound(l) > 0:
        raise ValueError("owned_rows[rank] must be a 2-D array (rows x width, rows may be 0): "
                         "every rank needs the round's width")
    if record is not None:
        account_transfer(record, "peer", int(m.npairs[l]) * width * 8)
    nV = ds.nV[l]
    rows = torch.zeros((max(nV, 1), max(width, 1)), dtype=torch.float32, device=ds.device)
    for d in devices:
        n = int(m.n_own[l][d])
        if n and width:
            b = int(m.own_off[l][d])
            rows[b:b + n] = torch.as_tensor(np.asarray(owned_rows[d], dtype=np.float32).reshape(n, width),
                                            device=ds.device)
    P = ds.pair_bound(l)
    host = None
    if ds.g > 1 and P > 0 and width:
        stride = _r4(width)
        tp = transport or LocalTransport()
        if hasattr(tp, "begin_step"):
            tp.begin_step()
        shared = getattr(tp, "shared", None)
        bsend = shared(P, stride) if shared is not None else _f32(P, stride, device=ds.device)
        brecv = _f32(P, stride, device=ds.device)
        st = _lib.stream_ptr()
        for d in devices:
            _lib.call("sg_pack_from_owner", _lib.ptr(ds.ws), ds.lay, l, d, _lib.ptr(rows), width,
                      _lib.ptr(bsend), stride, int(m.recv_off[l][d + 1] - m.recv_off[l][d]), st)
        tp.from_owner(ds, l, bsend, brecv, stride)
        refs = _f32(P, width, device=ds.device)
        for d in devices:
            _lib.call("sg_unpack_refs", _lib.ptr(ds.ws), ds.lay, l, d, _lib.ptr(brecv), stride, width,
                      _lib.ptr(refs), int(m.n_ref[l][d]), st)
        host = refs.double().cpu().numpy()
        if hasattr(tp, "check"):
            tp.check()
    out = []
    for d in range(ds.g):
        n = int(m.n_ref[l][d])
        if d not in devices or n == 0 or width == 0 or host is None:
            out.append(np.zeros((n if d in devices else 0, width)))
        else:
            b = int(m.ref_off[l][d])
            out.append(host[b:b + n].copy())
    return out


def allreduce_and_step(params, per_device_grads, lr, num_targets):
    """engine.py:633-647: device-order gradient sum + SGD.
    Mutates `params` (host ModelParams, reference semantics) and returns the
    summed gradients (reference dicts built on first access). Gradients from a
    captured SplitExecutor run are already on the host (one D2H with the
    loss): when `params` still holds the values the run used, one native call
    sums them and applies the step in place (sg_host_sum_sgd, the device
    kernel's arithmetic). Otherwise the sum + SGD run on the GPU
    (sg_sum_sgd) and the updated parameters come back with one D2H."""
    if isinstance(params, DeviceParams):
        dp = params
        host_params = None
    else:
        host_params = params if isinstance(params, ModelParams) else ModelParams.from_reference(params)
        dp = None
        snap = getattr(per_device_grads[0], "param_snapshot", None) if per_device_grads else None
        hfl = [getattr(gd, "host_flat", None) for gd in per_device_grads]
        if snap is not None and hfl and all(h is not None for h in hfl):
            tab = _param_table(host_params) if params is host_params else None
            if tab is not None:  # one native call: unchanged-check, device-order sum, SGD, write-back
                dpr = per_device_grads[0].dparams
                if tab.n == dpr.n and all(h.dtype == np.float32 and h.flags.c_contiguous for h in hfl):
                    total = np.empty(dpr.n, dtype=np.float32)
                    gp = (ctypes.c_void_p * len(hfl))(*[h.ctypes.data for h in hfl])
                    _lib.call("sg_host_sum_sgd", tab.k, tab.a_ptrs, tab.a_sizes, tab.a_eb, snap.ctypes.data, gp,
                              len(hfl), dpr.n, float(lr) / float(num_targets), total.ctypes.data, tab.a_applied)
                    if tab.applied[0]:
                        return GradDict(dparams=dpr, host_flat=total)
            else:
                cur = _host_flat(host_params)
                if np.array_equal(cur, snap):
                    return _host_sum_sgd(params, host_params, per_device_grads, hfl, cur, lr, num_targets)
        cand = getattr(per_device_grads[0], "dparams", None) if per_device_grads else None
        if snap is not None and cand is not None and all(getattr(gd, "dparams", None) is cand
                                                         for gd in per_device_grads):
            if np.array_equal(_host_flat(host_params), snap):
                dp = cand
        if dp is None:
            dp = DeviceParams.from_host(host_params)
    flats = []
    for gd in per_device_grads:
        f = getattr(gd, "device_flat", None)
        if f is None:
            t = np.concatenate([np.asarray(gd[k], dtype=np.float32).reshape(-1) for k in dp.names])
            f = torch.from_numpy(t).to(dp.flat.device)
        flats.append(f)
    ptrs = np.asarray([f.data_ptr() for f in flats], dtype=np.int64)
    total = torch.empty(dp.n, dtype=torch.float32, device=dp.flat.device)
    _lib.call("sg_sum_sgd", _lib.ptr(dp.flat), _lib.ptr(total), _lib.ptr(ptrs), len(flats), dp.n,
              float(lr) / float(num_targets), _lib.stream_ptr())
    summed = GradDict(dparams=dp, device_flat=total)
    if host_params is not None:
        down = _pinned_of(dp, "down")  # one pinned D2H of the updated parameters
        down.wait()
        down.t.copy_(dp.flat, non_blocking=True)
        down.record()
        down.wait()
        new = {k: down.np[dp.offsets[i]:dp.offsets[i + 1]].reshape(dp.shapes[i]) for i, k in enumerate(dp.names)}
        for k, v in host_params.tensors().items():
            v[...] = new[k]
        if params is not host_params:  # reference object: write back in place
            _write_back_reference(params, new)
    return summed


def _host_sum_sgd(params, host_params, per_device_grads, hfl, cur, lr, num_targets):
    """allreduce_and_step for gradients a captured SplitExecutor run already
    brought to the host (with the loss, in one D2H): the device-order fp32 sum
    and p -= lr/num_targets * g of sg_sum_sgd (a fused multiply-add: the exact
    product of two fp32 values is formed in float64, then rounded once more),
    on the host parameters that the run used."""
    dp = per_device_grads[0].dparams
    n = dp.n
    total = np.array(hfl[0][:n], dtype=np.float32)
    for h in hfl[1:]:
        total += h[:n]
    scale = float(np.float32(float(lr) / float(num_targets)))
    newf = (cur.astype(np.float64) - scale * total.astype(np.float64)).astype(np.float32)
    off = dp.offsets
    t = host_params.tensors()
    if list(t.keys()) == list(dp.names):
        for i, v in enumerate(t.values()):
            v[...] = newf[off[i]:off[i + 1]].reshape(v.shape)
    else:
        for i, k in enumerate(dp.names):
            t[k][...] = newf[off[i]:off[i + 1]].reshape(dp.shapes[i])
    if params is not host_params:  # reference object: write back in place
        _write_back_reference(params, {k: newf[off[i]:off[i + 1]].reshape(dp.shapes[i])
                                       for i, k in enumerate(dp.names)})
    return GradDict(dparams=dp, host_flat=total)


def _write_back_reference(params, new):
    for i, layer in enumerate(params.layers):
        for k in vars(layer):
            key = f"layer{i}.{k}"
            if key in new:
                getattr(layer, k)[...] = new[key]
    params.w_cls[...] = new["cls.w"]
    params.b_cls[...] = new["cls.b"]


# ---- training driver (engine.py:655-870) -----------------------------------------

class Trainer:
    """Drives sample -> split -> cooperative step -> all-reduce + SGD, with the
    model parameters resident on the GPU for the whole epoch."""

    def __init__(self, graph, pm: PartitionMap, cache: CacheState | None, labels, features=None,
                 device="cuda"):
        feats = features if features is not None else graph.features
        if feats is None:
            raise ValueError("graph has no features attached")
        self.graph = graph
        self.pm = pm
        self.cache = cache
        self.labels = np.asarray(labels, dtype=np.int64)
        self.num_devices = pm.num_devices
        self.device = torch.device(device)
        self.feats = feats if isinstance(feats, FeatureStore) else FeatureStore.from_host(feats, cache, device=device)
        self._host_feats = None if isinstance(feats, FeatureStore) else np.asarray(feats)
        self.labels_dev = _labels_dev(self.labels, self.device)
        self._one = None

    def _one_device(self):
        """Single-device context for the `single` and `data_parallel` modes: a
        one-part map and the whole feature table resident (each micro-batch /
        mini-batch runs as the g = 1 case of the same kernels)."""
        if self._one is None:
            n = self.graph.num_vertices
            pm1 = PartitionMap(np.zeros(n, dtype=np.int64), 1, 0.0)
            cache1 = full_cache(pm1)
            if self._host_feats is not None:
                f1 = FeatureStore.from_host(self._host_feats, cache1, device=self.device)
            elif getattr(self.feats, "identity", False):
                f1 = self.feats
            else:
                raise ValueError("single/data_parallel modes need the whole feature table "
                                 "(construct the Trainer with host features)")
            masks = (self.cache.device_masks(n) if self.cache is not None and hasattr(self.cache, "device_masks")
                     else [np.zeros(n, dtype=bool) for _ in range(self.num_devices)])
            self._one = (pm1, cache1, f1, masks)
        return self._one

    def single_step(self, sample, dparams):
        """One device runs the whole mini-batch (engine.py:677-683)."""
        pm1, cache1, f1, _ = self._one_device()
        ds = DeviceSplit.from_sample(sample, pm1, cache1, self.device)
        step = SplitStep(dparams, ds, f1, self.labels_dev)
        step.run()
        return step

    def data_parallel_step(self, micro_samples, dparams, record=None):
        """Each device trains on its own independently sampled micro-batch
        (engine.py:701-725); returns the per-device steps (gradients in
        step.grads[0]), summed in device order by the caller."""
        pm1, cache1, f1, masks = self._one_device()
        if record is not None:
            for d, m in enumerate(micro_samples):
                v0 = np.asarray(m.vertices(0), dtype=np.int64)
                missed = int(np.count_nonzero(~masks[d][v0]))
                account_transfer(record, "host", missed * self.graph_feat_dim() * 8)
        steps = []
        for m in micro_samples:
            ds = DeviceSplit.from_sample(m, pm1, cache1, self.device)
            st = SplitStep(dparams, ds, f1, self.labels_dev)
            st.run()
            steps.append(st)
        return steps

    def split_step(self, sample, dparams, record=None):
        ds = DeviceSplit.from_sample(sample, self.pm, self.cache, self.device)
        step = SplitStep(dparams, ds, self.feats, self.labels_dev)
        step.run()
        return step, ds

    def run_epoch(self, mode, params, *, seed, epoch, fanouts, batch_size, lr, workers=1,
                  train_set=None):
        if mode not in ("single", "split", "data_parallel"):
            raise ValueError(f"unknown mode {mode!r}")
        g = self.num_devices
        if train_set is None:
            train_set = np.arange(self.graph.num_vertices, dtype=np.int64)
        ss = np.random.SeedSequence([seed, epoch])
        batches = epoch_batches(train_set, batch_size, np.random.default_rng(ss.spawn(1)[0]))
        host_params = params if isinstance(params, ModelParams) else ModelParams.from_reference(params)
        dp = DeviceParams.from_host(host_params, self.device)
        metrics = EpochMetrics(epoch=epoch, mode=mode, num_devices=g)
        for it, targets in enumerate(batches):
            brng = np.random.default_rng(ss.spawn(1)[0])
            rec = IterationMetrics(iteration=it, mode=mode, num_devices=g)
            t0 = time.perf_counter()
            if mode == "data_parallel":
                micros = sample_microbatches(self.graph, targets, g, fanouts, brng)
            else:
                sample = sample_minibatch(self.graph, targets, fanouts, brng)
            t1 = time.perf_counter()
            rec.sample_ms = (t1 - t0) * 1e3
            if mode != "split":
                t2 = time.perf_counter()
                if mode == "single":
                    rec.host_bytes = len(sample.vertices(0)) * self.graph_feat_dim() * 8
                    steps = [self.single_step(sample, dp)]
                    rec.edges_per_device[0] = sample.total_edges
                    rec.local_edge_fraction = 1.0
                else:
                    steps = self.data_parallel_step(micros, dp, rec)
                    for d in range(g):
                        rec.edges_per_device[d] = micros[d].total_edges
                    total = int(sum(m.total_edges for m in micros))
                    rec.redundant_edges = total - union_edge_count(micros)
                    counts = rec.edges_per_device.astype(np.float64)
                    mean = counts.mean()
                    rec.edge_skew = float((counts.max() - counts.min()) / mean) if mean else 0.0
                    rec.local_edge_fraction = 1.0
                ptrs = np.asarray([st.grads[0].data_ptr() for st in steps], dtype=np.int64)
                _lib.call("sg_sum_sgd", _lib.ptr(dp.flat), None, _lib.ptr(ptrs), len(steps), dp.n,
                          float(lr) / len(targets), _lib.stream_ptr())
                loss = sum(float(st.grads[0][dp.n].item()) for st in steps)
                t3 = time.perf_counter()
                rec.train_ms = (t3 - t2) * 1e3
                rec.loss = loss / len(targets)
                metrics.iterations.append(rec)
                continue
            ds = DeviceSplit.from_sample(sample, self.pm, self.cache, self.device)
            m = ds.host_meta()
            t2 = time.perf_counter()
            rec.split_ms = (t2 - t1) * 1e3
            account_transfer(rec, "host", int(m.load_off[g]) * self.graph_feat_dim() * 8)
            step = SplitStep(dp, ds, self.feats, self.labels_dev)
            step.run()
            ptrs = np.asarray([step.grads[d].data_ptr() for d in range(g)], dtype=np.int64)
            _lib.call("sg_sum_sgd", _lib.ptr(dp.flat), None, _lib.ptr(ptrs), g, dp.n,
                      float(lr) / len(targets), _lib.stream_ptr())
            loss = sum(float(step.grads[d][dp.n].item()) for d in range(g))
            for l in range(1, ds.L + 1):
                d_in, d_out = dp.layer_dims(l - 1)
                width = (2 * d_in + 1) if dp.kind == "graphsage" else (2 * d_out + 8)
                account_transfer(rec, "peer", int(m.npairs[l]) * width * 8)
            rec.wire_bytes = step.wire_bytes
            rec.edges_per_device = np.array([sum(int(m.n_edge[l][d]) for l in range(ds.L)) for d in range(g)],
                                            dtype=np.int64)
            report = split_cost_packed(ds.V, ds.esrc, ds.edst, ds.nV, ds.nE, self.pm, g)
            rec.edge_skew = report.edge_skew
            rec.local_edge_fraction = report.local_edge_fraction
            t3 = time.perf_counter()
            rec.train_ms = (t3 - t2) * 1e3
            rec.loss = loss / len(targets)
            metrics.iterations.append(rec)
        new = dp.to_host().tensors()
        for k, v in host_params.tensors().items():
            v[...] = new[k]
        if params is not host_params:
            _write_back_reference(params, new)
        return metrics

    def graph_feat_dim(self):
        return int(self.feats.feat_dim)


def train_model(graph, pm, cache, labels, *, model_kind, num_layers, hidden, fanouts, batch_size,
                lr, epochs, seed, mode="split", workers=1, train_set=None, num_classes=None):
    """engine.py:829-870."""
    if num_classes is None:
        num_classes = int(np.max(labels)) + 1 if len(labels) else 1
    trainer = Trainer(graph, pm, cache, labels)
    params = init_params(model_kind, trainer.graph_feat_dim(), hidden, num_classes, num_layers, seed=seed)
    records = [trainer.run_epoch(mode, params, seed=seed, epoch=e, fanouts=fanouts, batch_size=batch_size,
                                 lr=lr, workers=workers, train_set=train_set) for e in range(epochs)]
    return records, params


# ---- CUDA-graph captured step ------------------------------------------------------

class StaticSample:
    """Fixed-capacity device buffers holding one sample (CUDA-graph inputs).

    Layer l's vertices live at the capacity offset voff[l]; the actual sizes
    go to a small device array the kernels read, so one captured graph serves
    every sample that fits the capacities. All inputs are views of ONE int32
    buffer [sizes (int64) | V | esrc | edst], so a sample crosses PCIe as one
    contiguous prefix copy."""

    def __init__(self, cap_nV, cap_nE, device):
        self.cap_nV = [int(x) for x in cap_nV]
        self.cap_nE = [int(x) for x in cap_nE]
        self.L = len(self.cap_nE)
        self.voff = np.r_[0, np.cumsum(self.cap_nV)].astype(np.int64)
        self.eoff = np.r_[0, np.cumsum(self.cap_nE)].astype(np.int64)
        VC, EC = int(self.voff[-1]), max(int(self.eoff[-1]), 1)
        S = 2 * (2 * self.L + 1)
        self.o_V, self.o_es, self.o_ed = S, S + VC, S + VC + EC
        self.words = S + VC + 2 * EC
        dev = torch.device(device)
        self.buf = torch.zeros(self.words, dtype=torch.int32, device=dev)
        self.sizes = self.buf[:S].view(torch.int64)
        self.V = self.buf[self.o_V:self.o_V + VC]
        self.es = self.buf[self.o_es:self.o_es + EC]
        self.ed = self.buf[self.o_ed:self.o_ed + EC]
        self.hbuf = None
        self.bytes_h2d = 0

    def fits(self, sample):
        nV, nE = sample.sizes()
        return all(a <= b for a, b in zip(nV, self.cap_nV)) and all(a <= b for a, b in zip(nE, self.cap_nE))

    def pack(self, sample, out=None):
        """Write `sample` in this layout into a host int32 array; returns the
        number of words used (the prefix that has to cross PCIe)."""
        if not self.fits(sample):
            raise ValueError("sample exceeds the captured capacities")
        if not sample.is_dst_grouped():
            raise ValueError("captured steps need destination-grouped samples")
        nV, nE = sample.sizes()
        used = self.o_ed + int(self.eoff[self.L - 1] + nE[self.L - 1])
        if out is None:
            out = np.zeros(used, dtype=np.int32)
        out[:self.o_V].view(np.int64)[:] = list(nV) + list(nE)
        for l, v in enumerate(sample.layer_vertices):
            o = self.o_V + self.voff[l]
            out[o:o + nV[l]] = v
        for l, (a, b) in enumerate(sample.layer_edges):
            o = self.eoff[l]
            out[self.o_es + o:self.o_es + o + nE[l]] = a
            out[self.o_ed + o:self.o_ed + o + nE[l]] = b
        return used

    def load(self, sample):
        """Stage the sample into pinned memory and copy it to the device
        buffer (async, on the current stream). Two pinned staging slots, each
        reused only after its previous H2D copy has completed (the copy is
        asynchronous: packing the next sample into a slot whose copy is still
        queued behind a running step would corrupt that step's input)."""
        if self.hbuf is None:
            self.hbuf = [torch.zeros(self.words, dtype=torch.int32, pin_memory=True) for _ in range(2)]
            self.hev = [None, None]
            self.slot = 0
        k = self.slot
        self.slot ^= 1
        if self.hev[k] is not None:
            self.hev[k].synchronize()
        hb = self.hbuf[k]
        used = self.pack(sample, hb.numpy())
        self.buf[:used].copy_(hb[:used], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self.hev[k] = ev
        self.bytes_h2d = 4 * used
        return self.bytes_h2d


class PinnedSample:
    """One sample packed into pinned host memory, ready for the pipelined H2D
    (CapturedStep.run_pipelined). This is the form a host sampler hands to the
    trainer. compact=True (the default) sends the StaticSample prefix up to
    the last source position (header, V, es) plus one run start per
    destination instead of the per-edge destination lists (~40 % fewer bytes
    across PCIe; sg_pipe_stage_compact rebuilds ed on the copy stream, off the
    step's critical path). compact=False: the full layout in one buffer."""

    def __init__(self, sample, static, compact=True):
        host = np.zeros(static.words, dtype=np.int32)
        used = static.pack(sample, host)
        self.num_targets = len(sample.targets)
        self.full_bytes = 4 * used
        # the compact form rebuilds each layer's destination list from run
        # starts, which holds only when destinations are in ascending order
        # (a dst-grouped sample may list its groups in any order)
        self.compact = bool(compact) and all(
            len(b) < 2 or bool(np.all(np.diff(np.asarray(b)) >= 0)) for _, b in sample.layer_edges)
        if not self.compact:
            self.buf = pinned_from(host[:used].copy())
            self.h2d_bytes = 4 * used
            return
        nV, nE = sample.sizes()
        L = static.L
        prefix = static.o_es + int(static.eoff[L - 1] + nE[L - 1])
        starts = []
        for l, (_, b) in enumerate(sample.layer_edges):
            cnt = np.bincount(np.asarray(b, dtype=np.int64), minlength=nV[l + 1])
            st = np.zeros(nV[l + 1], dtype=np.int32)
            np.cumsum(cnt[:-1], out=st[1:])
            starts.append(st)
        st = np.concatenate(starts) if starts else np.zeros(0, np.int32)
        self.prefix_words = prefix
        self.buf = pinned_from(np.concatenate([host[:prefix], st]))
        self.starts_off = 4 * prefix
        self.starts_bytes = 4 * len(st)
        self.h2d_bytes = 4 * prefix + self.starts_bytes


def capacities_for(samples, slack=1.0):
    """Per-layer capacities covering `samples` (optionally with slack)."""
    L = samples[0].num_layers
    nV = [max(s.sizes()[0][l] for s in samples) for l in range(L + 1)]
    nE = [max(s.sizes()[1][l] for s in samples) for l in range(L)]
    return [int(np.ceil(x * slack)) for x in nV], [int(np.ceil(x * slack)) for x in nE]


class CapturedStep:
    """The whole split-parallel training step on ONE GPU captured once as a
    CUDA graph: split -> layer-0 rows (+ cache-miss staging) -> forward ->
    loss -> backward -> gradient reduction -> SGD, replayed per sample with
    only the sample's H2D copy in front. Kernels read every size from device
    memory. g = pm.num_devices parts: g = 1 is the single-GPU split; g > 1
    runs all g parts on this GPU (the reference's simulated devices, its
    exchange rounds as copy kernels) and sums their gradients in device
    order before the SGD step."""

    def __init__(self, dparams, pm, cache, feats, labels_dev, cap_nV, cap_nE, lr_scale,
                 device="cuda", record_events=False, lr=None):
        self.p = dparams
        self.pm, self.cache, self.f, self.labels = pm, cache, feats, labels_dev
        self.dev = torch.device(device)
        self.inp = StaticSample(cap_nV, cap_nE, self.dev)
        self._init_lr(lr_scale, lr)
        self.record_events = record_events
        self.graph = None

    def _init_lr(self, lr_scale, lr):
        """The SGD step inside the graph is p -= lr / num_targets * g with
        num_targets read on the device from each replayed sample's sizes
        (allreduce_and_step divides by that sample's target count). `lr`
        given, or derived at capture as lr_scale x the warm-up sample's
        target count (the captured batch)."""
        self.scale = float(lr_scale)
        self.lr = None if lr is None else float(lr)

    def _num_targets_dev(self):
        return self.inp.sizes[self.inp.L:self.inp.L + 1]

    def _fix_lr(self, warm_sample):
        if self.lr is None:
            self.lr = self.scale * len(warm_sample.targets)

    def _body(self):
        inp = self.inp
        ev = []
        if self.record_events and self.record_events != "agg":
            for _ in range(2):
                try:
                    ev.append(torch.cuda.Event(enable_timing=True, external=True))
                except TypeError:
                    ev.append(torch.cuda.Event(enable_timing=True))
            ev[0].record()
        ds = self._split(inp)
        if ev:
            ev[1].record()
        return self._after_split(ds, ev)

    def _split(self, inp):
        return DeviceSplit(inp.V, inp.es, inp.ed, inp.cap_nV, inp.cap_nE, self.pm, self.cache, True, self.dev,
                           sizes=inp.sizes)

    def _after_split(self, ds, ev=()):
        step = SplitStep(self.p, ds, self.f, self.labels, exact=False, record_events=self.record_events)
        if ev:
            step.events["ph:split:s"] = [ev[0]]
            step.events["ph:split:e"] = [ev[1]]
        g = self.pm.num_devices
        if g == 1:
            step.sgd = (self.p.flat, self.lr, self._num_targets_dev())  # one device: SGD rides on the reduction
        step.run()
        gbuf = step.grads[0]
        if g > 1:
            # g parts on this GPU (the reference's simulated devices): device-order
            # sum of the per-part gradients (+ loss slot) and the SGD step
            if getattr(self, "_gsum", None) is None:
                self._gsum = torch.empty(self.p.n + 1, dtype=torch.float32, device=self.dev)
            ptrs = np.asarray([step.grads[d].data_ptr() for d in range(g)], dtype=np.int64)
            _lib.call("sg_sum_sgd_nt", _lib.ptr(self.p.flat), _lib.ptr(self._gsum), _lib.ptr(ptrs), g, self.p.n,
                      self.p.n + 1, float(self.lr), self._num_targets_dev().data_ptr(), _lib.stream_ptr())
            gbuf = self._gsum
        self.ds, self.step = ds, step
        return gbuf

    def capture(self, warm_sample):
        """Eager warm-up on the static buffers, then capture. The warm-up
        applies real SGD updates (it is a training step); callers that need
        untouched parameters restore them afterwards."""
        self._fix_lr(warm_sample)
        self.inp.load(warm_sample)
        self.warm_out = self._body()  # the eager warm-up step's gradients (+ loss slot)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with _capturing(self.graph):
            self.out = self._body()
        torch.cuda.synchronize()
        return self

    def replay(self):
        self.graph.replay()
        return self.out

    def run(self, sample):
        self.inp.load(sample)
        return self.replay()

    def loss_sum(self):
        return self.out[self.p.n]

    def prepare_pinned(self, samples, compact=True):
        """Pack samples into PinnedSamples and DMA each buffer once (untimed):
        the first transfer from a freshly pinned buffer pays a one-time
        mapping cost that a sampler's reused pinned ring never sees again."""
        pinned = [PinnedSample(smp, self.inp, compact) for smp in samples]
        scratch = torch.empty(self.inp.words, dtype=torch.int32, device=self.dev)
        for ps in pinned:
            scratch[:ps.buf.numel()].copy_(ps.buf, non_blocking=True)
        torch.cuda.synchronize(self.dev)
        if _pipe_direct() and self._twin_ok:
            self._twin()  # captured here, outside any timed loop
        return pinned

    _twin_ok = True  # RankCapturedStep: one graph (its exchange rounds share the transport's buffers)

    def _twin(self):
        """Two staging slots for run_pipelined, each with its own input buffer
        and its step captured as TWO graphs: the split (which reads only the
        sample) and the rest. Each sample's H2D lands directly in its slot's
        input, and its split runs on the copy stream right after it, while the
        previous step is still computing; the main stream then runs only the
        rest (no device-to-device copy, and the split off the critical path).
        Capturing runs no kernels, so the parameters are untouched; the state of
        the single-graph capture (ds, step, the per-phase events) is restored
        afterwards."""
        tw = getattr(self, "_tw", None)
        if tw is None:
            keep = (self.inp, self.graph, self.out, getattr(self, "ds", None), getattr(self, "step", None))
            tw = []
            for slot in range(2):
                inp = keep[0] if slot == 0 else StaticSample(keep[0].cap_nV, keep[0].cap_nE, self.dev)
                if slot:
                    inp.buf.copy_(keep[0].buf)
                self.inp = inp
                gs, gm = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
                with _capturing(gs):
                    ds = self._split(inp)
                with _capturing(gm):
                    out = self._after_split(ds)
                torch.cuda.synchronize()
                tw.append((inp, gs, gm, out, ds))
            self._tw = tw
            self.inp, self.graph, self.out, self.ds, self.step = keep
        return tw

    def run_pipelined(self, pinned):
        """Train on a sequence of PinnedSamples end to end: per step an async
        H2D of the sample (native copy stream, double-buffered device
        staging, sg_pipe_stage), an on-device copy into the graph's input
        buffer, the graph replay and a D2H read of the step's loss sum. Step
        i+1's H2D overlaps step i's compute; the host reads step i's loss
        after step i+1 is queued. Returns (mean loss per step, H2D bytes,
        D2H bytes)."""
        lib = _lib.load()
        if getattr(self, "_pipe", None) is None:
            inp = self.inp
            h = lib.sg_pipe_create2((4 * inp.words + 15) // 16 * 16, 4 * int(sum(inp.cap_nV[1:])) + 16)
            if not h:
                _lib.check(2, "sg_pipe_create")
            self._pipe = h
            self._pipe_eoff = np.ascontiguousarray(inp.eoff[:inp.L], dtype=np.int64)
        h = self._pipe
        st = _lib.stream_ptr()
        dst = _lib.ptr(self.inp.buf)
        loss_ptr = self.out.data_ptr() + 4 * self.p.n
        out = ctypes.c_float()
        losses, h2d, d2h = [], 0, 0
        pending = None
        pc = time.perf_counter
        t_stage = t_replay = t_wait = 0.0
        direct = _pipe_direct() and self._twin_ok
        if direct:
            tw = self._twin()
            copy_st = torch.cuda.ExternalStream(lib.sg_pipe_copy_stream(h), device=self.dev)
            split_done = [torch.cuda.Event(), torch.cuda.Event()]
            main_st = torch.cuda.current_stream()
        for i, ps in enumerate(pinned):
            b = i & 1
            t0 = pc()
            if direct:
                inp_b, gsplit, gmain, out_b, _ = tw[b]
                base = ps.buf.data_ptr()
                if ps.compact:
                    _lib.check(lib.sg_pipe_stage_direct(h, b, base, ps.starts_off, base + ps.starts_off,
                                                        ps.starts_bytes, self.inp.L, self._pipe_eoff.ctypes.data,
                                                        self.inp.o_ed, _lib.ptr(inp_b.buf), st),
                               "sg_pipe_stage_direct")
                else:
                    _lib.check(lib.sg_pipe_stage_direct(h, b, base, ps.h2d_bytes, None, 0, self.inp.L,
                                                        self._pipe_eoff.ctypes.data, self.inp.o_ed,
                                                        _lib.ptr(inp_b.buf), st), "sg_pipe_stage_direct")
                with torch.cuda.stream(copy_st):  # the split, behind the sample's H2D on the copy stream
                    gsplit.replay()
                    split_done[b].record(copy_st)
                main_st.wait_event(split_done[b])
                t1 = pc()
                gmain.replay()
                t2 = pc()
                _lib.check(lib.sg_pipe_release(h, b, st), "sg_pipe_release")
                _lib.check(lib.sg_pipe_finish(h, b, out_b.data_ptr() + 4 * self.p.n, st), "sg_pipe_finish")
                h2d += ps.h2d_bytes
                d2h += 4
                t3 = pc()
                if pending is not None:
                    _lib.check(lib.sg_pipe_wait(h, pending[0], ctypes.byref(out)), "sg_pipe_wait")
                    losses.append(out.value / pending[1])
                t4 = pc()
                t_stage += t3 - t2 + t1 - t0
                t_replay += t2 - t1
                t_wait += t4 - t3
                pending = (b, ps.num_targets)
                continue
            if ps.compact:
                base = ps.buf.data_ptr()
                _lib.check(lib.sg_pipe_stage_compact(h, b, base, ps.starts_off, base + ps.starts_off, ps.starts_bytes,
                                                     self.inp.L, self._pipe_eoff.ctypes.data, self.inp.o_ed,
                                                     ps.full_bytes, dst, st), "sg_pipe_stage_compact")
            else:
                _lib.check(lib.sg_pipe_stage(h, b, ps.buf.data_ptr(), ps.h2d_bytes, dst, st), "sg_pipe_stage")
            t1 = pc()
            self.graph.replay()
            t2 = pc()
            _lib.check(lib.sg_pipe_finish(h, b, loss_ptr, st), "sg_pipe_finish")
            h2d += ps.h2d_bytes
            d2h += 4
            t3 = pc()
            if pending is not None:
                _lib.check(lib.sg_pipe_wait(h, pending[0], ctypes.byref(out)), "sg_pipe_wait")
                losses.append(out.value / pending[1])
            t4 = pc()
            t_stage += t3 - t2 + t1 - t0
            t_replay += t2 - t1
            t_wait += t4 - t3
            pending = (b, ps.num_targets)
        n = max(len(pinned), 1)
        self.pipe_stats = {"host_issue_us": 1e6 * t_stage / n, "host_replay_us": 1e6 * t_replay / n,
                           "host_wait_us": 1e6 * t_wait / n}
        if pending is not None:
            _lib.check(lib.sg_pipe_wait(h, pending[0], ctypes.byref(out)), "sg_pipe_wait")
            losses.append(out.value / pending[1])
        return losses, h2d, d2h

    def __del__(self):
        h = getattr(self, "_pipe", None)
        if h:
            try:
                _lib.load().sg_pipe_destroy(h)
            except Exception:
                pass
            self._pipe = None


# ---- reference-API captured step ----------------------------------------------------

class _ApiGraphStep(CapturedStep):
    """The reference-API executor's captured step: split -> layer-0 rows ->
    forward -> loss -> backward -> per-device gradient reduction, no SGD
    (allreduce_and_step applies it). Cached per (model shape, partition,
    cache, features, labels, capacity bucket); the sample arrives as a
    device-to-device copy of split_minibatch's packed buffer, the parameters as
    an H2D copy of the host ModelParams."""

    def _body(self):
        inp = self.inp
        ds = DeviceSplit(inp.V, inp.es, inp.ed, inp.cap_nV, inp.cap_nE, self.pm, self.cache, True, self.dev,
                         sizes=inp.sizes)
        step = SplitStep(self.p, ds, self.f, self.labels, exact=False)
        step.run()
        self.ds, self.step = ds, step
        return [step.grads[d] for d in range(self.pm.num_devices)]

    def load_packed(self, packed):
        buf, used, _ = packed
        self.inp.buf[:used].copy_(buf[:used])

    def capture_packed(self, packed):
        self.load_packed(packed)
        with _pdl_for(self.p.kind):
            self._body()  # eager warm-up (no SGD: parameters untouched)
            torch.cuda.synchronize()
            self.graph = torch.cuda.CUDAGraph()
            with _capturing(self.graph):
                self.out = self._body()
        torch.cuda.synchronize()
        return self


_API_GRAPHS = {}
_API_GRAPHS_MAX = 8


def _api_graph(params, ds, feats, labels):
    """Cached _ApiGraphStep for this model shape / capacity bucket (LRU of 8;
    the entries hold the partition, cache, feature store and labels they were
    captured with, so their ids stay unique while cached)."""
    geo = ds.packed[2]
    # parameter names follow from (kind, layer count); shapes from the arrays
    key = (params.kind, len(params.layers), tuple(np.shape(v) for v in _param_arrays(params)),
           float(params.leaky_slope), id(ds.pm), id(ds.cache), id(feats), labels.data_ptr(), tuple(geo.cap_nV),
           tuple(geo.cap_nE), ds.device)
    gs = _API_GRAPHS.pop(key, None)
    if gs is None:
        dp = DeviceParams.from_host(params, ds.device)
        gs = _ApiGraphStep(dp, ds.pm, ds.cache, feats, labels, geo.cap_nV, geo.cap_nE, 1.0, device=ds.device, lr=1.0)
        gs.capture_packed(ds.packed)
        while len(_API_GRAPHS) >= _API_GRAPHS_MAX:
            _API_GRAPHS.pop(next(iter(_API_GRAPHS)))
    _API_GRAPHS[key] = gs
    return gs


# ---- one process per GPU ------------------------------------------------------------

class SampledCapturedStep(CapturedStep):
    """The single-GPU step with the k-hop sampler inside the same CUDA graph:
    targets + seed (one small H2D) -> GpuSampler -> split -> forward/backward
    -> reduction + SGD. The sample never exists on the host; the captured
    capacities must cover every sample (the sampler flags an overflow in
    `sampler.err`, checked by `check()`)."""

    def __init__(self, sampler, fanouts, batch, dparams, pm, cache, feats, labels_dev, cap_nV, cap_nE,
                 lr_scale, device="cuda", record_events=False, lr=None):
        super().__init__(dparams, pm, cache, feats, labels_dev, cap_nV, cap_nE, lr_scale, device, record_events,
                         lr=lr)
        self.sampler = sampler
        self.fanouts = [int(f) for f in fanouts]
        self.batch = int(batch)
        self.tgt = torch.zeros(self.batch + 1, dtype=torch.int64, device=self.dev)  # targets | seed
        self.htgt = [torch.zeros(self.batch + 1, dtype=torch.int64, pin_memory=True) for _ in range(2)]
        self.tev = [None, None]
        self.tslot = 0

    def _body(self):
        inp = self.inp
        self.sampler.sample_into(self.tgt[:self.batch], self.fanouts, 0, inp.V, inp.es, inp.ed, inp.sizes,
                                 inp.voff, inp.eoff, seed_dev=self.tgt[self.batch:])
        return super()._body()

    def load_targets(self, targets, seed):
        t = np.asarray(targets, dtype=np.int64)
        if len(t) != self.batch:
            raise ValueError(f"the captured step samples exactly {self.batch} targets")
        k = self.tslot  # two pinned slots, each reused after its copy completed (see StaticSample.load)
        self.tslot ^= 1
        if self.tev[k] is not None:
            self.tev[k].synchronize()
        h = self.htgt[k].numpy()
        h[:self.batch] = t
        h[self.batch] = np.int64(np.uint64(int(seed) & (2**64 - 1)).view(np.int64))
        self.tgt.copy_(self.htgt[k], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self.tev[k] = ev

    def capture_targets(self, targets, seed):
        if self.lr is None:
            self.lr = self.scale * self.batch
        self.load_targets(targets, seed)
        self._body()
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with _capturing(self.graph):
            self.out = self._body()
        torch.cuda.synchronize()
        return self

    def run_targets(self, targets, seed):
        self.load_targets(targets, seed)
        return self.replay()

    def check(self):
        if int(self.sampler.err.item()):
            raise RuntimeError("GPU sampler: a sample exceeded the captured capacities")

    def pin_targets(self, plan):
        """Pack [(targets, seed), ...] into pinned host buffers (untimed)."""
        out = []
        for t, sd in plan:
            h = torch.zeros(self.batch + 1, dtype=torch.int64, pin_memory=True)
            a = h.numpy()
            a[:self.batch] = np.asarray(t, dtype=np.int64)
            a[self.batch] = np.int64(np.uint64(int(sd) & (2**64 - 1)).view(np.int64))
            out.append(h)
        return out

    def run_pipelined_targets(self, pinned):
        """End to end from host targets: per step an async H2D of the targets
        and seed (8 B x (batch + 1)), the graph replay (sample + split + step)
        and an async D2H of the step's loss sum; one synchronisation at the
        end. Returns (loss sums, H2D bytes, D2H bytes)."""
        n = self.p.n
        outs = torch.zeros(len(pinned), dtype=torch.float32, pin_memory=True)
        for i, h in enumerate(pinned):
            self.tgt.copy_(h, non_blocking=True)
            self.graph.replay()
            outs[i:i + 1].copy_(self.out[n:n + 1], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return outs.tolist(), sum(8 * h.numel() for h in pinned), 4 * len(pinned)


class RankSplitTrainer:
    """Split-parallel training where this process is device `rank` of a
    `world`-GPU split (torchrun, one process per GPU). Every rank runs the
    splitter on the replicated sample, computes only its own part, exchanges
    partial aggregates with its peers over the transport (NCCL all-to-all-v)
    and all-reduces the flat gradient before the SGD step."""

    def __init__(self, params, pm, cache, feats, labels, rank, world, transport, device="cuda"):
        self.pm, self.cache = pm, cache
        self.rank, self.world = int(rank), int(world)
        self.dev = torch.device(device)
        host = params if isinstance(params, ModelParams) else ModelParams.from_reference(params)
        self.dp = params if isinstance(params, DeviceParams) else DeviceParams.from_host(host, self.dev)
        self.feats = feats
        self.labels = labels if isinstance(labels, torch.Tensor) else _labels_dev(labels, self.dev)
        self.transport = transport

    def step(self, sample, lr, record_events=False, dsplit=None):
        ds = dsplit if dsplit is not None else DeviceSplit.from_sample(sample, self.pm, self.cache, self.dev)
        peer = hasattr(self.transport, "all_reduce_sgd")
        st = SplitStep(self.dp, ds, self.feats, self.labels, devices=[self.rank],
                       transport=self.transport, exact=not peer, record_events=record_events)
        st.run()
        gbuf = st.grads[self.rank]
        scale = float(lr) / len(sample.targets)
        if peer:  # all-reduce + SGD over peer memory (no host round trip)
            out = torch.empty_like(gbuf)
            self.transport.all_reduce_sgd(gbuf, self.dp.n, self.dp.flat, scale, grads_out=out)
            gbuf = out
        else:
            self.transport.all_reduce(gbuf)          # sum over ranks (includes the loss slot)
            ptrs = np.asarray([gbuf.data_ptr()], dtype=np.int64)
            _lib.call("sg_sum_sgd", _lib.ptr(self.dp.flat), None, _lib.ptr(ptrs), 1, self.dp.n,
                      scale, _lib.stream_ptr())
        self.last = st
        return gbuf


class RankCapturedStep(CapturedStep):
    """This rank's part of the multi-GPU split step (rank = split part) as ONE
    CUDA graph: replicated split -> rank-local forward/backward whose exchange
    rounds run over the PeerTransport's mapped buffers -> peer all-reduce +
    SGD. Sizes are read on the device; nothing returns to the host."""

    _twin_ok = False

    def __init__(self, dparams, pm, cache, feats, labels_dev, cap_nV, cap_nE, lr_scale, rank, transport,
                 device="cuda", record_events=False, lr=None):
        if not hasattr(transport, "all_reduce_sgd"):
            raise ValueError("RankCapturedStep needs a PeerTransport (no host-side sizes inside a graph)")
        self.p = dparams
        self.pm, self.cache, self.f, self.labels = pm, cache, feats, labels_dev
        self.dev = torch.device(device)
        self.inp = StaticSample(cap_nV, cap_nE, self.dev)
        self._init_lr(lr_scale, lr)
        self.record_events = record_events
        self.graph = None
        self.rank = int(rank)
        self.transport = transport
        self.gsum = None

    def _body(self):
        inp = self.inp
        ds = DeviceSplit(inp.V, inp.es, inp.ed, inp.cap_nV, inp.cap_nE, self.pm, self.cache, True,
                         self.dev, sizes=inp.sizes)
        step = SplitStep(self.p, ds, self.f, self.labels, devices=[self.rank], transport=self.transport,
                         exact=False, record_events=self.record_events)
        step.run()
        gbuf = step.grads[self.rank]
        if self.gsum is None:
            self.gsum = torch.empty_like(gbuf)
        self.transport.all_reduce_sgd(gbuf, self.p.n, self.p.flat, None, grads_out=self.gsum, lr=self.lr,
                                      num_targets=self._num_targets_dev())
        self.ds, self.step = ds, step
        return self.gsum
