"""Online splitting of a mini-batch sample on the GPU.

`split_minibatch(sample, pm, cache)` keeps the reference signature and return
types (scheduler.py:164-254: list[LocalSplit], ShufflePlan) but the work is
done by the sm_100a splitter (sg_split_run): the returned objects are host
VIEWS of a device-resident DeviceSplit, which the executor consumes directly.
No part of this module computes a split on the CPU.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from paper_2303_13775_b200 import _lib
from paper_2303_13775_b200.partition import CacheState, PartitionMap
from paper_2303_13775_b200.sampling import MiniBatchSample, as_sample


@dataclass
class LocalSplit:
    """One device's non-overlapping share of a sample (scheduler.py:24-66)."""

    device: int
    num_layers: int
    owned_gids: list
    owned_pos: list
    ref_gids: list
    ref_owner: list
    edges_src: list
    edges_dst: list
    self_rows: list
    load_gids: np.ndarray

    def num_owned(self, l):
        return len(self.owned_gids[l])

    def num_ref(self, l):
        return len(self.ref_gids[l])

    def edges(self, l):
        return self.edges_src[l - 1], self.edges_dst[l - 1]

    def num_edges(self, l):
        return len(self.edges_src[l - 1])

    @property
    def total_edges(self):
        return int(sum(len(e) for e in self.edges_src))

    def self_index(self, l):
        return self.self_rows[l - 1]

    def edge_gids(self, l):
        src, dst = self.edges(l)
        n_own = self.num_owned(l)
        own = dst < n_own
        dst_gid = np.empty(len(dst), dtype=np.int64)
        dst_gid[own] = self.owned_gids[l][dst[own]]
        dst_gid[~own] = self.ref_gids[l][dst[~own] - n_own]
        return self.owned_gids[l - 1][src], dst_gid


@dataclass
class PlanEntry:
    gids: np.ndarray
    holder_idx: np.ndarray
    owner_idx: np.ndarray

    @property
    def count(self):
        return len(self.gids)


@dataclass
class ShufflePlan:
    """Exchange descriptors (scheduler.py:82-122)."""

    num_layers: int
    num_devices: int
    entries: dict = field(default_factory=dict)
    device_split: object = field(default=None, repr=False, compare=False)

    def entry(self, l, holder, owner):
        return self.entries.get((l, holder, owner))

    def push_to_owner(self, l, src_dev, dst_dev):
        e = self.entry(l, src_dev, dst_dev)
        return e.gids if e is not None else np.empty(0, dtype=np.int64)

    def push_from_owner(self, l, src_dev, dst_dev):
        return self.push_to_owner(l, dst_dev, src_dev)

    def holders_of(self, l, owner):
        return [s for s in range(self.num_devices) if s != owner and (l, s, owner) in self.entries]

    def owners_for(self, l, holder):
        return [o for o in range(self.num_devices) if o != holder and (l, holder, o) in self.entries]

    def pair_count(self, l):
        return sum(e.count for (ll, _, _), e in self.entries.items() if ll == l)


class SplitList(list):
    """list[LocalSplit] that also carries the device-resident split."""

    device_split = None


def _carr(a):
    return np.ctypeslib.as_array(a)


class HostMeta:
    """numpy view of the SgMeta counts (one D2H per iteration)."""

    def __init__(self, raw: _lib.SgMeta):
        self.raw = raw
        for name, _ in _lib.SgMeta._fields_:
            v = getattr(raw, name)
            setattr(self, name, _carr(v).copy() if not isinstance(v, int) else v)


class DeviceSplit:
    """The split of all g devices, resident in one GPU workspace.

    Built by sg_split_run from the replicated sample. Index spaces (all
    per layer): owned rows grouped by device (own_off), reference rows
    grouped by holder == pair slots (ref_off / pair_off, holder-major),
    receive slots (recv_off, owner-major)."""

    def __init__(self, V, esrc, edst, nV, nE, pm: PartitionMap, cache: CacheState | None,
                 dst_grouped: bool, device=None, host_V=None, sizes=None):
        """nV / nE are the CAPACITIES the layout is built for; `sizes` (device
        int64 [nV_0..nV_L, nE_1..nE_L]) gives the actual sizes (default: the
        capacities). V / esrc / edst hold layer l at the capacity offsets."""
        lib = _lib.load()
        self.device = torch.device(device or "cuda")
        self.pm = pm
        self.cache = cache
        self.g = pm.num_devices
        self.L = len(nE)
        self.nV = [int(x) for x in nV]
        self.nE = [int(x) for x in nE]
        self.dst_grouped = bool(dst_grouped)
        lay = _lib.SgSplitLayout()
        nVa = (C.c_int64 * (self.L + 1))(*self.nV)
        nEa = (C.c_int64 * max(self.L, 1))(*(self.nE or [0]))
        _lib.check(lib.sg_split_layout(self.L, self.g, nVa, nEa, len(pm.assignment), C.byref(lay)),
                   "split_layout")
        self.lay = lay
        self.ws = torch.empty(int(lay.total_bytes), dtype=torch.uint8, device=self.device)
        self.V, self.esrc, self.edst = V, esrc, edst
        self.host_V = host_V
        bits = cache.device_bits(len(pm.assignment), self.device) if cache is not None else None
        n = len(pm.assignment)
        if cache is not None and getattr(cache, "_all", None) is None:
            cache._all = cache.covers_all(n)
        flags = (1 if self.dst_grouped else 0) | (2 if cache is not None and cache._all else 0)
        self.all_cached = bool(flags & 2)
        self.sizes = sizes
        _lib.check(lib.sg_split_run(_lib.ptr(self.ws), C.byref(lay), _lib.ptr(V), _lib.ptr(esrc),
                                    _lib.ptr(edst), _lib.ptr(sizes), _lib.ptr(pm.device_u8(self.device)),
                                    _lib.ptr(bits), flags, _lib.stream_ptr()),
                   "split_run")
        self._meta = None
        self._views = None

    # -- construction from a host sample ------------------------------------
    @classmethod
    def from_sample(cls, sample, pm, cache=None, device=None):
        sample = as_sample(sample)
        nV, nE = sample.sizes()
        V, es, ed = sample.packed()
        dev = torch.device(device or "cuda")
        Vt = torch.from_numpy(V).pin_memory().to(dev, non_blocking=True)
        st = torch.from_numpy(es).pin_memory().to(dev, non_blocking=True)
        dt = torch.from_numpy(ed).pin_memory().to(dev, non_blocking=True)
        return cls(Vt, st, dt, nV, nE, pm, cache, sample.is_dst_grouped(), dev, host_V=V)

    # -- device views -------------------------------------------------------
    def i32(self, off, count, start=0):
        b = int(off) + 4 * int(start)
        return self.ws[b:b + 4 * int(count)].view(torch.int32)

    def meta_dev(self):
        return self.ws[int(self.lay.o_meta):int(self.lay.o_meta) + C.sizeof(_lib.SgMeta)]

    def host_meta(self) -> HostMeta:
        """D2H of the count descriptor (synchronises the current stream)."""
        if self._meta is None:
            raw = self.meta_dev().cpu().numpy().tobytes()
            m = _lib.SgMeta.from_buffer_copy(raw)
            if m.err & 1:
                raise ValueError("sample vertex missing from partition map")
            self._meta = HostMeta(m)
        return self._meta

    @property
    def voff(self):
        return [int(x) for x in self.lay.voff]

    @property
    def eoff(self):
        return [int(x) for x in self.lay.eoff]

    def pair_bound(self, l):
        return int(self.lay.pbase[l + 1] - self.lay.pbase[l])

    def pair_count(self, l):
        return int(self.host_meta().npairs[l])

    # -- host views in the reference's types ----------------------------------
    def to_reference_types(self):
        m = self.host_meta()
        ws = self.ws.cpu().numpy()
        lay = self.lay
        L, g = self.L, self.g

        def arr(off, n, start=0):
            b = int(off) + 4 * int(start)
            return ws[b:b + 4 * int(n)].view(np.int32).astype(np.int64)

        nVtot = int(lay.nVtot)
        V = self.host_V if self.host_V is not None else self.V.cpu().numpy()
        V = np.asarray(V, dtype=np.int64)
        vo, eo = self.voff, self.eoff
        Vl = [V[vo[l]:vo[l] + int(m.nV[l])] for l in range(L + 1)]
        grouped = arr(lay.o_grouped, nVtot + self.nV[0])
        rank = arr(lay.o_rank, nVtot + self.nV[0])
        lsrc = arr(lay.o_lsrc, lay.nEtot)
        ldst = arr(lay.o_ldst, lay.nEtot)
        selfrow = arr(lay.o_selfrow, nVtot)
        pairs = arr(lay.o_pairs, lay.nPtot)
        phidx = arr(lay.o_pair_hidx, lay.nPtot)
        asn = self.pm.assignment
        splits = SplitList()
        for d in range(g):
            owned_pos, owned_gids, ref_gids, ref_owner = [], [], [], []
            for l in range(L + 1):
                b = vo[l] + m.own_off[l][d]
                pos = grouped[b:b + m.n_own[l][d]]
                owned_pos.append(pos)
                owned_gids.append(Vl[l][pos])
                if l == 0 or g == 1:
                    ref_gids.append(np.empty(0, dtype=np.int64))
                    ref_owner.append(np.empty(0, dtype=np.int64))
                    continue
                pb = int(lay.pbase[l])
                sl = slice(pb + m.ref_off[l][d], pb + m.ref_off[l][d + 1])
                rp = np.empty(m.n_ref[l][d], dtype=np.int64)
                rp[phidx[sl]] = pairs[sl]
                rg = Vl[l][rp]
                ref_gids.append(rg)
                ref_owner.append(asn[rg])
            es, ed, sr = [], [], []
            for l in range(1, L + 1):
                b = eo[l - 1] + m.edge_off[l - 1][d]
                es.append(lsrc[b:b + m.n_edge[l - 1][d]])
                ed.append(ldst[b:b + m.n_edge[l - 1][d]])
                b2 = vo[l] + m.own_off[l][d]
                sr.append(selfrow[b2:b2 + m.n_own[l][d]])
            lb = nVtot + m.load_off[d]
            load = Vl[0][grouped[lb:lb + m.n_load[d]]]
            splits.append(LocalSplit(d, L, owned_gids, owned_pos, ref_gids, ref_owner, es, ed, sr,
                                     load))
        plan = ShufflePlan(L, g, device_split=self)
        for l in range(1, L + 1):
            pb = int(lay.pbase[l])
            for s in range(g):
                for o in range(g):
                    c = int(m.cnt[l][s][o])
                    if c == 0:
                        continue
                    sl = slice(pb + m.pair_off[l][s][o], pb + m.pair_off[l][s][o] + c)
                    p = pairs[sl]
                    plan.entries[(l, s, o)] = PlanEntry(Vl[l][p], phidx[sl], rank[vo[l] + p])
        splits.device_split = self
        return splits, plan


def split_minibatch(sample, pm: PartitionMap, cache: CacheState | None = None):
    """scheduler.py:164-254 on the GPU. Returns (list[LocalSplit], ShufflePlan)
    host views; both carry `.device_split` for the executor. Raises ValueError
    for a sampled vertex outside the partition map (scheduler.py:175-178)."""
    sample = as_sample(sample)
    n = len(pm.assignment)
    for v in sample.layer_vertices:
        v = np.asarray(v)
        if len(v) and (v.max() >= n or v.min() < 0):
            raise ValueError("sample vertex missing from partition map")
    ds = DeviceSplit.from_sample(sample, pm, cache)
    return ds.to_reference_types()


@dataclass
class TransferManifest:
    host_bytes_per_device: np.ndarray
    peer_feature_bytes: np.ndarray

    @property
    def host_bytes_total(self):
        return int(self.host_bytes_per_device.sum())


def transfer_manifest(splits, cache, feat_dim) -> TransferManifest:
    """Host-load bytes per device (scheduler.py:324-347, float64 accounting
    as in the reference); zero peer feature bytes by construction."""
    g = len(splits)
    host = np.array([len(s.load_gids) * feat_dim * 8 for s in splits], dtype=np.int64)
    loads = np.concatenate([s.load_gids for s in splits]) if splits else np.empty(0, np.int64)
    assert len(np.unique(loads)) == len(loads), "a feature vector loaded twice"
    if cache is not None and len(loads):
        cached = np.concatenate(cache.cached) if cache.cached else loads[:0]
        assert not np.intersect1d(loads, cached).size, "splits predate this cache"
    return TransferManifest(host, np.zeros((g, g), dtype=np.int64))


@dataclass
class SplitCostReport:
    """Communication-cost view of one sample under a vertex assignment
    (scheduler.py:126-147)."""

    num_devices: int
    per_layer_cost: list  # per layer 1..L: C[v^l] array over V^(l)
    cost_per_layer: list
    cost_total: int
    edges_per_device_per_layer: list
    edges_per_device: np.ndarray
    edges_local_per_layer: list
    edges_total_per_layer: list
    skew_per_layer: list
    edge_skew: float
    local_edge_fraction: float

    @property
    def edges_total(self) -> int:
        return int(sum(self.edges_total_per_layer))

    @property
    def edges_local(self) -> int:
        return int(sum(self.edges_local_per_layer))


def _skew(counts) -> float:
    """(max - min) / mean (scheduler.py:150-154)."""
    counts = np.asarray(counts)
    mean = counts.mean() if len(counts) else 0.0
    if mean == 0:
        return 0.0
    return float((counts.max() - counts.min()) / mean)


def split_cost(sample, assignment, num_devices: int | None = None, device=None) -> SplitCostReport:
    """scheduler.py:257-309 on the GPU (sg_split_cost): per-vertex shuffle cost
    C[v^l] = number of foreign devices holding a source of v's in-edges, edge
    skew and edge locality of the sample under `assignment`."""
    sample = as_sample(sample)
    if isinstance(assignment, PartitionMap):
        pm = assignment
        if num_devices is None:
            num_devices = pm.num_devices
    else:
        asn = np.asarray(assignment, dtype=np.int64)
        gg = int(num_devices if num_devices is not None else asn.max() + 1)
        pm = PartitionMap(asn, gg, float(gg))
    g = int(num_devices if num_devices is not None else pm.num_devices)
    if g > pm.num_devices:
        pm = PartitionMap(pm.assignment, g, float(g))
    dev = torch.device(device or "cuda")
    nV, nE = sample.sizes()
    L = len(nE)
    n = len(pm.assignment)
    for v in sample.layer_vertices:
        v = np.asarray(v)
        if len(v) and (v.max() >= n or v.min() < 0):
            raise ValueError("sample vertex missing from partition map")
    V, es, ed = sample.packed()
    return split_cost_packed(torch.from_numpy(V).to(dev), torch.from_numpy(es).to(dev),
                             torch.from_numpy(ed).to(dev), nV, nE, pm, g)


def split_cost_packed(Vt, st_, dt_, nV, nE, pm: PartitionMap, g: int) -> SplitCostReport:
    """split_cost on a sample already resident on the device (packed int32
    V / esrc / edst, as DeviceSplit holds it)."""
    dev = Vt.device
    L = len(nE)
    n = len(pm.assignment)
    nrows = max(sum(nV[1:]), 1)
    mask = torch.empty(nrows, dtype=torch.int32, device=dev)
    cost_rows = torch.empty(nrows, dtype=torch.int32, device=dev)
    counts = torch.empty(L * g, dtype=torch.int64, device=dev)
    local = torch.empty(L, dtype=torch.int64, device=dev)
    cost = torch.empty(L, dtype=torch.int64, device=dev)
    err = torch.empty(1, dtype=torch.int32, device=dev)
    nVa = np.asarray(nV, dtype=np.int64)
    nEa = np.asarray(nE, dtype=np.int64)
    _lib.call("sg_split_cost", _lib.ptr(Vt), _lib.ptr(st_), _lib.ptr(dt_), _lib.ptr(nVa), _lib.ptr(nEa), L,
              _lib.ptr(pm.device_u8(dev)), n, g, _lib.ptr(mask), _lib.ptr(cost_rows), _lib.ptr(counts),
              _lib.ptr(local), _lib.ptr(cost), _lib.ptr(err), _lib.stream_ptr())
    if int(err.item()):
        raise ValueError("sample vertex missing from partition map")
    cr = cost_rows.cpu().numpy().astype(np.int64)
    cnt = counts.cpu().numpy().reshape(L, g) if L else np.zeros((0, g), np.int64)
    loc = local.cpu().numpy()
    cpl = cost.cpu().numpy()
    per_layer_cost, off = [], 0
    for l in range(1, L + 1):
        per_layer_cost.append(cr[off:off + nV[l]].copy())
        off += nV[l]
    edges_pd_pl = [cnt[l].astype(np.int64) for l in range(L)]
    edges_per_device = np.sum(edges_pd_pl, axis=0) if edges_pd_pl else np.zeros(g, dtype=np.int64)
    total = int(sum(nE))
    return SplitCostReport(
        num_devices=g,
        per_layer_cost=per_layer_cost,
        cost_per_layer=[int(c) for c in cpl],
        cost_total=int(cpl.sum()),
        edges_per_device_per_layer=edges_pd_pl,
        edges_per_device=edges_per_device,
        edges_local_per_layer=[int(x) for x in loc],
        edges_total_per_layer=[int(x) for x in nE],
        skew_per_layer=[_skew(c) for c in edges_pd_pl],
        edge_skew=_skew(edges_per_device),
        local_edge_fraction=(int(loc.sum()) / total) if total else 1.0,
    )
