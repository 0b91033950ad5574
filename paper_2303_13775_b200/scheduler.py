"""Online splitting of a mini-batch sample on the GPU.

`split_minibatch(sample, pm, cache)` keeps the reference signature and return
types (scheduler.py:164-254: list[LocalSplit], ShufflePlan) but the work is
done by the sm_100a splitter (sg_split_run): the returned objects are host
VIEWS of a device-resident DeviceSplit, which the executor consumes directly.
No part of this module computes a split on the CPU.
"""

from __future__ import annotations

import ctypes as C
import os
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
        if self.device_split is not None:  # from the device counts, without building host views
            return self.device_split.pair_count(l)
        return sum(e.count for (ll, _, _), e in self.entries.items() if ll == l)


class SplitList(list):
    """list[LocalSplit] that also carries the device-resident split. From
    split_minibatch its LocalSplit host views are built lazily, on the first
    access to the list's contents."""

    device_split = None
    _fill_fn = None

    def _fill(self):
        f = self._fill_fn
        if f is not None:
            self._fill_fn = None
            f()

    def __getitem__(self, i):
        self._fill()
        return list.__getitem__(self, i)

    def __iter__(self):
        self._fill()
        return list.__iter__(self)

    def __len__(self):
        if self._fill_fn is not None and self.device_split is not None:
            return self.device_split.g
        return list.__len__(self)

    def __bool__(self):
        return len(self) > 0

    def __contains__(self, x):
        self._fill()
        return list.__contains__(self, x)

    def __reversed__(self):
        self._fill()
        return list.__reversed__(self)

    def __eq__(self, other):
        self._fill()
        return list.__eq__(self, other)

    def __repr__(self):
        self._fill()
        return list.__repr__(self)

    def index(self, *a):
        self._fill()
        return list.index(self, *a)

    def count(self, x):
        self._fill()
        return list.count(self, x)

    def copy(self):
        self._fill()
        return list(list.__iter__(self))


class _LazyEntries(dict):
    """ShufflePlan.entries built on first access (see SplitList)."""

    def __init__(self, fn):
        super().__init__()
        self._fn = fn

    def _fill(self):
        f = self._fn
        if f is not None:
            self._fn = None
            dict.update(self, f())

    for _m in ("__getitem__", "__iter__", "__len__", "__contains__", "__repr__", "__eq__", "keys", "values",
               "items", "get", "copy"):
        def _wrap(self, *a, _name=_m, **k):
            self._fill()
            return getattr(dict, _name)(self, *a, **k)
        locals()[_m] = _wrap
    del _m, _wrap


def pinned_from(a):
    """A page-locked copy of host array `a` allocated pinned from the start
    (torch.empty(..., pin_memory=True)): H2D from such buffers measured 48 GB/s
    on B200 boxes against 22-28 GB/s from Tensor.pin_memory() copies
    (tools/h2d_pinned_probe.py)."""
    a = np.ascontiguousarray(a)
    t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
    t.numpy()[...] = a
    return t


def _bucket(x):
    """Capacity bucket: x rounded up to 1/8 of its power of two (>= 64)."""
    x = int(x)
    if x <= 64:
        return 64
    q = 1 << (x.bit_length() - 4)
    return (x + q - 1) // q * q


class PackGeometry:
    """Offsets (int32 words) of the captured-step sample layout for given
    capacities (engine.StaticSample uses the same geometry)."""

    _cache = {}

    def __init__(self, cap_nV, cap_nE):
        self.cap_nV = [int(x) for x in cap_nV]
        self.cap_nE = [int(x) for x in cap_nE]
        self.L = len(self.cap_nE)
        self.voff = np.r_[0, np.cumsum(self.cap_nV)].astype(np.int64)
        self.eoff = np.r_[0, np.cumsum(self.cap_nE)].astype(np.int64)
        VC, EC = int(self.voff[-1]), max(int(self.eoff[-1]), 1)
        self.S = 2 * (2 * self.L + 1)
        self.EC = EC
        self._voff_l = [int(x) for x in self.voff]
        self._eoff_l = [int(x) for x in self.eoff]
        self._relgeo = None
        self.o_V, self.o_es, self.o_ed = self.S, self.S + VC, self.S + VC + EC
        self.words = self.S + VC + 2 * EC

    @classmethod
    def for_sizes(cls, nV, nE, scope=None):
        """The current geometry of `scope` if the sizes fit it, else a grown
        one (every capacity at least the bucket of 1.15 x the size): the
        geometry -- and so the executor's cached graph -- changes only when
        a larger sample than any before arrives."""
        cur = cls._cache.get(scope)
        if cur is not None and len(cur.cap_nV) == len(nV) and \
                all(a <= b for a, b in zip(nV, cur.cap_nV)) and all(a <= b for a, b in zip(nE, cur.cap_nE)):
            return cur
        grow = lambda x: _bucket(int(x * 1.15) + 1)  # noqa: E731
        if cur is not None and len(cur.cap_nV) == len(nV):
            cV = [max(c, grow(x)) for c, x in zip(cur.cap_nV, nV)]
            cE = [max(c, grow(x)) for c, x in zip(cur.cap_nE, nE)]
        else:
            cV, cE = [grow(x) for x in nV], [grow(x) for x in nE]
        geo = cls._cache[scope] = cls(cV, cE)
        return geo

    def pack(self, sample, out):
        """Write the sample into host int32 `out` (sg_pack_sample: native,
        multi-threaded); returns the words used."""
        nV, nE = sample.sizes()
        if any(a > b for a, b in zip(nV, self.cap_nV)) or any(a > b for a, b in zip(nE, self.cap_nE)):
            raise ValueError("sample exceeds the captured capacities")
        used = self.o_ed + int(self.eoff[self.L - 1] + nE[self.L - 1]) if self.L else self.o_es
        L = self.L
        arrs = [_i32_or_i64(v) for v in sample.layer_vertices] + \
               [_i32_or_i64(a) for a, _ in sample.layer_edges] + [_i32_or_i64(b) for _, b in sample.layer_edges]
        off = np.array([self.o_V + self.voff[l] for l in range(L + 1)] +
                       [self.o_es + self.eoff[l] for l in range(L)] +
                       [self.o_ed + self.eoff[l] for l in range(L)], dtype=np.int64)
        sizes = np.array(list(nV) + list(nE), dtype=np.int64)
        ptrs = np.array([a.ctypes.data for a in arrs], dtype=np.uint64)
        eb = np.array([a.itemsize for a in arrs], dtype=np.int32)
        vr = np.zeros(2, dtype=np.int64)
        _lib.call("sg_pack_sample", out.ctypes.data, L, sizes.ctypes.data, off.ctypes.data, ptrs.ctypes.data,
                  eb.ctypes.data, 4, vr.ctypes.data)
        self.last_vrange = (int(vr[0]), int(vr[1]))
        return used

    def relayout_from_stage(self, sample, pin, stage, buf, nE):
        """A native-sampler sample (PinnedArrays) already sent to the device
        staging buffer by _h2d_pinned: one kernel moves its segments to this
        layout's offsets in `buf`, deriving them from the sample's own sizes
        header on the device (sg_relayout_sample_hdr; the capacity geometry is
        a cached host array); in the compact form the destination lists are
        rebuilt from the run starts (sg_relayout_sample_compact). Returns the
        words used."""
        g = self._relgeo
        if g is None:
            L = self.L
            arr = np.array([L, self.S, self.o_V, self.o_es, self.o_ed] + self._voff_l + self._eoff_l,
                           dtype=np.int64)
            g = self._relgeo = (arr, arr.ctypes.data, max(self.cap_nV + self.cap_nE + [self.S]))
        _lib.call("sg_relayout_sample_compact" if pin.RS else "sg_relayout_sample_hdr", stage.data_ptr(),
                  buf.data_ptr(), g[1], g[2], _lib.stream_ptr())
        L = self.L
        return self.o_ed + self._eoff_l[L - 1] + nE[L - 1] if L else self.o_es


def _h2d_pinned(pin, device):
    """One H2D of a native-sampler sample's pinned buffer into the reused
    device staging buffer (current stream); the pinned buffer stays referenced
    until an event after the copy has completed (_InFlight)."""
    n = pin.dma_words
    stage = _STAGE.get(n, device)
    _lib.call("sg_copy_async", stage.data_ptr(), pin.base, 4 * n, _lib.stream_ptr())
    _INFLIGHT.hold(pin.tensor)
    return stage


class _Stage:
    """Device staging buffer of the direct path, reused across calls (its uses
    are ordered on the current stream)."""

    def __init__(self):
        self.t = None

    def get(self, n, device):
        idx = device.index if device.index is not None else torch._C._cuda_getDevice()
        t = self.t
        if t is not None and t.numel() >= n and t.device.index == idx:
            return t
        device = torch.device("cuda", idx)
        if self.t is None or self.t.numel() < n or self.t.device != device:
            self.t = torch.empty(max(int(n * 1.25), 1 << 16), dtype=torch.int32, device=device)
        return self.t


class _InFlight:
    """Pinned sample buffers whose H2D may still be running: each is kept
    alive until an event recorded after its copy has completed (the caller
    may drop the sample right after split_minibatch)."""

    def __init__(self):
        self.q = []
        self.free = []  # completed events, recorded again (no creation per call)

    def hold(self, t):
        ev = self.free.pop() if self.free else torch.cuda.Event()
        ev.record(_lib.current_stream())
        self.q.append((ev, t))
        while self.q and (len(self.q) > 64 or self.q[0][0].query()):
            if len(self.q) > 64:
                self.q[0][0].synchronize()
            self.free.append(self.q.pop(0)[0])


_STAGE = _Stage()
_INFLIGHT = _InFlight()
_LAYOUTS = {}
_DIRECT = os.environ.get("SG_SAMPLE_DIRECT", "1") != "0"


def _i32_or_i64(a):
    a = np.asarray(a)
    if a.dtype not in (np.int32, np.int64):
        a = a.astype(np.int64)
    return np.ascontiguousarray(a)


class _PinnedRing:
    """Two reusable pinned staging slots for split_minibatch's H2D copy; a slot
    is repacked only after its previous copy completed (the copy is async)."""

    def __init__(self):
        self.bufs = [None, None]
        self.ev = [None, None]
        self.slot = 0

    def pack(self, geo, sample):
        k = self.slot
        if self.ev[k] is not None:
            self.ev[k].synchronize()
        if self.bufs[k] is None or self.bufs[k].numel() < geo.words:
            self.bufs[k] = torch.empty(max(geo.words, 1 << 16), dtype=torch.int32, pin_memory=True)
        hb = self.bufs[k]
        used = geo.pack(sample, hb.numpy())
        return hb, used

    def record(self):
        ev = torch.cuda.Event()
        ev.record()
        self.ev[self.slot] = ev
        self.slot ^= 1


_PINNED = _PinnedRing()


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
                 dst_grouped: bool, device=None, host_V=None, sizes=None, defer=False, views=None):
        """nV / nE are the CAPACITIES the layout is built for; `sizes` (device
        int64 [nV_0..nV_L, nE_1..nE_L]) gives the actual sizes (default: the
        capacities). V / esrc / edst hold layer l at the capacity offsets.
        defer=True postpones the workspace and the split kernel to the first
        use of `ws` (split_minibatch: a SplitExecutor on the captured path
        re-splits inside its graph and never needs it)."""
        lib = _lib.load()
        self.device = torch.device(device or "cuda")
        self.pm = pm
        self.cache = cache
        self.g = pm.num_devices
        self.L = len(nE)
        self.nV = [int(x) for x in nV]
        self.nE = [int(x) for x in nE]
        self.dst_grouped = bool(dst_grouped)
        key = (self.L, self.g, tuple(self.nV), tuple(self.nE), len(pm.assignment))
        lay = _LAYOUTS.get(key)  # read-only once built: shared by splits of one geometry
        if lay is None:
            lay = _lib.SgSplitLayout()
            nVa = (C.c_int64 * (self.L + 1))(*self.nV)
            nEa = (C.c_int64 * max(self.L, 1))(*(self.nE or [0]))
            _lib.check(lib.sg_split_layout(self.L, self.g, nVa, nEa, len(pm.assignment), C.byref(lay)),
                       "split_layout")
            if len(_LAYOUTS) > 256:
                _LAYOUTS.clear()
            _LAYOUTS[key] = lay
        self.lay = lay
        if views is None:
            self.V, self.esrc, self.edst = V, esrc, edst
            self.sizes = sizes
        else:  # (V, esrc, edst, sizes) built on first access (__getattr__)
            self._views_fn = views
        self._host_V = host_V
        n = len(pm.assignment)
        if cache is not None and getattr(cache, "_all", None) is None:
            cache._all = cache.covers_all(n)
        self._flags = (1 if self.dst_grouped else 0) | (2 if cache is not None and cache._all else 0)
        self.all_cached = bool(self._flags & 2)
        self.packed = None
        self._meta = None
        self._views = None
        if not defer:
            self._run_split()

    def _run_split(self):
        """Allocate the workspace and launch sg_split_run (on the current stream)."""
        ws = torch.empty(int(self.lay.total_bytes), dtype=torch.uint8, device=self.device)
        n = len(self.pm.assignment)
        bits = self.cache.device_bits(n, self.device) if self.cache is not None else None
        _lib.check(_lib.load().sg_split_run(_lib.ptr(ws), C.byref(self.lay), _lib.ptr(self.V), _lib.ptr(self.esrc),
                                            _lib.ptr(self.edst), _lib.ptr(self.sizes),
                                            _lib.ptr(self.pm.device_u8(self.device)), _lib.ptr(bits), self._flags,
                                            _lib.stream_ptr()),
                   "split_run")
        self.ws = ws

    def __getattr__(self, name):
        # only reached for attributes not set yet: the deferred sample views
        # and workspace
        d = self.__dict__
        if name in ("V", "esrc", "edst", "sizes") and "_views_fn" in d:
            d["V"], d["esrc"], d["edst"], d["sizes"] = d.pop("_views_fn")()
            return d[name]
        if name == "ws" and "lay" in d:
            self._run_split()
            return d["ws"]
        raise AttributeError(name)

    @property
    def host_V(self):
        hv = self._host_V
        if callable(hv):
            hv = self._host_V = hv()
        return hv

    @host_V.setter
    def host_V(self, v):
        self._host_V = v

    # -- construction from a host sample ------------------------------------
    @classmethod
    def from_sample_packed(cls, sample, pm, cache=None, device=None, defer=True):
        """The sample in the captured-step layout (StaticSample: one int32
        buffer [sizes | V | esrc | edst], layer l at its capacity offset) with
        capacities from a geometry that only grows (PackGeometry.for_sizes),
        so that successive samples map onto one cached CUDA graph of the
        executor.
        One pinned pack + one H2D; the split kernel is deferred (see __init__).
        Needs a destination-grouped sample."""
        sample = as_sample(sample)
        dev = torch.device(device or "cuda")
        pin = getattr(sample, "pinned", None)
        stage = None
        if pin is not None and pin.vbound <= len(pm.assignment) and _DIRECT and pin.intact(sample):
            stage = _h2d_pinned(pin, dev)  # first: the host work below overlaps the DMA
        nV, nE = sample.sizes()
        geo = PackGeometry.for_sizes(nV, nE, scope=(len(nE), len(pm.assignment), pm.num_devices))
        buf = torch.empty(geo.words, dtype=torch.int32, device=dev)
        if stage is not None:  # the geometry fits the sizes (for_sizes)
            used = geo.relayout_from_stage(sample, pin, stage, buf, nE)
            h2d = 4 * pin.dma_words
        else:
            h2d = None
            hb, used = _PINNED.pack(geo, sample)
            lo, hi = geo.last_vrange
            if sum(nV) and (lo < 0 or hi >= len(pm.assignment)):  # checked while packing
                raise ValueError("sample vertex missing from partition map")
            buf[:used].copy_(hb[:used], non_blocking=True)
            _PINNED.record()
        VC = int(geo.voff[-1])

        def views():  # built on first use: the captured executor path reads only `packed`
            return (buf[geo.o_V:geo.o_V + VC], buf[geo.o_es:geo.o_es + geo.EC], buf[geo.o_ed:geo.o_ed + geo.EC],
                    buf[:geo.S].view(torch.int64))

        def host_V():
            out = np.zeros(VC, dtype=np.int32)
            for l, v in enumerate(sample.layer_vertices):
                out[geo.voff[l]:geo.voff[l] + len(v)] = v
            return out

        ds = cls(None, None, None, geo.cap_nV, geo.cap_nE, pm, cache, True, dev, host_V=host_V, defer=defer,
                 views=views)
        ds.packed = (buf, used, geo)
        ds.h2d_bytes = h2d if h2d is not None else 4 * used  # what crossed PCIe for this sample
        ds.num_targets = len(sample.targets)
        return ds

    @classmethod
    def from_sample(cls, sample, pm, cache=None, device=None):
        sample = as_sample(sample)
        nV, nE = sample.sizes()
        V, es, ed = sample.packed()
        dev = torch.device(device or "cuda")
        Vt = pinned_from(V).to(dev, non_blocking=True)
        st = pinned_from(es).to(dev, non_blocking=True)
        dt = pinned_from(ed).to(dev, non_blocking=True)
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
    if sample.is_dst_grouped():  # the vertex range is checked while packing
        ds = DeviceSplit.from_sample_packed(sample, pm, cache)
    else:
        n = len(pm.assignment)
        for v in sample.layer_vertices:
            v = np.asarray(v)
            if len(v) and (v.max() >= n or v.min() < 0):
                raise ValueError("sample vertex missing from partition map")
        ds = DeviceSplit.from_sample(sample, pm, cache)
    return _lazy_views(ds)


def _lazy_views(ds):
    """(splits, plan) whose host contents are built from the device split on
    first access (one D2H of the workspace); SplitExecutor reads only
    `.device_split` and never triggers it."""
    splits = SplitList()
    splits.device_split = ds
    plan = ShufflePlan(ds.L, ds.g, device_split=ds)
    state = {}

    def fill():
        if not state:
            state["v"] = ds.to_reference_types()
        return state["v"]

    splits._fill_fn = lambda: list.extend(splits, fill()[0])
    plan.entries = _LazyEntries(lambda: fill()[1].entries)
    return splits, plan


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
