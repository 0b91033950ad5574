"""GPU-resident partitioned feature cache (replaces _load_inputs, engine.py:160-167).

Rows of the cached vertices live in one fp32 table on the device, grouped by
owner partition; `cache_slot[gid]` maps a vertex to its row (-1 = not cached).
Per-iteration misses (the reference's load_gids / host_bytes) are read by a
zero-copy device gather from the host feature matrix (page-locked and mapped
into the device address space) into a staging area appended to the table;
the counts come from the device split, so the staging runs inside captured
steps too. The
aggregation kernels read the table through an int32 row indirection (no h0
materialisation).
"""

from __future__ import annotations

import numpy as np
import torch

from paper_2303_13775_b200 import _lib


def padded_stride(feat_dim, pad_rows):
    """Row stride of the device table. With pad_rows, a width > 64 that is not
    a multiple of 32 floats is padded (with zeros) to whole 128-byte lines: a
    warp then gathers a row as full lines, measured ~1.4x faster than 400-byte
    rows on B200 (tools/gather_roof.py)."""
    F = int(feat_dim)
    if pad_rows and F > 64 and F % 32:
        return (F + 31) // 32 * 32
    return F


class FeatureStore:
    def __init__(self, table, cache_slot, n_cached, feat_dim, host_features=None, identity=False):
        self.table = table                  # [n_cached + staging, row_stride] fp32 cuda
        self.cache_slot = cache_slot        # [n] int32 cuda
        self.n_cached = int(n_cached)
        self.feat_dim = int(feat_dim)
        self.row_stride = int(table.shape[1]) if table.dim() == 2 else int(feat_dim)
        self.host_features = host_features  # numpy [n, F] for misses (or None)
        self.identity = bool(identity)      # row of vertex v is v (whole graph cached in id order)

    @property
    def padded(self):
        return self.row_stride != self.feat_dim

    @staticmethod
    def _alloc(rows, feat_dim, stride, device):
        t = torch.empty((rows, stride), dtype=torch.float32, device=device)
        if stride != feat_dim:
            t[:, feat_dim:].zero_()
        return t

    @property
    def device(self):
        return self.table.device

    @classmethod
    def from_host(cls, features, cache=None, devices=None, device="cuda", pad_rows=False, staging_rows=0):
        """Upload the cached rows of `devices` (default: all) from a host
        feature matrix; uncached rows are served as misses from `features`
        (staging_rows: miss rows to reserve up front, e.g. the captured
        layer-0 capacity; grown on demand otherwise)."""
        feats = np.ascontiguousarray(features, dtype=np.float32)
        n, F = feats.shape
        S = padded_stride(F, pad_rows)
        slot = np.full(n, -1, dtype=np.int32)
        if cache is not None:
            devs = range(cache.num_devices) if devices is None else devices
            ids = np.concatenate([cache.cached[d] for d in devs]) if len(list(devs)) else np.empty(0, np.int64)
            ids = np.asarray(ids, dtype=np.int64)
        else:
            ids = np.empty(0, dtype=np.int64)
        slot[ids] = np.arange(len(ids), dtype=np.int32)
        table = cls._alloc(len(ids) + int(staging_rows), F, S, device)
        if len(ids):
            table[:len(ids), :F].copy_(torch.from_numpy(feats[ids]))
        return cls(table, torch.from_numpy(slot).to(device), len(ids), F, feats)

    @classmethod
    def synthetic(cls, n, feat_dim, seed, row_ids=None, device="cuda", pad_rows=False):
        """Fully cached synthetic U[0,1) features generated ON the device
        (sg_fill_uniform); row_ids (sorted global ids, default all) selects the
        vertices this device caches. Values equal graph.synthetic_features."""
        lib = _lib.load()
        S = padded_stride(feat_dim, pad_rows)

        def fill(dst, rows, row0):
            # generate [rows, F] contiguously, then place into the (padded) rows in chunks
            if S == feat_dim:
                _lib.check(lib.sg_fill_uniform(_lib.ptr(dst), int(rows), int(feat_dim), int(seed), int(row0),
                                               _lib.stream_ptr()), "fill_uniform")
                return
            chunk = 1 << 20
            tmp = torch.empty((min(rows, chunk), feat_dim), dtype=torch.float32, device=device)
            for a in range(0, rows, chunk):
                b = min(rows, a + chunk)
                _lib.check(lib.sg_fill_uniform(_lib.ptr(tmp), int(b - a), int(feat_dim), int(seed),
                                               int(row0 + a), _lib.stream_ptr()), "fill_uniform")
                dst[a:b, :feat_dim].copy_(tmp[:b - a])

        if row_ids is None:
            rows = int(n)
            table = cls._alloc(rows, feat_dim, S, device)
            fill(table, rows, 0)
            slot = torch.arange(n, dtype=torch.int32, device=device)
            return cls(table, slot, rows, feat_dim, None, identity=True)
        row_ids = np.asarray(row_ids, dtype=np.int64)
        table = cls._alloc(len(row_ids), feat_dim, S, device)
        # contiguous runs are generated directly
        runs = np.flatnonzero(np.r_[True, np.diff(row_ids) != 1, True])
        for a, b in zip(runs[:-1], runs[1:]):
            fill(table[a:b], int(b - a), int(row_ids[a]))
        slot = np.full(int(n), -1, dtype=np.int32)
        slot[row_ids] = np.arange(len(row_ids), dtype=np.int32)
        return cls(table, torch.from_numpy(slot).to(device), len(row_ids), feat_dim, None)

    # -- cache misses -------------------------------------------------------------
    def host_device_ptr(self):
        """Device address of the host feature matrix (mapped once, refcounted
        per host range): the source of the zero-copy miss gather."""
        if self.host_features is None:
            raise RuntimeError("feature cache miss but no host feature matrix to load from "
                               "(build the FeatureStore with FeatureStore.from_host)")
        if getattr(self, "_hmap", None) is None:
            self._hmap = _map_host(self.host_features)
        return self._hmap

    def ensure_staging(self, rows):
        """Grow the table so `rows` miss rows fit behind the cached ones (must
        run outside CUDA-graph capture; a captured step calls it from its eager
        warm-up)."""
        need = self.n_cached + int(rows)
        if self.table.shape[0] < need:
            if torch.cuda.is_current_stream_capturing():
                raise RuntimeError("feature staging area must be sized before CUDA-graph capture")
            t = self._alloc(need, self.feat_dim, self.row_stride, self.device)
            if self.n_cached:
                t[: self.n_cached] = self.table[: self.n_cached]
            # a CUDA graph captured earlier may still read the old table: keep it alive
            self._retired = getattr(self, "_retired", []) + [self.table]
            self.table = t
        return self.table

    @property
    def staging_rows(self):
        return int(self.table.shape[0]) - self.n_cached

    def stage_misses(self, dsplit, devices=None):
        """Copy this iteration's uncached layer-0 rows of `devices` (default
        all; the global load order of scheduler.py:193-203) behind the cached
        rows, on the device (sg_stage_misses: counts from the device split, no
        host sync). Returns the table."""
        devs = list(range(dsplit.g)) if devices is None else sorted(int(d) for d in devices)
        self.ensure_staging(dsplit.nV[0])
        src = self.host_device_ptr()
        st = _lib.stream_ptr()
        # contiguous device ranges (a rank stages only its own load list)
        runs, a = [], None
        for d in devs:
            if a is None or d != runs[-1][1]:
                runs.append([d, d + 1])
            else:
                runs[-1][1] = d + 1
            a = d
        for d0, d1 in runs:
            _lib.call("sg_stage_misses", _lib.ptr(dsplit.ws), dsplit.lay, d0, d1, _lib.ptr(dsplit.V), src,
                      self.feat_dim, _lib.ptr(self.table), self.row_stride, self.n_cached, self.staging_rows, st)
        return self.table

    def __del__(self):
        h = getattr(self, "_hmap", None)
        if h is not None and self.host_features is not None:
            try:
                _unmap_host(self.host_features)
            except Exception:
                pass
            self._hmap = None


_MAPPED = {}  # host address -> [refcount, device address]


def _map_host(arr):
    import ctypes
    key = int(arr.ctypes.data)
    ent = _MAPPED.get(key)
    if ent is None:
        dptr = ctypes.c_void_p()
        _lib.check(_lib.load().sg_host_map(key, int(arr.nbytes), ctypes.byref(dptr)), "sg_host_map")
        ent = _MAPPED[key] = [0, int(dptr.value)]
    ent[0] += 1
    return ent[1]


def _unmap_host(arr):
    key = int(arr.ctypes.data)
    ent = _MAPPED.get(key)
    if ent is None:
        return
    ent[0] -= 1
    if ent[0] <= 0:
        del _MAPPED[key]
        _lib.load().sg_host_unmap(key)
