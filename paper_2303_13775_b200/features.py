"""GPU-resident partitioned feature cache (replaces _load_inputs, engine.py:160-167).

Rows of the cached vertices live in one fp32 table on the device, grouped by
owner partition; `cache_slot[gid]` maps a vertex to its row (-1 = not cached).
Per-iteration misses (the reference's load_gids / host_bytes) are gathered on
the host and copied into a staging area appended to the table. The
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
    def from_host(cls, features, cache=None, devices=None, device="cuda", pad_rows=False):
        """Upload the cached rows of `devices` (default: all) from a host
        feature matrix; uncached rows are served as misses from `features`."""
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
        table = cls._alloc(len(ids), F, S, device)
        if len(ids):
            table[:, :F].copy_(torch.from_numpy(feats[ids]))
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

    def stage_misses(self, dsplit, meta):
        """Copy this iteration's uncached layer-0 rows (all devices' load
        lists, global load order) behind the cached rows. Returns bytes moved."""
        total = int(meta.load_off[dsplit.g])
        if total == 0:
            return 0
        if self.host_features is None:
            raise RuntimeError("feature cache miss but no host feature matrix to load from")
        lay = dsplit.lay
        grouped = dsplit.i32(lay.o_grouped, total, start=int(lay.nVtot)).cpu().numpy()
        V0 = np.asarray(dsplit.host_V[: dsplit.nV[0]]) if dsplit.host_V is not None else \
            dsplit.V[: dsplit.nV[0]].cpu().numpy()
        gids = V0[grouped]
        rows = torch.from_numpy(self.host_features[gids]).pin_memory()
        need = self.n_cached + total
        if self.table.shape[0] < need:
            t = self._alloc(need, self.feat_dim, self.row_stride, self.device)
            t[: self.n_cached] = self.table[: self.n_cached]
            self.table = t
        self.table[self.n_cached:need, :self.feat_dim].copy_(rows, non_blocking=True)
        self._keep = rows
        return int(rows.numel() * 4)
