"""Graph container (in-CSR) and the synthetic power-law generator.

Mirrors splitgnn.graph.Graph (graph.py:23-100): `col_indices[row_offsets[v]:
row_offsets[v+1]]` are the sources of the edges entering v. Column indices are
int32 (every supported graph has < 2^31 vertices) so the 1.6B-edge
papers100M shape fits in host RAM; features are optional float32 (the
reference holds float64; fp32 is the arithmetic type of the B200 path).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from paper_2303_13775_b200 import _lib


class GraphError(ValueError):
    """Malformed graph data (graph.py:19-20)."""


@dataclass(frozen=True)
class Graph:
    num_vertices: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    features: np.ndarray | None = None

    def __post_init__(self):
        ro = np.ascontiguousarray(self.row_offsets, dtype=np.int64)
        ci = np.ascontiguousarray(self.col_indices, dtype=np.int32)
        object.__setattr__(self, "row_offsets", ro)
        object.__setattr__(self, "col_indices", ci)
        if self.features is not None:
            object.__setattr__(self, "features",
                               np.ascontiguousarray(self.features, dtype=np.float32))
        n = self.num_vertices
        if ro.shape != (n + 1,) or ro[0] != 0 or ro[-1] != len(ci):
            raise GraphError("row_offsets inconsistent with num_vertices / edge count")
        if self.features is not None and self.features.shape[0] != n:
            raise GraphError(f"feature rows ({self.features.shape[0]}) != num_vertices ({n})")

    @property
    def num_edges(self) -> int:
        return int(len(self.col_indices))

    @property
    def feat_dim(self) -> int:
        return 0 if self.features is None else int(self.features.shape[1])

    def in_degrees(self):
        return np.diff(self.row_offsets)

    def out_degrees(self):
        return np.bincount(self.col_indices, minlength=self.num_vertices).astype(np.int64)

    def with_features(self, features):
        return Graph(self.num_vertices, self.row_offsets, self.col_indices, features)


def from_edges(num_vertices, src, dst, features=None) -> Graph:
    """In-CSR from parallel edge arrays, stable within each destination
    (graph.py:103-128)."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    if len(src) != len(dst):
        raise GraphError("src and dst length mismatch")
    if len(src) and (min(src.min(), dst.min()) < 0 or max(src.max(), dst.max()) >= num_vertices):
        raise GraphError("vertex id out of range")
    order = np.argsort(dst, kind="stable")
    offsets = np.zeros(num_vertices + 1, dtype=np.int64)
    np.cumsum(np.bincount(dst, minlength=num_vertices), out=offsets[1:])
    return Graph(num_vertices, offsets, src[order], features)


def from_reference(graph) -> Graph:
    """Adopt a reference splitgnn.graph.Graph (or any object with the same
    fields) without copying its topology semantics."""
    feats = None if graph.features is None else np.asarray(graph.features, dtype=np.float32)
    return Graph(int(graph.num_vertices), graph.row_offsets, graph.col_indices, feats)


def generate_powerlaw(n, m, *, blocks=64, p_local=0.92, gamma=2.1, seed=0, threads=0) -> Graph:
    """Block-planted Chung-Lu power-law graph, native + threaded.

    Vertex weight w_v = r_v^(-1/(gamma-1)) with r a seeded permutation of
    1..n; each edge draws dst ~ w, then src ~ w restricted to dst's
    contiguous-id block with probability p_local, else src ~ w globally.
    Features are NOT attached (they are generated on the GPU, see
    features.FeatureStore.synthetic); use synthetic_features() for host rows.
    """
    lib = _lib.load()
    ro = np.empty(n + 1, dtype=np.int64)
    ci = np.empty(m, dtype=np.int32)
    _lib.check(lib.sg_gen_powerlaw(int(n), int(m), int(blocks), float(p_local), float(gamma),
                                   int(seed), int(threads), _lib.ptr(ro), _lib.ptr(ci)),
               "gen_powerlaw")
    return Graph(int(n), ro, ci)


def synthetic_features(rows, feat_dim, seed, row_ids=None) -> np.ndarray:
    """Host twin of the GPU feature generator: U[0,1) with 24 random bits,
    bit-identical to sg_fill_uniform for the same (seed, row, col)."""
    lib = _lib.load()
    if row_ids is not None:
        row_ids = np.ascontiguousarray(row_ids, dtype=np.int64)
        rows = len(row_ids)
    out = np.empty((int(rows), int(feat_dim)), dtype=np.float32)
    _lib.check(lib.sg_fill_uniform_host(_lib.ptr(out), int(rows), int(feat_dim), int(seed), 0,
                                        _lib.ptr(row_ids) if row_ids is not None else None),
               "fill_uniform_host")
    return out


def synthetic_labels(n, num_classes, seed) -> np.ndarray:
    lib = _lib.load()
    out = np.empty(int(n), dtype=np.int32)
    _lib.check(lib.sg_gen_labels(int(n), int(num_classes), int(seed), _lib.ptr(out)), "gen_labels")
    return out


# ---- SPLG binary CSR (graph.py:238-273 of the reference: same byte layout) -------
BINARY_MAGIC = b"SPLG"
BINARY_VERSION = 1


def save_binary_csr(graph: Graph, path):
    """magic, u32 version, u64 n, m, feat_dim, then i64 row_offsets, i64
    col_indices and (feat_dim > 0) f64 features, little-endian."""
    import struct
    with open(path, "wb") as fh:
        fh.write(BINARY_MAGIC)
        fh.write(struct.pack("<I", BINARY_VERSION))
        fh.write(struct.pack("<QQQ", graph.num_vertices, graph.num_edges, graph.feat_dim))
        fh.write(graph.row_offsets.astype("<i8").tobytes())
        chunk = 1 << 26
        for i in range(0, graph.num_edges, chunk):
            fh.write(graph.col_indices[i:i + chunk].astype("<i8").tobytes())
        if graph.features is not None:
            for i in range(0, graph.num_vertices, 1 << 20):
                fh.write(graph.features[i:i + (1 << 20)].astype("<f8").tobytes())


def load_binary_csr(path) -> Graph:
    """Memory-mapped SPLG reader: the i64 arrays are mapped, not read, and
    narrowed chunk by chunk (papers100M: 1.6B edges)."""
    import struct
    with open(path, "rb") as fh:
        magic = fh.read(4)
        if magic != BINARY_MAGIC:
            raise GraphError(f"{path}: bad magic {magic!r}")
        (version,) = struct.unpack("<I", fh.read(4))
        if version != BINARY_VERSION:
            raise GraphError(f"{path}: unsupported version {version}")
        n, m, fd = struct.unpack("<QQQ", fh.read(24))
    base = 4 + 4 + 24
    mm = np.memmap(path, dtype="<i8", mode="r", offset=base, shape=(n + 1 + m,))
    offsets = np.asarray(mm[:n + 1], dtype=np.int64)
    indices = np.empty(m, dtype=np.int32)
    chunk = 1 << 26
    for i in range(0, m, chunk):
        indices[i:i + chunk] = mm[n + 1 + i:n + 1 + min(m, i + chunk)]
    feats = None
    if fd:
        fm = np.memmap(path, dtype="<f8", mode="r", offset=base + 8 * (n + 1 + m), shape=(n, fd))
        feats = np.empty((n, fd), dtype=np.float32)
        for i in range(0, n, 1 << 20):
            feats[i:i + (1 << 20)] = fm[i:i + (1 << 20)]
    del mm
    return Graph(int(n), offsets, indices, feats)
