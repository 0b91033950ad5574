"""Partition map and per-device feature-cache selection.

Mirrors splitgnn.partition's data types (partition.py:20-91) and the cache
policy build_cache (:358-377). The offline multilevel partitioner itself is
out of scope for the B200 hot path; range_partition
gives the contiguous-id map the benchmark configs use.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


def max_part_size(n: int, g: int, eps: float) -> int:
    """Largest allowed per-device vertex count (partition.py:94-99)."""
    if n == 0:
        return 0
    return max(math.ceil(n / g), math.ceil((1.0 + eps) * n / g - 1e-7))


@dataclass
class PartitionMap:
    assignment: np.ndarray
    num_devices: int
    balance_eps: float = 0.05

    def __post_init__(self):
        self.assignment = np.ascontiguousarray(self.assignment, dtype=np.int64)
        if self.num_devices < 1:
            raise ValueError("num_devices must be >= 1")
        if self.balance_eps < 0:
            raise ValueError("balance_eps must be >= 0")
        a = self.assignment
        if len(a) and (a.min() < 0 or a.max() >= self.num_devices):
            raise ValueError("device id out of range in assignment")
        cap = max_part_size(len(a), self.num_devices, self.balance_eps)
        counts = self.counts()
        if counts.max(initial=0) > cap:
            raise ValueError(f"partition violates balance: max part {counts.max()} > cap {cap}")
        self._dev_u8 = None

    def counts(self):
        return np.bincount(self.assignment, minlength=self.num_devices)

    def device_vertices(self, d):
        return np.flatnonzero(self.assignment == d)

    def device_u8(self, device="cuda"):
        """uint8 copy of the map resident on the GPU (cached)."""
        import torch
        dev = torch.device(device)
        if dev.type == "cuda" and dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        if self._dev_u8 is None or self._dev_u8.device != dev:
            if self.num_devices > 16:
                raise ValueError("the B200 splitter supports at most 16 devices")
            self._dev_u8 = torch.from_numpy(self.assignment.astype(np.uint8)).to(dev)
        return self._dev_u8


def range_partition(n: int, g: int) -> PartitionMap:
    """Contiguous-id map P(v) = floor(v*g/n) (block-aligned)."""
    return PartitionMap((np.arange(n, dtype=np.int64) * g) // max(n, 1), g, 1.0)


@dataclass
class CacheState:
    """Per-device cached vertex ids, each inside its own partition
    (partition.py:55-91)."""

    cached: list
    capacity_fraction: float

    def __post_init__(self):
        self.cached = [np.ascontiguousarray(c, dtype=np.int64) for c in self.cached]
        self._bits = None

    @property
    def num_devices(self):
        return len(self.cached)

    def global_mask(self, n):
        mask = np.zeros(n, dtype=bool)
        for ids in self.cached:
            mask[ids] = True
        return mask

    def device_masks(self, n):
        """Per-device boolean cache masks (partition.py:77-83)."""
        masks = []
        for ids in self.cached:
            m = np.zeros(n, dtype=bool)
            m[ids] = True
            masks.append(m)
        return masks

    def device_bits(self, n, device="cuda"):
        """Global cache mask as a uint32 bitmap on the GPU (cached)."""
        import torch
        if self._bits is None:
            words = (n + 31) // 32
            mask = np.zeros(words * 32, dtype=bool)
            mask[:n] = self.global_mask(n)
            packed = np.packbits(mask, bitorder="little")
            self._bits = torch.from_numpy(packed.view(np.uint32).copy()).to(device)
        return self._bits

    def covers_all(self, n):
        """True when every vertex is cached somewhere (no host loads ever)."""
        return int(sum(len(c) for c in self.cached)) >= n and bool(self.global_mask(n).all())

    def validate(self, pm, n):
        cap = math.ceil(self.capacity_fraction * n - 1e-9)
        for d, ids in enumerate(self.cached):
            if len(ids) > cap:
                raise ValueError(f"device {d} caches {len(ids)} > capacity {cap}")
            if len(ids) and np.any(pm.assignment[ids] != d):
                raise ValueError(f"device {d} caches vertices outside its partition")


def build_cache(graph, pm: PartitionMap, capacity_fraction: float) -> CacheState:
    """Highest in+out degree vertices of each partition, ties by lower id
    (partition.py:358-377)."""
    if not (0.0 <= capacity_fraction <= 1.0):
        raise ValueError("capacity_fraction must be in [0, 1]")
    n = graph.num_vertices
    cap = math.ceil(capacity_fraction * n - 1e-9)
    degree = graph.in_degrees() + graph.out_degrees()
    cached = []
    for d in range(pm.num_devices):
        ids = pm.device_vertices(d)
        order = np.lexsort((ids, -degree[ids]))
        cached.append(np.sort(ids[order][:cap]))
    return CacheState(cached, capacity_fraction)


def full_cache(pm: PartitionMap) -> CacheState:
    """Every partition fully cached on its device (zero host bytes,
    test_acceptance.py:161-172)."""
    n = len(pm.assignment)
    frac = (pm.counts().max() / n) if n else 0.0
    return CacheState([pm.device_vertices(d) for d in range(pm.num_devices)], float(frac))


# ---- balanced k-way partitioning on the GPU (csrc/partition.cu) -------------------

class _DeviceGraph:
    """In-CSR and out-CSR (the transpose, by a stable device sort) of a graph."""

    def __init__(self, graph, device="cuda"):
        import torch
        dev = torch.device(device)
        n = int(graph.num_vertices)
        self.n = n
        self.ro = torch.from_numpy(np.asarray(graph.row_offsets, dtype=np.int64)).to(dev)
        self.ci = torch.from_numpy(np.asarray(graph.col_indices, dtype=np.int32)).to(dev)
        deg = self.ro[1:] - self.ro[:-1]
        dst = torch.repeat_interleave(torch.arange(n, dtype=torch.int32, device=dev), deg)
        src_sorted, perm = torch.sort(self.ci, stable=True)
        self.oci = dst[perm].contiguous()
        cnt = torch.bincount(self.ci.long(), minlength=n)
        self.oro = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        self.oro[1:] = torch.cumsum(cnt, 0)
        del src_sorted, perm, dst

    def cut(self, part):
        import torch
        out = torch.zeros(1, dtype=torch.int64, device=part.device)
        from paper_2303_13775_b200 import _lib
        _lib.call("sg_partition_cut", _lib.ptr(self.ro), _lib.ptr(self.ci), self.n, _lib.ptr(part), _lib.ptr(out),
                  _lib.stream_ptr())
        return int(out.item())


def _refine_device(dg, part, g, cap, seed, max_passes):
    """Parallel refinement rounds (two rounds per reference pass: each round
    moves a seeded half of the vertices); a round that raised the cut is
    undone, so the history never increases."""
    import torch
    from paper_2303_13775_b200 import _lib
    dev = part.device
    sizes = torch.bincount(part.long(), minlength=g).to(torch.int64)
    ws = torch.empty(8 * dg.n + 4 * 16 * 65 + 64, dtype=torch.uint8, device=dev)
    moved = torch.zeros(1, dtype=torch.int64, device=dev)
    cut = dg.cut(part)
    history = [cut]
    idle = 0
    for r in range(2 * max_passes):
        prev = part.clone()
        _lib.call("sg_partition_round", _lib.ptr(dg.ro), _lib.ptr(dg.ci), _lib.ptr(dg.oro), _lib.ptr(dg.oci), dg.n,
                  g, int(cap), int(seed) & (2**64 - 1), r, _lib.ptr(part), _lib.ptr(sizes), _lib.ptr(ws),
                  _lib.ptr(moved), _lib.stream_ptr())
        nmoved = int(moved.item())
        new = dg.cut(part) if nmoved else cut
        if new > cut:  # simultaneous moves of neighbours made it worse: undo
            part.copy_(prev)
            sizes = torch.bincount(part.long(), minlength=g).to(torch.int64)
            nmoved = 0
        else:
            cut = new
        if r % 2 == 1:
            history.append(cut)
        idle = idle + 1 if nmoved == 0 else 0
        if idle >= 2:
            break
    return part, history


def refine_assignment(graph, assignment, num_devices, balance_eps=0.05, max_passes=10, seed=0):
    """Refine an existing assignment on the full graph (partition.py:273-295),
    on the GPU. Returns (refined assignment, cut history per pass) -- the
    history is in directed-arc units and never increases."""
    import torch
    g = int(num_devices)
    if g > 16:
        raise ValueError("the GPU partitioner supports at most 16 parts")
    n = int(graph.num_vertices)
    cap = max_part_size(n, g, balance_eps)
    dg = _DeviceGraph(graph)
    part = torch.from_numpy(np.asarray(assignment, dtype=np.int32)).cuda()
    part, hist = _refine_device(dg, part, g, cap, seed, max_passes)
    return part.cpu().numpy().astype(np.int64), hist


def partition_graph(graph, g, balance_eps=0.05, seed=0, max_passes=25) -> PartitionMap:
    """Balanced k-way partition with a small edge cut (partition.py:298-349),
    GPU edition: the contiguous-id map (balanced by construction) refined by
    parallel gain moves on the symmetrised graph within the balance cap.
    Deterministic given `seed`. Not the reference's multilevel heuristic (so
    not the same assignment); same contract: balanced within eps, cut never
    worse than the starting map."""
    import torch
    n = int(graph.num_vertices)
    if g < 1:
        raise ValueError("g must be >= 1")
    if g > n:
        raise ValueError(f"g={g} exceeds num_vertices={n}")
    if balance_eps < 0:
        raise ValueError("balance_eps must be >= 0")
    if g == 1:
        return PartitionMap(np.zeros(n, dtype=np.int64), 1, balance_eps)
    if g > 16:
        raise ValueError("the GPU partitioner supports at most 16 parts")
    cap = max_part_size(n, g, balance_eps)
    dg = _DeviceGraph(graph)
    part = ((torch.arange(n, dtype=torch.int64, device="cuda") * g) // n).to(torch.int32)
    part, _ = _refine_device(dg, part, g, cap, seed, max_passes)
    return PartitionMap(part.cpu().numpy().astype(np.int64), g, balance_eps)


def cut_size(graph, pm: PartitionMap) -> int:
    """Directed edges whose endpoints live on different devices (partition.py:352-355)."""
    import torch
    dg = _DeviceGraph.__new__(_DeviceGraph)
    dg.n = int(graph.num_vertices)
    dg.ro = torch.from_numpy(np.asarray(graph.row_offsets, dtype=np.int64)).cuda()
    dg.ci = torch.from_numpy(np.asarray(graph.col_indices, dtype=np.int32)).cuda()
    return dg.cut(torch.from_numpy(pm.assignment.astype(np.int32)).cuda())
