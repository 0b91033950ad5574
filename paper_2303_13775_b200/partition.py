"""Partition map and per-device feature-cache selection.

Mirrors splitgnn.partition's data types (partition.py:20-91), the cache
policy build_cache (:358-377, selected on the GPU) and the offline multilevel
partitioner (:298-349) as a GPU multilevel scheme;
range_partition gives the contiguous-id map the benchmark configs use
(PAPER.md:821).
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
    (partition.py:358-377), selected on the GPU: degrees by device bincount,
    one stable device sort of (part, -degree) keys over the id-ordered vertices
    (so equal degrees keep ascending ids), the first `cap` of every part."""
    import torch
    if not (0.0 <= capacity_fraction <= 1.0):
        raise ValueError("capacity_fraction must be in [0, 1]")
    n = int(graph.num_vertices)
    cap = math.ceil(capacity_fraction * n - 1e-9)
    g = pm.num_devices
    if n == 0:
        return CacheState([np.empty(0, dtype=np.int64) for _ in range(g)], capacity_fraction)
    dev = torch.device("cuda")
    ro = torch.from_numpy(np.asarray(graph.row_offsets, dtype=np.int64)).to(dev)
    ci = torch.from_numpy(np.asarray(graph.col_indices, dtype=np.int64)).to(dev)
    degree = (ro[1:] - ro[:-1]) + torch.bincount(ci, minlength=n)
    part = torch.from_numpy(np.asarray(pm.assignment, dtype=np.int64)).to(dev)
    key = (part << 40) | (int(degree.max()) - degree)
    _, order = torch.sort(key, stable=True)
    counts = torch.bincount(part, minlength=g).cpu().numpy()
    starts = np.concatenate([[0], np.cumsum(counts)[:-1]])
    order = order.cpu().numpy()
    cached = [np.sort(order[s:s + min(cap, int(c))]) for s, c in zip(starts, counts)]
    return CacheState(cached, capacity_fraction)


def full_cache(pm: PartitionMap) -> CacheState:
    """Every partition fully cached on its device (zero host bytes,
    test_acceptance.py:161-172)."""
    n = len(pm.assignment)
    frac = (pm.counts().max() / n) if n else 0.0
    return CacheState([pm.device_vertices(d) for d in range(pm.num_devices)], float(frac))


# ---- balanced k-way partitioning on the GPU (csrc/partition.cu, csrc/host.cpp) ------

class _Level:
    """Symmetric weighted CSR of one level (device tensors): off int64[n+1],
    nbr / wt int32[nnz], vw int32[n]; cmap maps the finer level onto it."""

    def __init__(self, off, nbr, wt, vw):
        self.off, self.nbr, self.wt, self.vw = off, nbr, wt, vw
        self.n = int(vw.numel())

    def cut(self, part):
        """Directed-arc units (entries are counted from both ends)."""
        import torch
        from paper_2303_13775_b200 import _lib
        out = torch.zeros(1, dtype=torch.int64, device=part.device)
        _lib.call("sg_partition_cut_w", _lib.ptr(self.off), _lib.ptr(self.nbr), _lib.ptr(self.wt), self.n,
                  _lib.ptr(part), _lib.ptr(out), _lib.stream_ptr())
        return int(out.item()) // 2

    def sizes(self, part, g):
        import torch
        from paper_2303_13775_b200 import _lib
        out = torch.empty(g, dtype=torch.int64, device=part.device)
        _lib.call("sg_partition_sizes", _lib.ptr(part), _lib.ptr(self.vw), self.n, g, _lib.ptr(out),
                  _lib.stream_ptr())
        return out


def _csr_from_keys(keys, wts, n):
    """Sorted unique (u * n + v) keys with weights -> CSR level."""
    import torch
    u = keys // n
    off = torch.zeros(n + 1, dtype=torch.int64, device=keys.device)
    off[1:] = torch.cumsum(torch.bincount(u, minlength=n), 0)
    return off, (keys - u * n).to(torch.int32), wts.to(torch.int32)


def _symmetric_level(graph, device="cuda"):
    """Level 0: the input graph symmetrised, weight(u,v) = arcs u->v + arcs
    v->u, self loops dropped (partition.py:123-136)."""
    import torch
    dev = torch.device(device)
    n = int(graph.num_vertices)
    ro = torch.from_numpy(np.asarray(graph.row_offsets, dtype=np.int64)).to(dev)
    src = torch.from_numpy(np.asarray(graph.col_indices, dtype=np.int64)).to(dev)
    dst = torch.repeat_interleave(torch.arange(n, dtype=torch.int64, device=dev), ro[1:] - ro[:-1])
    keep = src != dst
    src, dst = src[keep], dst[keep]
    keys = torch.cat([src * n + dst, dst * n + src])
    del src, dst, keep
    uk, cnt = torch.unique(keys, sorted=True, return_counts=True)
    del keys
    off, nbr, wt = _csr_from_keys(uk, cnt, n)
    return _Level(off, nbr, wt, torch.ones(n, dtype=torch.int32, device=dev))


def _match_siblings(level, match, wcap):
    """Two-hop matching for what heavy-edge matching leaves unmatched (on
    power-law graphs: the many low-degree vertices whose only neighbours are
    already-matched hubs): unmatched vertices with the same heaviest neighbour
    (the anchor; ties by lower id) are paired in id order, within the weight
    cap. Without it coarsening stalls after a few levels."""
    import torch
    dev = match.device
    n = level.n
    un = torch.nonzero(match < 0).squeeze(1)
    if un.numel() < 2:
        return
    deg = level.off[1:] - level.off[:-1]
    row = torch.repeat_interleave(torch.arange(n, dtype=torch.int64, device=dev), deg)
    # per-vertex argmax of (weight, -neighbour id) over the CSR row
    key = (level.wt.to(torch.int64) << 32) | (2**31 - 1 - level.nbr.to(torch.int64))
    best = torch.full((n,), -1, dtype=torch.int64, device=dev).scatter_reduce_(0, row, key, "amax")
    anchor = torch.where(best >= 0, 2**31 - 1 - (best & 0xFFFFFFFF), torch.full_like(best, -1))[un]
    keep = anchor >= 0
    un, anchor = un[keep], anchor[keep]
    if un.numel() < 2:
        return
    order = torch.argsort(anchor * n + un)
    un, anchor = un[order], anchor[order]
    m = un.numel()
    pos = torch.arange(m, device=dev)
    start = torch.ones(m, dtype=torch.bool, device=dev)
    start[1:] = anchor[1:] != anchor[:-1]
    run0 = torch.cummax(torch.where(start, pos, torch.zeros_like(pos)), 0).values
    first = ((pos - run0) % 2 == 0)[:-1] & ~start[1:]  # even position in its run, next in the same run
    a, b = un[:-1][first], un[1:][first]
    ok = level.vw[a].to(torch.int64) + level.vw[b].to(torch.int64) <= wcap
    a, b = a[ok], b[ok]
    match[a] = b.to(torch.int32)
    match[b] = a.to(torch.int32)


def _coarsen(level, wcap, seed, rounds=6, two_hop=True):
    """Heavy-edge matching (sg_partition_match_round) and contraction. Returns
    (coarse level, cmap int64[n])."""
    import torch
    from paper_2303_13775_b200 import _lib
    dev = level.vw.device
    n = level.n
    match = torch.full((n,), -1, dtype=torch.int32, device=dev)
    ws = torch.empty(4 * max(n, 1), dtype=torch.uint8, device=dev)
    matched = torch.zeros(1, dtype=torch.int64, device=dev)
    for r in range(rounds):
        _lib.call("sg_partition_match_round", _lib.ptr(level.off), _lib.ptr(level.nbr), _lib.ptr(level.wt),
                  _lib.ptr(level.vw), n, int(wcap), int(seed) & (2**64 - 1), r, _lib.ptr(match), _lib.ptr(ws),
                  _lib.ptr(matched), _lib.stream_ptr())
    idx = torch.arange(n, dtype=torch.int64, device=dev)
    if two_hop:
        _match_siblings(level, match, wcap)
    mate = torch.where(match >= 0, match.to(torch.int64), idx)
    leader = idx <= mate
    cid = torch.cumsum(leader.to(torch.int64), 0) - 1
    cmap = cid[torch.minimum(idx, mate)]
    nc = int(cid[-1].item()) + 1 if n else 0
    vw = torch.zeros(nc, dtype=torch.int64, device=dev).index_add_(0, cmap, level.vw.to(torch.int64))
    u = torch.repeat_interleave(cmap, level.off[1:] - level.off[:-1])
    v = cmap[level.nbr.to(torch.int64)]
    keep = u != v
    keys = u[keep] * nc + v[keep]
    w = level.wt.to(torch.int64)[keep]
    del u, v, keep
    uk, inv = torch.unique(keys, sorted=True, return_inverse=True)
    cw = torch.zeros(uk.numel(), dtype=torch.int64, device=dev).index_add_(0, inv, w)
    off, nbr, wt = _csr_from_keys(uk, cw, nc)
    return _Level(off, nbr, wt, vw.to(torch.int32)), cmap


def _refine_device(level, part, g, cap, seed, max_passes):
    """Parallel refinement rounds on one level (two rounds per reference pass:
    each round moves a seeded half of the vertices); a round that raised the
    cut is undone, so the history (directed-arc units) never increases."""
    import torch
    from paper_2303_13775_b200 import _lib
    dev = part.device
    n = level.n
    sizes = level.sizes(part, g)
    ws = torch.empty(8 * n + 8 * 16 * 64 + 64, dtype=torch.uint8, device=dev)
    moved = torch.zeros(1, dtype=torch.int64, device=dev)
    cut = level.cut(part)
    history = [cut]
    idle = 0
    for r in range(2 * max_passes):
        prev = part.clone()
        _lib.call("sg_partition_round", _lib.ptr(level.off), _lib.ptr(level.nbr), _lib.ptr(level.wt),
                  _lib.ptr(level.vw), n, g, int(cap), int(seed) & (2**64 - 1), r, _lib.ptr(part),
                  _lib.ptr(sizes), _lib.ptr(ws), _lib.ptr(moved), _lib.stream_ptr())
        nmoved = int(moved.item())
        new = level.cut(part) if nmoved else cut
        if new > cut:  # simultaneous moves of neighbours made it worse: undo
            part.copy_(prev)
            sizes = level.sizes(part, g)
            nmoved = 0
        else:
            cut = new
        if r % 2 == 1:
            history.append(cut)
        idle = idle + 1 if nmoved == 0 else 0
        if idle >= 2:
            break
    return part, history


def _refine_host(level, part, g, cap, max_passes):
    """Sequential refinement of a small level on the host (csrc/host.cpp)."""
    import ctypes as C
    import torch
    from paper_2303_13775_b200 import _lib
    p = part.cpu().numpy().astype(np.int32)
    off, nbr, wt, vw = (t.cpu().numpy() for t in (level.off, level.nbr, level.wt, level.vw))  # alive for the call
    cut = C.c_int64(0)
    _lib.call("sg_partition_refine_host", level.n, _lib.ptr(off), _lib.ptr(nbr), _lib.ptr(wt), _lib.ptr(vw),
              g, int(cap), int(max_passes), _lib.ptr(p), C.byref(cut))
    return torch.from_numpy(p).to(part.device)


# levels with at most this many vertices are refined sequentially on the host
# (a move there updates its neighbours' gains at once); larger ones by GPU rounds
HOST_REFINE_MAX = int(__import__("os").environ.get("SG_PART_HOST_REFINE", 1 << 18))


def _refine(level, part, g, cap, seed, max_passes):
    if level.n <= HOST_REFINE_MAX or int(level.sizes(part, g).max()) > cap:
        # (a level above the host threshold is repaired there only if it came out
        # over the cap: the GPU rounds never move a vertex into a full part)
        part = _refine_host(level, part, g, cap, max_passes)
    part, _ = _refine_device(level, part, g, cap, seed, max_passes)
    return part


def _coarse_partition(level, g, cap, seed, restarts=4):
    """Initial partition of the coarsest level on the host (csrc/host.cpp)."""
    import ctypes as C
    import torch
    from paper_2303_13775_b200 import _lib
    off = level.off.cpu().numpy()
    nbr = level.nbr.cpu().numpy()
    wt = level.wt.cpu().numpy()
    vw = level.vw.cpu().numpy()
    part = np.empty(level.n, dtype=np.int32)
    cut = C.c_int64(0)
    _lib.call("sg_partition_coarse_host", level.n, _lib.ptr(off), _lib.ptr(nbr), _lib.ptr(wt), _lib.ptr(vw), g,
              int(cap), int(seed) & (2**64 - 1), restarts, _lib.ptr(part), C.byref(cut))
    return torch.from_numpy(part).to(level.vw.device)


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
    level = _symmetric_level(graph)
    part = torch.from_numpy(np.asarray(assignment, dtype=np.int32)).cuda()
    part, hist = _refine_device(level, part, g, cap, seed, max_passes)
    return part.cpu().numpy().astype(np.int64), hist


def partition_graph(graph, g, balance_eps=0.05, seed=0, max_passes=10) -> PartitionMap:
    """Balanced k-way partition with a small edge cut (partition.py:298-349),
    multilevel on the GPU: coarsen by heavy-edge matching
    (sg_partition_match_round, then two-hop sibling matching of what is left
    unmatched, and contraction) until at most max(20g, 200) vertices remain
    (merged weight capped at n / 2g, partition.py:324-335), partition the
    coarsest level by greedy region growing + sequential refinement (best of 4
    restarts, csrc/host.cpp), then project back level by level with boundary
    refinement: sequential on the host for levels of <= HOST_REFINE_MAX
    vertices, then parallel GPU rounds (sg_partition_round). The contiguous-id
    map, refined the same way on the input graph, is kept instead when its cut
    is lower.
    Deterministic given `seed`; not the reference's exact assignment (its
    matching and refinement visit vertices sequentially), same contract:
    balanced within eps, comparable cut (tests/test_gpu_partition.py pins the
    cut against reference runs)."""
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
    levels = [_symmetric_level(graph)]
    cmaps = []
    coarse_target = max(20 * g, 200)
    wcap = max(2, n // (2 * g))
    import os
    two_hop = os.environ.get("SG_PART_TWO_HOP", "1") == "1"
    trace = os.environ.get("SG_PART_TRACE") == "1"
    while levels[-1].n > coarse_target:
        coarse, cmap = _coarsen(levels[-1], wcap, seed + 7919 * len(cmaps), two_hop=two_hop)
        if coarse.n > 0.95 * levels[-1].n:
            break  # matching stalled; coarser levels would not help
        levels.append(coarse)
        cmaps.append(cmap)
    part = _coarse_partition(levels[-1], g, cap, seed)
    if trace:
        print(f"[partition] levels {[lv.n for lv in levels]}, coarsest cut {levels[-1].cut(part)}")
    part = _refine(levels[-1], part, g, cap, seed, max_passes)
    for lvl in range(len(cmaps) - 1, -1, -1):
        part = part[cmaps[lvl]].contiguous()
        part = _refine(levels[lvl], part, g, cap, seed + lvl + 1, max_passes)
        if trace:
            print(f"[partition] level {lvl} (n {levels[lvl].n}): cut {levels[lvl].cut(part)}")
    # one more candidate: the contiguous-id map refined on the input graph (ids
    # often carry locality -- the benchmark generators plant their blocks by id
    # range); the lower cut wins, ties to the multilevel result
    base = levels[0]
    alt = ((torch.arange(n, dtype=torch.int64, device=part.device) * g) // n).to(torch.int32)
    alt = _refine(base, alt, g, cap, seed + 104729, max_passes)
    if int(base.sizes(alt, g).max()) <= cap and base.cut(alt) < base.cut(part):
        part = alt
        if trace:
            print(f"[partition] contiguous map refined: cut {base.cut(part)} (kept)")
    return PartitionMap(part.cpu().numpy().astype(np.int64), g, balance_eps)


def cut_size(graph, pm: PartitionMap) -> int:
    """Directed edges whose endpoints live on different devices (partition.py:352-355)."""
    import torch
    from paper_2303_13775_b200 import _lib
    ro = torch.from_numpy(np.asarray(graph.row_offsets, dtype=np.int64)).cuda()
    ci = torch.from_numpy(np.asarray(graph.col_indices, dtype=np.int32)).cuda()
    part = torch.from_numpy(pm.assignment.astype(np.int32)).cuda()
    out = torch.zeros(1, dtype=torch.int64, device=part.device)
    _lib.call("sg_partition_cut", _lib.ptr(ro), _lib.ptr(ci), int(graph.num_vertices), _lib.ptr(part),
              _lib.ptr(out), _lib.stream_ptr())
    return int(out.item())
