"""Mini-batch samples and the native k-hop sampler.

MiniBatchSample mirrors splitgnn.sampling.MiniBatchSample (sampling.py:18-102):
layer_vertices[l] global ids of V^l (l = 0..L, V^l a positional prefix of
V^(l-1)), layer_edges[l-1] = (src_pos in V^(l-1), dst_pos in V^l).
sample_minibatch has the reference semantics (sampling.py:118-177) but runs in
native threaded C++ with a counter-based RNG; parity with the reference is
established on EXPORTED samples (same sample -> same split and same step).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from paper_2303_13775_b200 import _lib


@dataclass
class MiniBatchSample:
    num_layers: int
    layer_vertices: list
    layer_edges: list
    dst_grouped: bool | None = field(default=None, compare=False)
    pinned: object = field(default=None, compare=False, repr=False)

    @property
    def targets(self):
        return self.layer_vertices[self.num_layers]

    def vertices(self, l):
        return self.layer_vertices[l]

    def edges(self, l):
        return self.layer_edges[l - 1]

    def num_edges(self, l):
        return len(self.layer_edges[l - 1][0])

    @property
    def total_edges(self):
        return int(sum(len(s) for s, _ in self.layer_edges))

    def sizes(self):
        nV = [len(v) for v in self.layer_vertices]
        nE = [len(s) for s, _ in self.layer_edges]
        return nV, nE

    def is_dst_grouped(self) -> bool:
        """True when each destination's in-edges are contiguous in every layer
        (always the case for sampler output: edges are emitted per destination)."""
        if self.dst_grouped is None:
            ok = True
            for _, dst in self.layer_edges:
                dst = np.asarray(dst)
                if len(dst) > 1:
                    starts = np.flatnonzero(np.r_[True, dst[1:] != dst[:-1]])
                    if np.bincount(dst[starts]).max() > 1:  # a destination starts two runs
                        ok = False
                        break
            self.dst_grouped = ok
        return bool(self.dst_grouped)

    def edge_gid_triples(self) -> np.ndarray:
        """All edges as (layer, src_gid, dst_gid) rows (sampling.py:52-66)."""
        rows = []
        for l in range(1, len(self.layer_edges) + 1):
            src, dst = self.layer_edges[l - 1]
            rows.append(np.column_stack([np.full(len(src), l, dtype=np.int64),
                                         np.asarray(self.layer_vertices[l - 1], np.int64)[src],
                                         np.asarray(self.layer_vertices[l], np.int64)[dst]]))
        return np.concatenate(rows) if rows else np.empty((0, 3), dtype=np.int64)

    def packed(self):
        """(V, esrc, edst) int32 concatenations used by the device splitter."""
        V = np.concatenate([np.asarray(v, dtype=np.int32) for v in self.layer_vertices])
        src = np.concatenate([np.asarray(s, dtype=np.int32) for s, _ in self.layer_edges])
        dst = np.concatenate([np.asarray(d, dtype=np.int32) for _, d in self.layer_edges])
        return V, src, dst

    def validate(self, num_vertices=None):
        """sampling.py:68-90."""
        L = self.num_layers
        assert len(self.layer_vertices) == L + 1 and len(self.layer_edges) == L
        for ids in self.layer_vertices:
            ids = np.asarray(ids)
            assert len(np.unique(ids)) == len(ids), "duplicate vertex in a layer"
            if num_vertices is not None and len(ids):
                assert ids.min() >= 0 and ids.max() < num_vertices
        for l in range(1, L + 1):
            lo, hi = np.asarray(self.layer_vertices[l - 1]), np.asarray(self.layer_vertices[l])
            assert np.array_equal(lo[: len(hi)], hi), "V^(l) must prefix V^(l-1)"
            src, dst = (np.asarray(a, dtype=np.int64) for a in self.edges(l))
            assert len(src) == len(dst)
            if len(src):
                assert src.min() >= 0 and src.max() < len(lo)
                assert dst.min() >= 0 and dst.max() < len(hi)
            key = src * len(hi) + dst
            assert len(np.unique(key)) == len(key), "duplicate edge in a layer"
            diag = np.arange(len(hi), dtype=np.int64) * (len(hi) + 1)
            assert np.isin(diag, key).all(), "missing self-edge"


@dataclass
class PinnedArrays:
    """A native-sampler sample's arrays as one page-locked int32 buffer
    [int64 header of the sizes (S words) | V^0..V^L (VS) | E^l sources (ES) |
    E^l destinations (ES)]; the sample's arrays are views of it. vbound: every
    vertex id is < vbound (the sampled graph's vertex count)."""

    tensor: object
    base: int
    S: int
    VS: int
    ES: int
    vbound: int
    views: tuple = ()  # the sampler's array objects: V^0..V^L, then (src, dst) per layer
    RS: int = 0  # run starts after es (compact form; the dst lists are read-only views)

    @property
    def dma_words(self):
        """Words split_minibatch sends: [header | V | es | starts] in the
        compact form, else [header | V | es | ed]."""
        return self.S + self.VS + self.ES + (self.RS if self.RS else self.ES)

    def __reduce__(self):
        # the page-locked buffer and its address belong to this process: a
        # pickled (e.g. sent to another process) sample is packed instead
        return (_no_pinned, ())

    def intact(self, sample) -> bool:
        """The sample still holds the sampler's own array objects (views into
        this buffer; in-place edits travel with the buffer). A caller that
        replaced one gets the packing path instead."""
        lv, le = sample.layer_vertices, sample.layer_edges
        L = len(le)
        w = self.views
        if len(lv) != L + 1 or len(w) != 2 * L + 1 or self.tensor.data_ptr() != self.base:
            return False
        for l in range(L + 1):
            if lv[l] is not w[l]:
                return False
        for l in range(L):
            e = le[l]
            if e[0] is not w[L + 1 + l][0] or e[1] is not w[L + 1 + l][1]:
                return False
            if self.RS and e[1].flags.writeable:  # made writable again: may have been edited
                return False
        return True


def _no_pinned():
    return None


_CUDA = None


def _cuda_present():
    global _CUDA
    if _CUDA is None:
        import os
        try:
            import torch
            _CUDA = bool(torch.cuda.is_available()) and os.environ.get("SG_SAMPLE_PINNED", "1") != "0"
        except Exception:
            _CUDA = False
    return _CUDA


def _pinned_int32(n):
    """Page-locked int32 host tensor from torch's caching host allocator (a
    freed sample's buffer is reused; an async copy from it is tracked)."""
    import torch
    try:
        return torch.empty(max(int(n), 1), dtype=torch.int32, pin_memory=True)
    except RuntimeError:
        return None


def as_sample(obj) -> MiniBatchSample:
    """Accept a reference splitgnn MiniBatchSample (duck-typed) or ours."""
    if isinstance(obj, MiniBatchSample):
        return obj
    return MiniBatchSample(int(obj.num_layers), list(obj.layer_vertices), list(obj.layer_edges))


class NativeSampler:
    """Reusable native sampler bound to one graph (keeps O(n) scratch)."""

    def __init__(self, graph, threads=0, pinned=None):
        """pinned: write samples into page-locked host memory (default: when
        a GPU is present, SG_SAMPLE_PINNED=0 disables) so that split_minibatch
        DMAs them without a host copy."""
        self.graph = graph
        self.threads = int(threads)
        self.pinned = _cuda_present() if pinned is None else bool(pinned)
        self._h = _lib.load().sg_sampler_create(int(graph.num_vertices),
                                                _lib.ptr(graph.row_offsets),
                                                _lib.ptr(graph.col_indices))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._h = None
            try:
                _lib.load().sg_sampler_destroy(h)
            except TypeError:  # interpreter shutdown: module globals already cleared
                pass

    def sample(self, targets, fanouts, seed) -> MiniBatchSample:
        lib = _lib.load()
        targets = np.ascontiguousarray(np.asarray(targets, dtype=np.int64))
        fan = np.ascontiguousarray(np.asarray(list(fanouts), dtype=np.int32))
        L = len(fan)
        if L == 0:
            raise ValueError("fanouts must be non-empty")
        nV = np.zeros(L + 1, dtype=np.int64)
        nE = np.zeros(max(L, 1), dtype=np.int64)
        _lib.check(lib.sg_sampler_run(self._h, _lib.ptr(targets), len(targets), _lib.ptr(fan), L,
                                      int(seed) & (2**64 - 1), self.threads, _lib.ptr(nV),
                                      _lib.ptr(nE)), "sample_minibatch")
        VS, ES = int(nV.sum()), int(nE[:L].sum())
        RS = VS - int(nV[0])  # one run start per destination of layers 1..L
        S = 2 * (2 * L + 1)  # int64 header of the sizes, as in the capacity layout
        pin = _pinned_int32(S + VS + 2 * ES + RS) if self.pinned else None
        if pin is not None:
            # one DMA-ready buffer [header | V | es | run starts | ed]:
            # split_minibatch sends the prefix before ed as is (no host pack)
            # and the device rebuilds the destination lists from the starts
            buf = pin.numpy()
            buf[:S].view(np.int64)[:] = np.r_[nV, nE[:L]]
            V, es = buf[S:S + VS], buf[S + VS:S + VS + ES]
            starts, ed = buf[S + VS + ES:S + VS + ES + RS], buf[S + VS + ES + RS:]
            _lib.check(lib.sg_sampler_fetch_starts(self._h, _lib.ptr(V), _lib.ptr(es), _lib.ptr(ed),
                                                   _lib.ptr(starts)), "sampler_fetch")
        else:
            buf = np.empty(VS + 2 * ES, dtype=np.int32)
            V, es, ed = buf[:VS], buf[VS:VS + ES], buf[VS + ES:]
            _lib.check(lib.sg_sampler_fetch(self._h, _lib.ptr(V), _lib.ptr(es), _lib.ptr(ed)),
                       "sampler_fetch")
        vo = np.r_[0, np.cumsum(nV)]
        eo = np.r_[0, np.cumsum(nE[:L])]
        lv = [V[vo[l]:vo[l + 1]] for l in range(L + 1)]
        le = [(es[eo[l]:eo[l + 1]], ed[eo[l]:eo[l + 1]]) for l in range(L)]
        if pin is not None:
            for _, d in le:  # the device rebuilds these from the starts: no in-place edits
                d.flags.writeable = False
        smp = MiniBatchSample(L, lv, le, dst_grouped=True)
        if pin is not None:
            smp.pinned = PinnedArrays(pin, buf.ctypes.data, S, VS, ES, int(self.graph.num_vertices),
                                      tuple(lv) + tuple(le), RS)
        return smp


_SAMPLERS = {}


def sample_minibatch(graph, targets, fanouts, rng) -> MiniBatchSample:
    """k-hop in-neighbourhood sample (sampling.py:118-177). `rng` is a numpy
    Generator (one 63-bit draw seeds the native counter-based stream) or an int
    seed."""
    targets = np.asarray(targets, dtype=np.int64)
    if targets.size == 0:
        raise ValueError("targets must be non-empty")
    if len(np.unique(targets)) != len(targets):
        raise ValueError("targets must be distinct")
    if targets.min() < 0 or targets.max() >= graph.num_vertices:
        raise ValueError("target id out of range")
    if not list(fanouts):
        raise ValueError("fanouts must be non-empty")
    seed = int(rng) if isinstance(rng, (int, np.integer)) else int(rng.integers(0, 2**63 - 1))
    key = id(graph)
    s = _SAMPLERS.get(key)
    if s is None or s.graph is not graph:
        s = NativeSampler(graph)
        _SAMPLERS.clear()
        _SAMPLERS[key] = s
    return s.sample(targets, fanouts, seed)


def sample_microbatches(graph, targets, g, fanouts, rng) -> list:
    """Round-robin split of `targets` into g independently sampled batches
    (sampling.py:180-196): the data-parallel baseline's micro-batches."""
    targets = np.asarray(targets, dtype=np.int64)
    if g < 1:
        raise ValueError("g must be >= 1")
    if g == 1:
        return [sample_minibatch(graph, targets, fanouts, rng)]
    groups = [targets[i::g] for i in range(g)]
    if any(len(gr) == 0 for gr in groups):
        raise ValueError(f"cannot split {len(targets)} targets into {g} micro-batches")
    children = rng.spawn(g)
    return [sample_minibatch(graph, gr, fanouts, child) for gr, child in zip(groups, children)]


def epoch_batches(train_set, batch_size, rng) -> list:
    """Shuffle and chunk (sampling.py:199-204)."""
    if batch_size < 1:
        raise ValueError("batch_size must be >= 1")
    perm = rng.permutation(np.asarray(train_set, dtype=np.int64))
    return [perm[i:i + batch_size] for i in range(0, len(perm), batch_size)]


class GpuSampler:
    """sample_minibatch (sampling.py:118-177) on the GPU (csrc/sampler.cu)
    from a device-resident copy of the graph's in-CSR. Same semantics and the
    same counter-based RNG as the native host sampler, so for the same seed
    both produce the identical sample. `sample()` returns a host
    MiniBatchSample; `sample_into()` writes a packed sample straight into a
    StaticSample's device buffers (a captured step's inputs) with no host
    round trip."""

    def __init__(self, graph, device="cuda"):
        import torch
        self.graph = graph
        self.n = int(graph.num_vertices)
        self.dev = torch.device(device)
        self.ro = torch.from_numpy(np.asarray(graph.row_offsets, dtype=np.int64)).to(self.dev)
        self.ci = torch.from_numpy(np.asarray(graph.col_indices, dtype=np.int32)).to(self.dev)
        self._ws = None
        self._ws_key = None
        self.err = torch.zeros(1, dtype=torch.int32, device=self.dev)

    @staticmethod
    def bounds(n_targets, fanouts):
        """Fanout-derived capacities: |V^L| = B, |E^l| <= |V^l|(1+f), |V^{l-1}| <= |E^l|."""
        L = len(fanouts)
        nV = [0] * (L + 1)
        nE = [0] * L
        nV[L] = int(n_targets)
        for l in range(L, 0, -1):
            nE[l - 1] = nV[l] * (1 + int(fanouts[l - 1]))
            nV[l - 1] = nE[l - 1]
        return nV, nE

    def _scratch(self, max_dst, max_edges, fmax):
        import torch
        key = (int(max_dst), int(max_edges), int(fmax))
        if self._ws is None or self._ws_key is None or any(a > b for a, b in zip(key, self._ws_key)):
            nbytes = int(_lib.load().sg_gpu_sampler_ws_bytes(self.n, key[0], key[1], key[2]))
            self._ws = torch.empty(nbytes, dtype=torch.uint8, device=self.dev)
            _lib.call("sg_gpu_sampler_ws_init", _lib.ptr(self._ws), self.n, self._ws.numel(), _lib.stream_ptr())
            self._ws_key = key
        return self._ws

    def sample_into(self, targets_dev, fanouts, seed, V, esrc, edst, sizes, voff, eoff, seed_dev=None):
        """Launch the sampler (current stream) into packed device buffers with
        capacity offsets voff (L+2) / eoff (L+1); sizes: device int64[2L+1].
        seed_dev (device uint64[1]) replaces `seed` when given (graph replays)."""
        L = len(fanouts)
        fan = np.asarray(fanouts, dtype=np.int32)
        if fan.min(initial=0) < 0 or fan.max(initial=0) > 64:
            raise ValueError("fanouts must be in [0, 64] for the GPU sampler")
        cap_v = np.diff(np.asarray(voff, dtype=np.int64))
        cap_e = np.diff(np.asarray(eoff, dtype=np.int64))
        max_dst = int(cap_v.max())
        max_edges = int(max(cap_e.max(), 1))
        ws = self._scratch(max_dst, max_edges, max(int(fan.max(initial=1)), 1))
        vo = np.ascontiguousarray(voff, dtype=np.int64)
        eo = np.ascontiguousarray(eoff, dtype=np.int64)
        _lib.call("sg_gpu_sample", _lib.ptr(self.ro), _lib.ptr(self.ci), self.n, _lib.ptr(targets_dev),
                  int(targets_dev.numel()), _lib.ptr(fan), L, int(seed) & (2**64 - 1), _lib.ptr(seed_dev),
                  int(ws.numel()), _lib.ptr(vo), _lib.ptr(eo), max_dst, max_edges, _lib.ptr(V), _lib.ptr(esrc), _lib.ptr(edst),
                  _lib.ptr(sizes), _lib.ptr(ws), _lib.ptr(self.err), _lib.stream_ptr())

    def sample(self, targets, fanouts, seed) -> MiniBatchSample:
        import torch
        targets = np.asarray(targets, dtype=np.int64)
        if targets.size == 0:
            raise ValueError("targets must be non-empty")
        if len(np.unique(targets)) != len(targets):
            raise ValueError("targets must be distinct")
        if targets.min() < 0 or targets.max() >= self.n:
            raise ValueError("target id out of range")
        if not list(fanouts):
            raise ValueError("fanouts must be non-empty")
        nV, nE = self.bounds(len(targets), fanouts)
        voff = np.r_[0, np.cumsum(nV)].astype(np.int64)
        eoff = np.r_[0, np.cumsum(nE)].astype(np.int64)
        V = torch.empty(int(voff[-1]), dtype=torch.int32, device=self.dev)
        es = torch.empty(max(int(eoff[-1]), 1), dtype=torch.int32, device=self.dev)
        ed = torch.empty_like(es)
        sizes = torch.zeros(2 * len(fanouts) + 1, dtype=torch.int64, device=self.dev)
        t = torch.from_numpy(targets).to(self.dev)
        self.sample_into(t, fanouts, seed, V, es, ed, sizes, voff, eoff)
        if int(self.err.item()):
            raise RuntimeError("GPU sampler: capacity exceeded or target out of range")
        sz = sizes.cpu().numpy()
        L = len(fanouts)
        Vh, esh, edh = V.cpu().numpy(), es.cpu().numpy(), ed.cpu().numpy()
        layers = [Vh[voff[l]:voff[l] + sz[l]].astype(np.int64) for l in range(L + 1)]
        edges = [(esh[eoff[l]:eoff[l] + sz[L + 1 + l]].astype(np.int64),
                  edh[eoff[l]:eoff[l] + sz[L + 1 + l]].astype(np.int64)) for l in range(L)]
        return MiniBatchSample(L, layers, edges)
