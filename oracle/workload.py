"""NumPy restatement of the benchmark WORKLOAD generators -- TEST / BENCH
INFRASTRUCTURE ONLY (imported by tests/ and by bench.py's reference arm).

The reference arm of bench.py must run without loading the product package
(its ctypes library), yet time the CPU reference on the very same workload
the GPU arm measures. This module regenerates that workload bit-identically
in plain NumPy / Python from the same counter-based hashes:

* `generate_powerlaw`  -- block-planted Chung-Lu power-law in-CSR (SURVEY §8(d)
  "Synthetic inputs"; the product's native generator, csrc/host.cpp
  sg_gen_powerlaw). Same hash counters, same inverse-CDF draws on the same
  float64 prefix sums, rows sorted by source id.
* `sample`             -- sample_minibatch semantics (reference
  sampling.py:118-177: self-edge first, up to fanout distinct in-neighbours by
  a partial Fisher-Yates, input self-loops and parallel edges dropped by first
  occurrence, new vertices appended in first-seen order so V^l prefixes
  V^(l-1)) with the counter-based draws of the product's native sampler
  (csrc/host.cpp sg_sampler_run) instead of NumPy's Generator stream.
* `epoch_batches`      -- reference sampling.py:199-204 (permutation + chunks).
* `synthetic_labels`, `synthetic_features` -- the counter-based label / U[0,1)
  feature generators (24-bit uniforms, exact in fp32 and fp64).

Pinned against the native implementations on small graphs by
tests/test_oracle_workload.py (bit-identical graphs, samples, labels and
features).
"""

from __future__ import annotations

import math

import numpy as np

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_GOLD = np.uint64(0x9E3779B97F4A7C15)
_K = np.uint64(0xD1B54A32D192ED03)
_MASK = (1 << 64) - 1


def mix64(x):
    """splitmix64 finaliser (csrc/rng.h sg_mix64), uint64 arrays (wrapping)."""
    with np.errstate(over="ignore"):
        x = np.asarray(x, dtype=np.uint64) + _GOLD
        x = (x ^ (x >> np.uint64(30))) * _M1
        x = (x ^ (x >> np.uint64(27))) * _M2
        return x ^ (x >> np.uint64(31))


def hash3(seed, a, b):
    """sg_hash3(seed, a, b) = mix64(mix64(mix64(seed) ^ a) ^ (b * K))."""
    s = mix64(np.uint64(int(seed) & _MASK))
    a = np.asarray(a, dtype=np.uint64)
    b = np.asarray(b, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return mix64(mix64(s ^ a) ^ (b * _K))


def uniform53(h):
    return (np.asarray(h, dtype=np.uint64) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def bounded(h, bound):
    """High 64 bits of h * bound for bound < 2^32 (Lemire multiply-shift)."""
    h = np.asarray(h, dtype=np.uint64)
    bound = np.asarray(bound, dtype=np.uint64)
    hi = h >> np.uint64(32)
    lo = h & np.uint64(0xFFFFFFFF)
    return (hi * bound + ((lo * bound) >> np.uint64(32))) >> np.uint64(32)


def _mix64_int(x):
    x = (x + 0x9E3779B97F4A7C15) & _MASK
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _MASK
    return x ^ (x >> 31)


# ---- graph --------------------------------------------------------------------

def _weights_prefix(n, gamma, seed):
    """C[v] = sum_{u<v} w_u with w_v = r_v^(-1/(gamma-1)), r_v = (A v + B) mod n + 1
    (a seeded relabelling permutation, gcd(A, n) = 1), summed sequentially."""
    A = (_mix64_int((int(seed) ^ 0xA5A5) & _MASK) % max(n, 1)) | 1
    while math.gcd(A, n) != 1:
        A += 2
    B = _mix64_int((int(seed) ^ 0x5A5A) & _MASK) % max(n, 1)
    v = np.arange(n, dtype=np.uint64)
    r = ((np.uint64(A) * v + np.uint64(B)) % np.uint64(n) + np.uint64(1)).astype(np.float64)
    w = np.power(r, -1.0 / (gamma - 1.0))
    C = np.empty(n + 1, dtype=np.float64)
    C[0] = 0.0
    np.cumsum(w, out=C[1:])
    return C


def _draw(C, u, lo, hi):
    """Inverse-CDF draw in [lo, hi): upper_bound of C[lo] + u (C[hi] - C[lo])."""
    t = C[lo] + u * (C[hi] - C[lo])
    x = np.searchsorted(C, t, side="right").astype(np.int64) - 1
    return np.minimum(np.maximum(x, lo), hi - 1)


def _edge_keys(C, n, blocks, p_local, seed, a, b):
    """dst * n + src of edges [a, b) (the per-edge hash counters e)."""
    e = np.arange(a, b, dtype=np.uint64)
    zero = np.zeros(b - a, dtype=np.int64)
    d = _draw(C, uniform53(hash3(seed, e, 0)), zero, zero + n)
    local = uniform53(hash3(seed, e, 1)) < p_local
    u = uniform53(hash3(seed, e, 2))
    blk = d * blocks // n
    lo = np.where(local, (blk * n + blocks - 1) // blocks, 0)
    hi = np.where(local, ((blk + 1) * n + blocks - 1) // blocks, n)
    s = _draw(C, u, lo, hi)
    return d * n + s


_POOL_STATE = {}


def _chunk_worker(args):
    a, b = args
    st = _POOL_STATE
    return _edge_keys(st["C"], st["n"], st["blocks"], st["p_local"], st["seed"], a, b)


def generate_powerlaw(n, m, *, blocks=64, p_local=0.92, gamma=2.1, seed=0, chunk=1 << 22, workers=1):
    """(row_offsets int64[n+1], col_indices int32[m]): the in-CSR of the
    block-planted Chung-Lu graph, each row's sources sorted ascending.
    workers > 1 draws the edge chunks in forked processes (counter-based
    draws: the result does not depend on the worker count)."""
    n, m = int(n), int(m)
    C = _weights_prefix(n, gamma, seed)
    keys = np.empty(m, dtype=np.int64)
    ranges = [(a, min(m, a + chunk)) for a in range(0, m, chunk)]
    if workers > 1 and len(ranges) > 1:
        import multiprocessing as mp
        _POOL_STATE.update(C=C, n=n, blocks=blocks, p_local=p_local, seed=seed)
        with mp.get_context("fork").Pool(min(workers, len(ranges))) as pool:
            for (a, b), k in zip(ranges, pool.imap(_chunk_worker, ranges)):
                keys[a:b] = k
        _POOL_STATE.clear()
    else:
        for a, b in ranges:
            keys[a:b] = _edge_keys(C, n, blocks, p_local, seed, a, b)
    keys.sort()
    dst = keys // n
    ro = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(dst, minlength=n), out=ro[1:])
    ci = (keys - dst * n).astype(np.int32)
    return ro, ci


def synthetic_labels(n, num_classes, seed):
    v = np.arange(int(n), dtype=np.uint64)
    return bounded(hash3(seed, v, 7), int(num_classes)).astype(np.int32)


def synthetic_features(row_ids, feat_dim, seed, dtype=np.float64):
    """U[0,1) with 24 random bits for rows `row_ids` (global ids)."""
    rid = np.asarray(row_ids, dtype=np.uint64)[:, None]
    c = np.arange(int(feat_dim), dtype=np.uint64)[None, :]
    return ((hash3(seed, rid, c) >> np.uint64(40)).astype(np.float64) * (1.0 / 16777216.0)).astype(dtype)


def epoch_batches(train_set, batch_size, rng):
    """Reference sampling.py:199-204."""
    perm = rng.permutation(np.asarray(train_set, dtype=np.int64))
    return [perm[i:i + batch_size] for i in range(0, len(perm), batch_size)]


# ---- sampler --------------------------------------------------------------------

def sample(ro, ci, targets, fanouts, seed):
    """(layer_vertices, layer_edges) of one mini-batch; see module docstring."""
    targets = np.asarray(targets, dtype=np.int64)
    if len(targets) == 0:
        raise ValueError("targets must be non-empty")
    if len(np.unique(targets)) != len(targets):
        raise ValueError("targets must be distinct")
    L = len(fanouts)
    layers = [None] * (L + 1)
    edges = [None] * L
    layers[L] = targets.copy()
    for l in range(L, 0, -1):
        cur = layers[l]
        nc = len(cur)
        f = max(0, int(fanouts[l - 1]))
        s0 = ro[cur]
        deg = ro[cur + 1] - s0
        k = np.minimum(f, deg)
        # draws of the partial Fisher-Yates for every (destination i, step j < k_i)
        part = np.flatnonzero(k < deg)
        r_all = {}
        if len(part) and f > 0:
            ii = np.repeat(part, k[part])
            jj = np.concatenate([np.arange(x) for x in k[part]]).astype(np.int64)
            h = hash3(seed, (np.uint64(l) << np.uint64(40)) ^ ii.astype(np.uint64), jj.astype(np.uint64))
            rr = jj + bounded(h, (deg[ii] - jj).astype(np.uint64)).astype(np.int64)
            starts = np.r_[0, np.cumsum(k[part])]
            for t, i in enumerate(part):
                r_all[int(i)] = rr[starts[t]:starts[t + 1]]
        pos_of = {int(v): i for i, v in enumerate(cur)}
        order = list(int(v) for v in cur)
        src, dst = [], []
        for i in range(nc):
            v = int(cur[i])
            src.append(i)
            dst.append(i)
            if k[i] <= 0:
                continue
            b = int(s0[i])
            m = int(deg[i])
            if k[i] >= m:
                cand = ci[b:b + m].tolist()
            else:
                swap = {}
                cand = []
                for j, r in enumerate(r_all[i].tolist()):
                    vj = swap.get(j, None)
                    vr = swap.get(r, None)
                    vj = int(ci[b + j]) if vj is None else vj
                    vr = int(ci[b + r]) if vr is None else vr
                    swap[r] = vj
                    swap[j] = vr
                    cand.append(vr)
            seen = []
            for u in cand:
                u = int(u)
                if u == v or u in seen:
                    continue
                seen.append(u)
                j = pos_of.get(u)
                if j is None:
                    j = len(order)
                    pos_of[u] = j
                    order.append(u)
                src.append(j)
                dst.append(i)
        layers[l - 1] = np.asarray(order, dtype=np.int64)
        edges[l - 1] = (np.asarray(src, dtype=np.int64), np.asarray(dst, dtype=np.int64))
    return layers, edges


def build_cache(ro, ci, assignment, g, capacity_fraction):
    """Reference partition.py:358-377: per device the highest (in + out)
    degree vertices of its partition, ties by lower id, ceil(frac * n) each;
    returns the sorted cached id lists."""
    n = len(ro) - 1
    cap = math.ceil(capacity_fraction * n - 1e-9)
    degree = np.diff(ro) + np.bincount(ci, minlength=n)
    out = []
    for d in range(g):
        ids = np.flatnonzero(np.asarray(assignment) == d)
        order = np.lexsort((ids, -degree[ids]))
        out.append(np.sort(ids[order][:cap]))
    return out
