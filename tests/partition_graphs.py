"""NumPy generators of the partitioner-quality graphs (test infrastructure;
shared by tests/test_gpu_partition.py and tests/golden/make_partition_golden.py)."""

import numpy as np


def reference_planted_edges(n, k, p_in, p_out, seed):
    """Restatement of reference graph.py:136-168 generate_planted_partition
    (contiguous-id blocks, each ordered pair u != v an edge with p_in inside a
    block and p_out across; the same Generator draws, row by row)."""
    rng = np.random.default_rng(seed)
    comm = np.arange(n, dtype=np.int64) // (n // k)
    src, dst = [], []
    for u in range(n):
        p_row = np.where(comm == comm[u], p_in, p_out)
        p_row[u] = 0.0
        hits = np.flatnonzero(rng.random(n) < p_row)
        src.append(np.full(len(hits), u, dtype=np.int64))
        dst.append(hits.astype(np.int64))
    return np.concatenate(src), np.concatenate(dst)


def permuted(n, src, dst, seed):
    perm = np.random.default_rng(seed).permutation(n)
    return perm[src], perm[dst]


def planted_blocks(n=20000, k=8, m=200000, p_local=0.9, seed=0):
    """k blocks with shuffled membership; a fraction p_local of the edges stays inside a block."""
    rng = np.random.default_rng(seed)
    blk = rng.integers(0, k, n)
    members = [np.flatnonzero(blk == b) for b in range(k)]
    dst = rng.integers(0, n, m)
    local = rng.random(m) < p_local
    src = rng.integers(0, n, m)
    for b in range(k):
        sel = local & (blk[dst] == b)
        src[sel] = members[b][rng.integers(0, len(members[b]), int(sel.sum()))]
    return src.astype(np.int64), dst.astype(np.int64)


def powerlaw_edges(n=50000, m=500000, seed=7):
    """Block-planted Chung-Lu power-law graph (oracle/workload.py, the bench generator family)."""
    from oracle.workload import generate_powerlaw
    ro, ci = generate_powerlaw(n, m, blocks=16, p_local=0.9, seed=seed)
    ro = np.asarray(ro, dtype=np.int64)
    dst = np.repeat(np.arange(n, dtype=np.int64), np.diff(ro))
    return np.asarray(ci, dtype=np.int64), dst
