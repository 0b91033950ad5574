"""CPU tests of the native library's host side: the C ABI loads and exports
every entry point include/splitgnn_b200.h declares, struct layouts agree,
and the host-native sampler / generator keep the reference semantics
(sampling.py:105-177). No GPU compute is called here."""

import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "splitgnn_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2303_13775_b200 import _lib
    lib = _lib.load()
    syms = _declared_symbols()
    assert len(syms) > 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # the ctypes binding covers every declared entry point
    assert not (set(syms) - set(_lib.EXPORTED)), sorted(set(syms) - set(_lib.EXPORTED))


def test_ctypes_signatures_match_header_arity():
    """Every ctypes binding in _lib._SIGS takes as many arguments as the header
    declaration (a stale binding fails only at call time, on a GPU box)."""
    from paper_2303_13775_b200 import _lib
    text = open(os.path.join(ROOT, "include", "splitgnn_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    decl = {}
    for m in re.finditer(r"\b(sg_[a-z0-9_]+)\s*\(([^;{]*?)\)\s*;", text, flags=re.S):
        params = m.group(2).strip()
        decl[m.group(1)] = 0 if params in ("", "void") else params.count(",") + 1
    bad = {k: (decl[k], len(args)) for k, (_, args) in _lib._SIGS.items() if k in decl and decl[k] != len(args)}
    assert not bad, bad


def test_struct_sizes_match_abi():
    from paper_2303_13775_b200 import _lib
    sizes = np.zeros(2, dtype=np.int64)
    _lib.load().sg_struct_sizes(sizes.ctypes.data)
    assert sizes.tolist() == [C.sizeof(_lib.SgMeta), C.sizeof(_lib.SgSplitLayout)]


def test_split_layout_is_aligned_and_bounded():
    from paper_2303_13775_b200 import _lib
    lay = _lib.SgSplitLayout()
    nV = (C.c_int64 * 4)(5000, 900, 200, 64)
    nE = (C.c_int64 * 3)(8000, 1500, 300)
    _lib.check(_lib.load().sg_split_layout(3, 4, nV, nE, 100000, C.byref(lay)))
    offs = [getattr(lay, n) for n, _ in _lib.SgSplitLayout._fields_ if n.startswith("o_")]
    assert all(o % 256 == 0 for o in offs)
    assert max(offs) < lay.total_bytes
    assert lay.nPtot == min(1500, 3 * 200) + min(300, 3 * 64) + min(8000, 3 * 900)
    with pytest.raises(ValueError):
        _lib.check(_lib.load().sg_split_layout(3, 17, nV, nE, 100000, C.byref(lay)))


def _graph():
    import paper_2303_13775_b200 as sg
    return sg.generate_powerlaw(20000, 200000, blocks=16, p_local=0.8, seed=5, threads=4)


def test_generator_deterministic_across_threads():
    import paper_2303_13775_b200 as sg
    a = sg.generate_powerlaw(5000, 40000, seed=3, threads=1)
    b = sg.generate_powerlaw(5000, 40000, seed=3, threads=7)
    assert np.array_equal(a.row_offsets, b.row_offsets)
    assert np.array_equal(a.col_indices, b.col_indices)
    assert a.num_edges == 40000
    # power law: a hub far above the mean in-degree
    assert a.in_degrees().max() > 20 * a.in_degrees().mean()


def test_sampler_reference_semantics():
    import paper_2303_13775_b200 as sg
    g = _graph()
    rng = np.random.default_rng(0)
    targets = rng.choice(g.num_vertices, 300, replace=False)
    s = sg.NativeSampler(g, threads=4).sample(targets, [7, 5, 3], seed=11)
    s.validate(g.num_vertices)  # prefix property, unique edges, self-edges (sampling.py:68-90)
    fan = [7, 5, 3]
    for l in range(1, 4):
        src, dst = (np.asarray(a) for a in s.edges(l))
        V_lo, V_hi = np.asarray(s.vertices(l - 1)), np.asarray(s.vertices(l))
        # destinations in order, each starting with its self-edge
        assert np.all(np.diff(dst) >= 0)
        first = np.r_[True, dst[1:] != dst[:-1]]
        assert np.array_equal(src[first], dst[first])
        deg = np.bincount(dst, minlength=len(V_hi))
        indeg = g.in_degrees()[V_hi]
        assert np.all(deg <= 1 + fan[l - 1])
        assert np.all(deg <= 1 + indeg)
        # every sampled neighbour is a real in-neighbour
        for i in rng.choice(len(src), 50):
            u, v = V_lo[src[i]], V_hi[dst[i]]
            if u != v:
                nb = g.col_indices[g.row_offsets[v]:g.row_offsets[v + 1]]
                assert u in nb
        # vertices with deg <= fanout take every distinct neighbour
        small = np.flatnonzero((indeg > 0) & (indeg <= fan[l - 1]))[:20]
        for i in small:
            v = V_hi[i]
            nb = set(g.col_indices[g.row_offsets[v]:g.row_offsets[v + 1]].tolist()) - {int(v)}
            assert deg[i] - 1 == len(nb)


def test_sampler_deterministic_and_thread_independent():
    import paper_2303_13775_b200 as sg
    g = _graph()
    t = np.arange(0, 20000, 37)
    a = sg.NativeSampler(g, threads=1).sample(t, [6, 4], seed=3)
    b = sg.NativeSampler(g, threads=8).sample(t, [6, 4], seed=3)
    c = sg.NativeSampler(g, threads=8).sample(t, [6, 4], seed=4)
    for x, y in zip(a.layer_vertices, b.layer_vertices):
        assert np.array_equal(x, y)
    for (xs, xd), (ys, yd) in zip(a.layer_edges, b.layer_edges):
        assert np.array_equal(xs, ys) and np.array_equal(xd, yd)
    assert not all(np.array_equal(x, y) for x, y in zip(a.layer_vertices, c.layer_vertices))


def test_sampler_errors_match_reference_messages():  # sampling.py:128-136
    import paper_2303_13775_b200 as sg
    g = _graph()
    rng = np.random.default_rng(0)
    with pytest.raises(ValueError, match="non-empty"):
        sg.sample_minibatch(g, [], [2], rng)
    with pytest.raises(ValueError, match="distinct"):
        sg.sample_minibatch(g, [1, 1], [2], rng)
    with pytest.raises(ValueError, match="out of range"):
        sg.sample_minibatch(g, [g.num_vertices], [2], rng)
    with pytest.raises(ValueError, match="fanouts"):
        sg.sample_minibatch(g, [1], [], rng)


def test_sampler_zero_fanout_and_path_graph():  # test_sampling.py:20-43
    import paper_2303_13775_b200 as sg
    # path 0 -> 1 -> 2 -> 3 (in-CSR: in-neighbour of v is v-1)
    g = sg.from_edges(4, [0, 1, 2], [1, 2, 3])
    s = sg.sample_minibatch(g, [3], [1, 1], np.random.default_rng(0))
    assert [v.tolist() for v in s.layer_vertices] == [[3, 2, 1], [3, 2], [3]]
    z = sg.sample_minibatch(g, [3, 1], [0], np.random.default_rng(0))
    assert z.layer_vertices[0].tolist() == [3, 1]
    assert np.asarray(z.edges(1)[0]).tolist() == [0, 1]


def test_synthetic_features_host_values():
    import paper_2303_13775_b200 as sg
    a = sg.synthetic_features(10, 7, seed=3)
    b = sg.synthetic_features(0, 7, seed=3, row_ids=np.array([4, 9]))
    assert np.array_equal(a[[4, 9]], b)
    assert a.dtype == np.float32 and a.min() >= 0 and a.max() < 1
    # 24-bit values: exact in fp32 and fp64
    assert np.array_equal((a * 2**24).astype(np.float64), np.round(a.astype(np.float64) * 2**24))


def test_init_params_matches_oracle_draws():
    import paper_2303_13775_b200 as sg
    from oracle.model_oracle import glorot_params
    for kind in ("graphsage", "gat"):
        p = sg.init_params(kind, 12, 8, 5, 3, seed=9).tensors()
        q = glorot_params(kind, 12, 8, 5, 3, seed=9)
        assert list(p) == list(q)
        for k in p:
            assert np.array_equal(p[k], q[k])


def _sym_csr(n, edges):
    import collections
    w = collections.Counter()
    for u, v in edges:
        if u != v:
            w[(u, v)] += 1
            w[(v, u)] += 1
    keys = sorted(w)
    off = np.zeros(n + 1, dtype=np.int64)
    for u, _ in keys:
        off[u + 1] += 1
    off = np.cumsum(off)
    nbr = np.array([v for _, v in keys], dtype=np.int32)
    wt = np.array([w[k] for k in keys], dtype=np.int32)
    return off, nbr, wt


@pytest.mark.parametrize("perm", [[0, 1, 2, 3, 4, 5], [0, 3, 1, 4, 2, 5], [5, 2, 4, 0, 3, 1]])
def test_coarse_partition_bridge_graph(perm):
    """csrc/host.cpp sg_partition_coarse_host (the multilevel partitioner's
    coarsest level): two bidirected 3-cliques joined by one arc, eps 0 -> the
    exhaustive optimum (cut 1, reference test_partition.py:49-58), whatever the
    vertex numbering."""
    import ctypes as C
    import itertools
    from paper_2303_13775_b200 import _lib
    p = np.array(perm)
    edges = [(p[u], p[v]) for blk in ([0, 1, 2], [3, 4, 5]) for u, v in itertools.permutations(blk, 2)]
    edges.append((p[2], p[3]))
    off, nbr, wt = _sym_csr(6, edges)
    vw = np.ones(6, dtype=np.int32)
    part = np.empty(6, dtype=np.int32)
    cut = C.c_int64(0)
    _lib.call("sg_partition_coarse_host", 6, _lib.ptr(off), _lib.ptr(nbr), _lib.ptr(wt), _lib.ptr(vw), 2, 3,
              0, 4, _lib.ptr(part), C.byref(cut))
    assert cut.value == 1
    assert np.bincount(part, minlength=2).tolist() == [3, 3]
    assert len(set(part[p[:3]])) == 1 and len(set(part[p[3:]])) == 1


def test_coarse_partition_weighted_balance():
    """Vertex weights count toward the cap; a ring of 40 weighted vertices
    splits into 4 contiguous arcs within the cap, deterministically."""
    import ctypes as C
    from paper_2303_13775_b200 import _lib
    n = 40
    off, nbr, wt = _sym_csr(n, [(i, (i + 1) % n) for i in range(n)])
    vw = (1 + (np.arange(n) % 3)).astype(np.int32)
    cap = int(np.ceil(vw.sum() / 4 * 1.1))
    outs = []
    for _ in range(2):
        part = np.empty(n, dtype=np.int32)
        cut = C.c_int64(0)
        _lib.call("sg_partition_coarse_host", n, _lib.ptr(off), _lib.ptr(nbr), _lib.ptr(wt), _lib.ptr(vw), 4, cap,
                  9, 4, _lib.ptr(part), C.byref(cut))
        sizes = np.bincount(part, weights=vw, minlength=4)
        assert sizes.max() <= cap
        assert cut.value <= 6  # 4 arcs is optimal on a ring; allow a little for the heuristic
        outs.append(part.copy())
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
def test_pack_sample_matches_numpy_layout(dtype):
    """sg_pack_sample (split_minibatch's native staging) writes the captured-step
    layout: int64 size header, V^l at the capacity offsets, then sources and
    destinations per layer -- for int32 and int64 sample arrays."""
    from paper_2303_13775_b200.sampling import MiniBatchSample
    from paper_2303_13775_b200.scheduler import PackGeometry
    rng = np.random.default_rng(0)
    nV = [50000, 7000, 900, 100]
    nE = [70000, 9000, 1000]
    V = [rng.integers(0, 1 << 30, k).astype(dtype) for k in nV]
    E = [(rng.integers(0, nV[l], nE[l]).astype(dtype), np.sort(rng.integers(0, nV[l + 1], nE[l])).astype(dtype))
         for l in range(3)]
    smp = MiniBatchSample(3, V, E, dst_grouped=True)
    geo = PackGeometry.for_sizes(nV, nE, scope=("test", dtype))
    assert all(c >= x for c, x in zip(geo.cap_nV, nV)) and all(c >= x for c, x in zip(geo.cap_nE, nE))
    out = np.full(geo.words, -7, dtype=np.int32)
    used = geo.pack(smp, out)
    assert out[:geo.S].view(np.int64).tolist() == nV + nE
    for l in range(4):
        o = geo.o_V + geo.voff[l]
        assert np.array_equal(out[o:o + nV[l]], V[l].astype(np.int32))
    for l in range(3):
        o = geo.eoff[l]
        assert np.array_equal(out[geo.o_es + o:geo.o_es + o + nE[l]], E[l][0].astype(np.int32))
        assert np.array_equal(out[geo.o_ed + o:geo.o_ed + o + nE[l]], E[l][1].astype(np.int32))
    assert used == geo.o_ed + geo.eoff[2] + nE[2]
    allv = np.concatenate(V)
    assert geo.last_vrange == (int(allv.min()), int(allv.max()))  # split_minibatch's range check
    # a smaller sample keeps the geometry (one cached graph serves both); a larger one grows it
    assert PackGeometry.for_sizes([x // 2 for x in nV], [x // 2 for x in nE], scope=("test", dtype)) is geo
    big = PackGeometry.for_sizes([2 * x for x in nV], nE, scope=("test", dtype))
    assert big is not geo and all(b >= c for b, c in zip(big.cap_nV, geo.cap_nV))


@pytest.mark.parametrize("g", [1, 3])
def test_host_sum_sgd_matches_fma_formula(g):
    """allreduce_and_step's host side (sg_host_params_gather + sg_host_sum_sgd,
    engine.py:633-647): the snapshot is the fp32 flattening, the sum runs in
    device order in fp32, and p <- fp32(p - scale * total) with the product
    exact (fp64) -- bit-exact against that formula in numpy, for fp64 and fp32
    parameter arrays; nothing is written when the parameters changed."""
    import copy
    import paper_2303_13775_b200 as sg
    from paper_2303_13775_b200 import engine
    params = sg.init_params("graphsage", 20, 8, 5, 2, seed=1)
    params.w_cls = params.w_cls.astype(np.float32)  # mixed element types
    tab = engine._param_table(params)
    assert tab is not None
    snap = engine._host_flat(params)
    np.testing.assert_array_equal(snap, np.concatenate([np.ravel(v) for v in params.tensors().values()])
                                  .astype(np.float32))
    rng = np.random.default_rng(0)
    grads = [rng.standard_normal(tab.n + 1).astype(np.float32) for _ in range(g)]
    total = np.empty(tab.n, np.float32)
    gp = (C.c_void_p * g)(*[h.ctypes.data for h in grads])
    scale = float(np.float32(0.37 / 64))
    before = copy.deepcopy(params)
    from paper_2303_13775_b200 import _lib
    _lib.call("sg_host_sum_sgd", tab.k, tab.a_ptrs, tab.a_sizes, tab.a_eb, snap.ctypes.data, gp, g, tab.n,
              scale, total.ctypes.data, tab.a_applied)
    assert tab.applied[0] == 1
    want_t = grads[0][:tab.n].copy()
    for h in grads[1:]:
        want_t += h[:tab.n]
    np.testing.assert_array_equal(total, want_t)
    want = (snap.astype(np.float64) - scale * want_t.astype(np.float64)).astype(np.float32)
    np.testing.assert_array_equal(engine._host_flat(params), want)
    for (k, a), b in zip(params.tensors().items(), before.tensors().values()):
        assert a.dtype == b.dtype, k
    # parameters changed since the snapshot: untouched, applied = 0
    cur = engine._host_flat(params)
    _lib.call("sg_host_sum_sgd", tab.k, tab.a_ptrs, tab.a_sizes, tab.a_eb, snap.ctypes.data, gp, g, tab.n,
              scale, total.ctypes.data, tab.a_applied)
    assert tab.applied[0] == 0
    np.testing.assert_array_equal(engine._host_flat(params), cur)
    # a replaced array rebuilds the table
    params.b_cls = params.b_cls.copy()
    assert engine._param_table(params) is not tab


def test_pinned_sample_does_not_survive_pickling():
    """A sample's page-locked buffer (PinnedArrays) is process-local: pickling
    the sample drops it, so split_minibatch packs the unpickled copy instead
    of DMAing from a stale address."""
    import pickle
    from paper_2303_13775_b200.sampling import MiniBatchSample, PinnedArrays
    buf = np.zeros(64, dtype=np.int32)
    lv = [buf[2:6], buf[6:8]]
    le = [(buf[8:10], buf[10:12])]
    smp = MiniBatchSample(1, lv, le, dst_grouped=True,
                          pinned=PinnedArrays(None, buf.ctypes.data, 2, 6, 2, 100, tuple(lv) + tuple(le)))
    back = pickle.loads(pickle.dumps(smp))
    assert back.pinned is None
    np.testing.assert_array_equal(back.layer_vertices[0], lv[0])


def test_sampler_fetch_starts_are_run_starts():
    """sg_sampler_fetch_starts (the compact form split_minibatch DMAs): the
    same V / es / ed as sg_sampler_fetch, and per layer one start per
    destination = the first index of its run in the ascending destination list."""
    import paper_2303_13775_b200 as sg
    from paper_2303_13775_b200 import _lib
    g = _graph()
    smp = sg.NativeSampler(g, threads=4, pinned=False)
    ref = smp.sample(np.arange(0, 20000, 41), [6, 4, 3], seed=5)
    nV, nE = ref.sizes()
    V = np.empty(sum(nV), np.int32)
    es = np.empty(sum(nE), np.int32)
    ed = np.empty(sum(nE), np.int32)
    st = np.full(sum(nV[1:]), -1, np.int32)
    _lib.check(_lib.load().sg_sampler_fetch_starts(smp._h, V.ctypes.data, es.ctypes.data, ed.ctypes.data,
                                                   st.ctypes.data))
    np.testing.assert_array_equal(V, np.concatenate(ref.layer_vertices))
    np.testing.assert_array_equal(es, np.concatenate([a for a, _ in ref.layer_edges]))
    np.testing.assert_array_equal(ed, np.concatenate([b for _, b in ref.layer_edges]))
    o = 0
    for l in range(1, len(nV)):
        d = ref.layer_edges[l - 1][1]
        assert np.all(np.diff(d) >= 0)
        np.testing.assert_array_equal(st[o:o + nV[l]], np.searchsorted(d, np.arange(nV[l]), side="left"))
        o += nV[l]
