"""GAT layers of the split step (engine.py:280-552) on the sm_100a kernels.

Five exchange rounds per layer instead of the reference's ten (gat.cu header):
forward  from_owner t, to_owner (U, m, s), from_owner (m, den);
backward from_owner (d_num, c), to_owner dt.
The peer-bytes metering of the API keeps the reference's formula; the bytes
actually moved are reported separately as wire bytes.
"""

from __future__ import annotations

import torch

from paper_2303_13775_b200 import _lib




def _f32(n, *shape, device):
    return torch.empty((max(int(n), 1),) + tuple(shape), dtype=torch.float32, device=device)


def _r4(x):
    return (int(x) + 3) // 4 * 4


def _hs(H):
    """Trailing head dimension (omitted for one head: reference shapes)."""
    return (H,) if H > 1 else ()


def _from_owner(step, l, rows, width):
    """Owner rows (global owned index) -> holders' pair-layout rows."""
    ds = step.ds
    P = ds.pair_bound(l)
    out = _f32(P, width, device=step.dev)
    if step.g > 1 and P > 0:
        send = step._xbuf(P, width)
        st = _lib.stream_ptr()
        for d in step.devices:
            _lib.call("sg_pack_from_owner", _lib.ptr(ds.ws), ds.lay, l, d, _lib.ptr(rows), width,
                      _lib.ptr(send), width, step.n_recv(l, d), st)
        step.transport.from_owner(ds, l, send, out, width)
        if step.meta is not None:
            step.wire_bytes += int(step.meta.npairs[l]) * width * 4
    return out


def _wgrad_dst_ok(step):
    """Layer 1 runs the destination-centric weight gradient (sg_gat_wgrad_dst):
    D = 64, heads in {1, 2, 4}, w % 4 == 0, w <= 128; SG_GAT_WGRAD_DST=0 turns
    it off (then k_gat_bwd_src + the weight-gradient kernel, as at every other layer)."""
    import os
    if os.environ.get("SG_GAT_WGRAD_DST", "1") != "1" or step.L < 1:
        return False
    w, dout = step.p.layer_dims(0)
    return dout == 64 and step.p.heads_of(0) in (1, 2, 4) and w % 4 == 0 and w <= 128


def _csr_lmin(step):
    """Lowest layer whose backward needs the CSR by source row."""
    return 2 if _wgrad_dst_ok(step) else 1


def gat_forward(step):
    if getattr(step.f, "padded", False):
        raise ValueError("the GAT kernels read unpadded feature rows (FeatureStore pad_rows=False)")
    ds, p = step.ds, step.p
    st = _lib.stream_ptr()
    slope = float(p.leaky_slope)
    with step.phase("layer0"):
        step.layer0()
    dperm = step._dst_perm()
    step._launch_src_csr_async(_csr_lmin(step))
    dp_ptr = (lambda d: _lib.ptr(dperm[d][0])) if dperm is not None else (lambda d: None)
    nEtot = int(ds.lay.nEtot)
    step.h[0] = step.f.table
    for l in range(1, step.L + 1):
        w, dout = p.layer_dims(l - 1)
        final = int(l == step.L)
        h_prev, src_row = (step.f.table, step.src_row0) if l == 1 else (step.h[l - 1], None)
        nVp, nV, P = ds.nV[l - 1], ds.nV[l], ds.pair_bound(l)
        W, a_s, a_d = (p.view(f"layer{l-1}.{k}") for k in ("w", "a_src", "a_dst"))
        H = p.heads_of(l - 1)
        z = _f32(nVp, dout, device=step.dev)
        s = _f32(nVp, *_hs(H), device=step.dev)
        t = _f32(nV, *_hs(H), device=step.dev)
        with step.phase(f"project{l}"):
            if l == 1:
                step._ev("roof1_start")
            for d in step.devices:
                _lib.call("sg_gat_project", _lib.ptr(ds.ws), ds.lay, l, d, _lib.ptr(h_prev), _lib.ptr(src_row),
                          w, dout, H, _lib.ptr(W), _lib.ptr(a_s), _lib.ptr(a_d), _lib.ptr(z), _lib.ptr(s),
                          _lib.ptr(t), step.n_own(l - 1, d), st)
            if l == 1:
                step._ev("roof1_end")
        t_recv = _from_owner(step, l, t, H)
        SW = _r4(dout + 2 * H)
        send = _f32(P, SW, device=step.dev)
        recv = step._xbuf(P, SW)
        pre_e = _f32(nEtot, *_hs(H), device=step.dev)
        if step.g == 1:
            # one device: the owner combine and alpha ride on the aggregation epilogue
            md = _f32(nV, 2 * H, device=step.dev)
            num = _f32(nV, dout, device=step.dev)
            h = _f32(nV, dout, device=step.dev)
            alpha = _f32(nEtot, *_hs(H), device=step.dev)
            with step.phase(f"agg{l}"):
                step._ev(f"agg{l}_start")
                _lib.call("sg_gat_agg_fused", _lib.ptr(ds.ws), ds.lay, l, dout, H, slope, _lib.ptr(z), _lib.ptr(s),
                          _lib.ptr(t), dp_ptr(0), _lib.ptr(pre_e), final, _lib.ptr(md), _lib.ptr(num), _lib.ptr(h),
                          _lib.ptr(alpha), step.n_rows(l, 0), st)
                step._ev(f"agg{l}_end")
            step.h[l] = h
            step.keep[l] = dict(z=z, s=s, num=num, md=md, alpha=alpha, pre_e=pre_e)
            continue
        loc_m = _f32(nV, *_hs(H), device=step.dev)
        loc_s = _f32(nV, *_hs(H), device=step.dev)
        loc_U = _f32(nV, dout, device=step.dev)
        with step.phase(f"agg{l}"):
            step._ev(f"agg{l}_start")
            for d in step.devices:
                _lib.call("sg_gat_agg", _lib.ptr(ds.ws), ds.lay, l, d, dout, H, slope, _lib.ptr(z),
                          _lib.ptr(s), _lib.ptr(t), _lib.ptr(t_recv), dp_ptr(d), _lib.ptr(pre_e),
                          _lib.ptr(loc_m), _lib.ptr(loc_s), _lib.ptr(loc_U), _lib.ptr(send), SW,
                          step.n_rows(l, d), st)
            step._ev(f"agg{l}_end")
        if step.g > 1 and P > 0:
            step.transport.to_owner(ds, l, send, recv, SW)
            if step.meta is not None:
                step.wire_bytes += int(step.meta.npairs[l]) * SW * 4
        md = _f32(nV, 2 * H, device=step.dev)
        num = _f32(nV, dout, device=step.dev)
        h = _f32(nV, dout, device=step.dev)
        with step.phase(f"combine{l}"):
            for d in step.devices:
                _lib.call("sg_gat_combine", _lib.ptr(ds.ws), ds.lay, l, d, dout, H, _lib.ptr(loc_m),
                          _lib.ptr(loc_s), _lib.ptr(loc_U), _lib.ptr(recv), SW, final, _lib.ptr(md), _lib.ptr(num),
                          _lib.ptr(h), step.n_own(l, d), st)
        md_recv = _from_owner(step, l, md, 2 * H)
        alpha = _f32(nEtot, *_hs(H), device=step.dev)
        with step.phase(f"alpha{l}"):
            for d in step.devices:
                ne = int(step.meta.n_edge[l - 1][d]) if step.meta is not None else ds.nE[l - 1]
                _lib.call("sg_gat_alpha", _lib.ptr(ds.ws), ds.lay, l, d, H, slope, _lib.ptr(pre_e), _lib.ptr(md),
                          _lib.ptr(md_recv), _lib.ptr(alpha), ne, st)
        step.h[l] = h
        step.keep[l] = dict(z=z, s=s, num=num, md=md, alpha=alpha, pre_e=pre_e)


def gat_backward(step):
    ds, p = step.ds, step.p
    st = _lib.stream_ptr()
    slope = float(p.leaky_slope)
    dperm = step._dst_perm()
    dp_ptr = (lambda d: _lib.ptr(dperm[d][0])) if dperm is not None else (lambda d: None)
    nEtot = int(ds.lay.nEtot)
    with step.phase("src_csr_join"):
        csr, kb = step._join_src_csr(_csr_lmin(step))
    d_h = step.d_h
    from paper_2303_13775_b200.engine import TSPMM_MIN_EDGES, _nblocks
    for l in range(step.L, 0, -1):
        w, dout = p.layer_dims(l - 1)
        final = int(l == step.L)
        keep = step.keep[l]
        h_prev, src_row = (step.f.table, step.src_row0) if l == 1 else (step.h[l - 1], None)
        nVp, nV, P = ds.nV[l - 1], ds.nV[l], ds.pair_bound(l)
        W, a_s, a_d = (p.view(f"layer{l-1}.{k}") for k in ("w", "a_src", "a_dst"))
        H = p.heads_of(l - 1)
        DS = dout + H
        dnc = _f32(nV, DS, device=step.dev)
        with step.phase(f"bwd_rows{l}"):
            for d in step.devices:
                _lib.call("sg_gat_bwd_rows", _lib.ptr(ds.ws), ds.lay, l, d, dout, H, _lib.ptr(d_h),
                          _lib.ptr(keep["num"]), final, _lib.ptr(dnc), step.n_own(l, d), st)
        dnc_recv = _from_owner(step, l, dnc, DS)
        d_pre = _f32(nEtot, *_hs(H), device=step.dev)
        dt_loc = _f32(nV, *_hs(H), device=step.dev)
        dt_send = _f32(P, *_hs(H), device=step.dev)
        dt_recv = step._xbuf(P, *_hs(H))
        with step.phase(f"bwd_dst{l}"):
            for d in step.devices:
                _lib.call("sg_gat_bwd_dst", _lib.ptr(ds.ws), ds.lay, l, d, dout, H, slope, _lib.ptr(keep["z"]),
                          _lib.ptr(keep["alpha"]), _lib.ptr(keep["pre_e"]), _lib.ptr(dnc), _lib.ptr(dnc_recv),
                          DS, dp_ptr(d), _lib.ptr(d_pre), _lib.ptr(dt_loc), _lib.ptr(dt_send),
                          step.n_rows(l, d), st)
        if step.g > 1 and P > 0:
            step.transport.to_owner(ds, l, dt_send, dt_recv, H)
            if step.meta is not None:
                step.wire_bytes += int(step.meta.npairs[l]) * 4 * H
        if l == 1 and _wgrad_dst_ok(step):
            # one destination-centric pass: dW, da_src, da_dst (no d_z / ds / dt_tot)
            npart = w * dout + 2 * dout
            with step.phase(f"bwd_param{l}"):
                step._ev("wgd1_start")
                for d in step.devices:
                    nb = int(_lib.load().sg_gat_wgrad_dst_blocks(step.n_rows(l, d)))
                    part = _f32(nb * npart, device=step.dev)
                    _lib.call("sg_gat_wgrad_dst", _lib.ptr(ds.ws), ds.lay, d, w, H, _lib.ptr(h_prev),
                              _lib.ptr(src_row), dp_ptr(d), _lib.ptr(keep["alpha"]), _lib.ptr(d_pre),
                              _lib.ptr(dnc), _lib.ptr(dnc_recv), DS, _lib.ptr(dt_loc), _lib.ptr(dt_recv),
                              _lib.ptr(W), _lib.ptr(a_s), _lib.ptr(a_d), _lib.ptr(part), nb, st)
                    step.jobs.append((part, nb, npart, step.grads[d], p.offset(f"layer{l-1}.w")))
                    step._partials.append(part)
                step._ev("wgd1_end")
            d_h = None
            continue
        d_z = _f32(nVp, dout, device=step.dev)
        dsb = _f32(nVp, *_hs(H), device=step.dev)
        dt_tot = _f32(nV, *_hs(H), device=step.dev)
        with step.phase(f"bwd_src{l}"):
            for d in step.devices:
                perm, beg, end, _, keys = csr[d][:5]
                if (dout + H + 3) // 4 * 4 <= 192 and ds.nE[l - 1] >= TSPMM_MIN_EDGES:  # load-balanced pieces
                    nf = int(_lib.load().sg_tspmm_part_floats(ds.nE[l - 1], dout, H))
                    part = _f32(nf, device=step.dev)
                    _lib.call("sg_gat_bwd_src_lb", _lib.ptr(ds.ws), ds.lay, l, d, dout, H, _lib.ptr(keys),
                              _lib.ptr(perm), _lib.ptr(beg), _lib.ptr(end), kb[l], _csr_lmin(step), _lib.ptr(keep["alpha"]),
                              _lib.ptr(d_pre), _lib.ptr(dnc), _lib.ptr(dnc_recv), DS, _lib.ptr(dt_loc),
                              _lib.ptr(dt_recv), _lib.ptr(a_s), _lib.ptr(a_d), _lib.ptr(d_z), _lib.ptr(dsb),
                              _lib.ptr(dt_tot), _lib.ptr(part), ds.nE[l - 1], step.n_own(l - 1, d), st)
                else:
                    _lib.call("sg_gat_bwd_src", _lib.ptr(ds.ws), ds.lay, l, d, dout, H, _lib.ptr(perm),
                              _lib.ptr(beg), _lib.ptr(end), kb[l], _lib.ptr(keep["alpha"]), _lib.ptr(d_pre),
                              _lib.ptr(dnc), _lib.ptr(dnc_recv), DS, _lib.ptr(dt_loc), _lib.ptr(dt_recv),
                              _lib.ptr(a_s), _lib.ptr(a_d), _lib.ptr(d_z), _lib.ptr(dsb), _lib.ptr(dt_tot),
                              step.n_own(l - 1, d), st)
        need_prev = l > 1
        d_prev = _f32(nVp, w, device=step.dev) if need_prev else None
        npart = w * dout + 2 * dout
        with step.phase(f"bwd_param{l}"):
            for d in step.devices:
                nb = int(_lib.load().sg_gat_bwd_param_blocks(w, dout, H, step.n_own(l - 1, d)))
                part = _f32(nb * npart, device=step.dev)
                _lib.call("sg_gat_bwd_param", _lib.ptr(ds.ws), ds.lay, l, d, _lib.ptr(h_prev), _lib.ptr(src_row),
                          w, dout, H, _lib.ptr(keep["z"]), _lib.ptr(d_z), _lib.ptr(dsb), _lib.ptr(dt_tot), _lib.ptr(W),
                          _lib.ptr(part), nb, _lib.ptr(d_prev), step.n_own(l - 1, d), st)
                step.jobs.append((part, nb, npart, step.grads[d], p.offset(f"layer{l-1}.w")))
                step._partials.append(part)
        d_h = d_prev
