"""ctypes binding of libsplitgnn_b200.so (the C ABI in include/splitgnn_b200.h).

The library is REQUIRED: there is no CPU fallback. Importing a compute entry
point without the built .so raises immediately with the build command.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsplitgnn_b200.so")

MAXL = 8
MAXG = 16

i32, i64, u64, f32, f64, vp = C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_double, C.c_void_p
u32 = C.c_uint32


class SgMeta(C.Structure):
    _fields_ = [
        ("L", i32), ("g", i32), ("err", i32), ("dst_grouped", i32),
        ("nV", i64 * (MAXL + 1)),
        ("nE", i64 * MAXL),
        ("voff", i64 * (MAXL + 2)),
        ("eoff", i64 * (MAXL + 1)),
        ("n_own", (i32 * MAXG) * (MAXL + 1)),
        ("own_off", (i32 * (MAXG + 1)) * (MAXL + 1)),
        ("n_edge", (i32 * MAXG) * MAXL),
        ("edge_off", (i32 * (MAXG + 1)) * MAXL),
        ("n_load", i32 * MAXG),
        ("load_off", i32 * (MAXG + 1)),
        ("n_uniq", i32 * (MAXL + 1)),
        ("n_ref", (i32 * MAXG) * (MAXL + 1)),
        ("ref_off", (i32 * (MAXG + 1)) * (MAXL + 1)),
        ("cnt", ((i32 * MAXG) * MAXG) * (MAXL + 1)),
        ("pair_off", ((i32 * MAXG) * MAXG) * (MAXL + 1)),
        ("recv_off", (i32 * (MAXG + 1)) * (MAXL + 1)),
        ("recv_in", ((i32 * MAXG) * MAXG) * (MAXL + 1)),
        ("npairs", i32 * (MAXL + 1)),
    ]


class SgSplitLayout(C.Structure):
    _fields_ = [
        ("total_bytes", i64), ("L", i32), ("g", i32), ("n_vertices", i64),
        ("nV", i64 * (MAXL + 1)), ("nE", i64 * MAXL), ("voff", i64 * (MAXL + 2)),
        ("eoff", i64 * (MAXL + 1)), ("pbase", i64 * (MAXL + 2)),
        ("nVtot", i64), ("nEtot", i64), ("nPtot", i64), ("bm_words", i64),
        ("pos_tiles", i64), ("edge_tiles", i64), ("pair_tiles", i64),
        ("o_meta", i64), ("o_keys", i64), ("o_rank", i64), ("o_grouped", i64),
        ("o_ekey", i64), ("o_egrouped", i64), ("o_lsrc", i64), ("o_ldst", i64),
        ("o_pmask", i64), ("o_bitmap", i64), ("o_wpre", i64), ("o_ctot", i64),
        ("o_uorder", i64), ("o_refrank", i64), ("o_contrib", i64),
        ("o_pairs", i64), ("o_pair_hidx", i64), ("o_sendpos", i64), ("o_xfer", i64),
        ("o_recv_row", i64), ("o_selfrow", i64), ("o_rowbeg", i64), ("o_rowend", i64),
        ("o_tiles_pos", i64), ("o_tiles_edge", i64), ("o_tiles_pair", i64),
        ("o_tilebase_pos", i64), ("o_tilebase_edge", i64), ("o_tilebase_pair", i64),
        ("rbase", i64 * (MAXL + 2)),
    ]


P = C.POINTER
_SIGS = {
    "sg_last_error": (C.c_char_p, []),
    "sg_version": (C.c_char_p, []),
    "sg_launch_count": (C.c_ulonglong, []),
    "sg_device_sm_count": (i32, []),
    "sg_struct_sizes": (None, [vp]),
    "sg_split_layout": (i32, [i32, i32, P(i64), P(i64), i64, P(SgSplitLayout)]),
    "sg_split_run": (i32, [vp, P(SgSplitLayout), vp, vp, vp, vp, vp, vp, i32, vp]),
    "sg_sort_ws_bytes": (i64, [i64]),
    "sg_sort_pairs": (i32, [vp, i64, vp, vp, vp, i32, vp]),
    "sg_src_csr": (i32, [vp, P(SgSplitLayout), i32, i32, i32, vp, i64, vp, vp, vp, vp, vp, i64, vp]),
    "sg_dst_csr": (i32, [vp, P(SgSplitLayout), i32, vp, i64, vp, vp, vp, vp]),
    "sg_layer0_rows": (i32, [vp, P(SgSplitLayout), i32, vp, vp, i32, vp, vp]),
    "sg_stage_misses": (i32, [vp, P(SgSplitLayout), i32, i32, vp, vp, i32, vp, i32, i32, i64, vp]),
    "sg_host_map": (i32, [vp, i64, P(vp)]),
    "sg_host_unmap": (i32, [vp]),
    "sg_gather_rows": (i32, [vp, vp, i64, i32, vp, vp]),
    "sg_fill_uniform": (i32, [vp, i64, i32, u64, i64, vp]),
    "sg_sage_agg_fwd": (i32, [vp, P(SgSplitLayout), i32, i32, vp, vp, i32, i32, vp, vp, vp, i32, i64, vp]),
    "sg_sage_agg_fwd_perm": (i32, [vp, P(SgSplitLayout), i32, i32, vp, vp, i32, i32, vp, vp, vp, i32,
                                   vp, i64, vp]),
    "sg_sage_fused_fwd": (i32, [vp, P(SgSplitLayout), i32, i32, vp, vp, i32, i32, i32, vp, vp, vp, i32, vp, vp,
                                vp, vp, i64, vp]),
    "sg_sage_final_fused": (i32, [vp, P(SgSplitLayout), i32, vp, vp, i32, i32, i32, vp, vp, vp, vp, vp,
                                  vp, vp, vp, vp, vp, vp, vp, vp, vp, i32, i64, vp]),
    "sg_set_pdl": (None, [i32]),
    "sg_sage_agg_fwd_peer": (i32, [vp, P(SgSplitLayout), i32, i32, vp, vp, i32, i32, vp, vp, vp, i32, vp, i64, vp]),
    "sg_partition_cut": (i32, [vp, vp, i64, vp, vp, vp]),
    "sg_partition_cut_w": (i32, [vp, vp, vp, i64, vp, vp, vp]),
    "sg_partition_sizes": (i32, [vp, vp, i64, i32, vp, vp]),
    "sg_partition_match_round": (i32, [vp, vp, vp, vp, i64, i64, u64, i32, vp, vp, vp, vp]),
    "sg_partition_round": (i32, [vp, vp, vp, vp, i64, i32, i64, u64, i32, vp, vp, vp, vp, vp]),
    "sg_partition_coarse_host": (i32, [i64, vp, vp, vp, vp, i32, i64, u64, i32, vp, vp]),
    "sg_partition_refine_host": (i32, [i64, vp, vp, vp, vp, i32, i64, i32, vp, vp]),
    "sg_pack_sample": (i32, [vp, i32, vp, vp, vp, vp, i32, vp]),
    "sg_host_params_gather": (i32, [i32, vp, vp, vp, vp]),
    "sg_host_sum_sgd": (i32, [i32, vp, vp, vp, vp, vp, i32, i64, f32, vp, vp]),
    "sg_gat_wgrad_dst_blocks": (i32, [i64]),
    "sg_gat_agg_fused": (i32, [vp, P(SgSplitLayout), i32, i32, i32, f32, vp, vp, vp, vp, vp, i32, vp, vp, vp, vp, i64,
                               vp]),
    "sg_gat_wgrad_dst": (i32, [vp, P(SgSplitLayout), i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, i32, vp, vp, vp, vp, vp, vp,
                               i32, vp]),
    "sg_gpu_sampler_ws_bytes": (i64, [i64, i64, i64, i32]),
    "sg_gpu_sampler_ws_init": (i32, [vp, i64, i64, vp]),
    "sg_gpu_sample": (i32, [vp, vp, i64, vp, i64, vp, i32, u64, vp, i64, vp, vp, i64, i64, vp, vp, vp, vp, vp, vp,
                            vp]),
    "sg_sage_scatter_bwd_rows": (i32, [vp, P(SgSplitLayout), i32, i32, vp, vp, vp, i32, vp, vp, vp, i64, vp, i32,
                                       i32, vp, vp, vp, vp, vp, vp, i32, vp, vp, i64, vp]),
    "sg_sage_combine_fwd": (i32, [vp, P(SgSplitLayout), i32, i32, vp, vp, i32, i32, i32, vp, vp, vp, i32, vp, vp, vp,
                                  i32, vp, vp, vp, i64, vp]),
    "sg_sage_final_combine": (i32, [vp, P(SgSplitLayout), i32, vp, vp, i32, i32, i32, vp, vp, vp, vp, vp, vp,
                                    vp, vp, vp, i32, vp, vp, vp, vp, vp, vp, vp, i32, i64, vp]),
    "sg_peer_rounds": (i32, []),
    "sg_peer_exchange": (i32, [vp, P(SgSplitLayout), i32, i32, i32, vp, i32, vp, vp]),
    "sg_peer_signal": (i32, [vp, i32, i32, i32, vp, vp]),
    "sg_peer_wait": (i32, [vp, i32, i32, i32, vp, vp, vp]),
    "sg_peer_epoch": (i32, [vp, vp]),
    "sg_peer_grad_stage": (i32, [vp, vp, i64, i64, vp, vp]),
    "sg_peer_allreduce_sgd": (i32, [vp, i32, i64, i64, i64, vp, vp, vp, f32, vp]),
    "sg_peer_allreduce_sgd_nt": (i32, [vp, i32, i64, i64, i64, vp, vp, vp, f64, vp, vp]),
    "sg_split_cost": (i32, [vp, vp, vp, vp, vp, i32, vp, i64, i32, vp, vp, vp, vp, vp, vp, vp]),
    "sg_reduce_partials_sgd": (i32, [vp, i32, i64, f32, vp]),
    "sg_reduce_partials_sgd_nt": (i32, [vp, i32, i64, f64, vp, vp]),
    "sg_get_pdl": (i32, []),
    "sg_sage_update": (i32, [vp, P(SgSplitLayout), i32, i32, vp, vp, i32, i32, vp, vp, vp, i32,
                             vp, vp, vp, i32, vp, vp, vp, i64, vp]),
    "sg_sage_bwd_rows": (i32, [vp, P(SgSplitLayout), i32, i32, vp, vp, i32, i32, vp, vp, i32, vp,
                               vp, vp, vp, vp, i32, vp, vp, i32, i64, vp]),
    "sg_sage_scatter_bwd": (i32, [vp, P(SgSplitLayout), i32, i32, i32, vp, vp, vp, i32, vp, vp,
                                  vp, i64, vp, i64, vp]),
    "sg_gat_project": (i32, [vp, P(SgSplitLayout), i32, i32, vp, vp, i32, i32, i32, vp, vp, vp, vp, vp,
                             vp, i64, vp]),
    "sg_gat_agg": (i32, [vp, P(SgSplitLayout), i32, i32, i32, i32, f32, vp, vp, vp, vp, vp, vp, vp, vp,
                         vp, vp, i32, i64, vp]),
    "sg_gat_combine": (i32, [vp, P(SgSplitLayout), i32, i32, i32, i32, vp, vp, vp, vp, i32, i32, vp, vp,
                             vp, i64, vp]),
    "sg_gat_alpha": (i32, [vp, P(SgSplitLayout), i32, i32, i32, f32, vp, vp, vp, vp, i64, vp]),
    "sg_gat_bwd_rows": (i32, [vp, P(SgSplitLayout), i32, i32, i32, i32, vp, vp, i32, vp, i64, vp]),
    "sg_gat_bwd_dst": (i32, [vp, P(SgSplitLayout), i32, i32, i32, i32, f32, vp, vp, vp, vp, vp, i32, vp,
                             vp, vp, vp, i64, vp]),
    "sg_gat_bwd_src": (i32, [vp, P(SgSplitLayout), i32, i32, i32, i32, vp, vp, vp, i64, vp, vp, vp, vp,
                             i32, vp, vp, vp, vp, vp, vp, vp, i64, vp]),
    "sg_gat_bwd_param_blocks": (i32, [i32, i32, i32, i64]),
    "sg_gat_bwd_param": (i32, [vp, P(SgSplitLayout), i32, i32, vp, vp, i32, i32, i32, vp, vp, vp, vp, vp,
                               vp, i32, vp, i64, vp]),
    "sg_xfer_to_owner": (i32, [vp, P(SgSplitLayout), i32, vp, vp, i32, vp]),
    "sg_xfer_from_owner": (i32, [vp, P(SgSplitLayout), i32, vp, vp, i32, vp]),
    "sg_pack_from_owner": (i32, [vp, P(SgSplitLayout), i32, i32, vp, i32, vp, i32, i64, vp]),
    "sg_unpack_refs": (i32, [vp, P(SgSplitLayout), i32, i32, vp, i32, i32, vp, i64, vp]),
    "sg_cls_loss": (i32, [vp, P(SgSplitLayout), i32, vp, vp, vp, i32, i32, vp, vp, vp, vp, i32,
                          i64, vp]),
    "sg_reduce_partials": (i32, [vp, i32, i64, vp]),
    "sg_sum_sgd_nt": (i32, [vp, vp, vp, i32, i64, i64, f64, vp, vp]),
    "sg_sum_sgd": (i32, [vp, vp, vp, i32, i64, f32, vp]),
    "sg_gen_powerlaw": (i32, [i64, i64, i32, f64, f64, u64, i32, vp, vp]),
    "sg_gen_labels": (i32, [i64, i32, u64, vp]),
    "sg_fill_uniform_host": (i32, [vp, i64, i32, u64, i64, vp]),
    "sg_sampler_create": (vp, [i64, vp, vp]),
    "sg_sampler_destroy": (None, [vp]),
    "sg_sampler_run": (i32, [vp, vp, i64, vp, i32, u64, i32, vp, vp]),
    "sg_sampler_fetch": (i32, [vp, vp, vp, vp]),
    "sg_sampler_fetch_starts": (i32, [vp, vp, vp, vp, vp]),
    "sg_tspmm_part_floats": (i64, [i64, i32, i32]),
    "sg_sage_scatter_bwd_lb": (i32, [vp, P(SgSplitLayout), i32, i32, i32, vp, vp, vp, i32, vp, vp, vp, vp, i64, i32, vp,
                                     i64, vp, i64, vp]),
    "sg_gat_bwd_src_lb": (i32, [vp, P(SgSplitLayout), i32, i32, i32, i32, vp, vp, vp, vp, i64, i32, vp, vp, vp, vp, i32,
                                vp, vp, vp, vp, vp, vp, vp, vp, i64, i64, vp]),
    "sg_pipe_create": (vp, [i64]),
    "sg_pipe_create2": (vp, [i64, i64]),
    "sg_pipe_stage_compact": (i32, [vp, i32, vp, i64, vp, i64, i32, vp, i64, i64, vp, vp]),
    "sg_pipe_destroy": (None, [vp]),
    "sg_pipe_stage": (i32, [vp, i32, vp, i64, vp, vp]),
    "sg_pipe_finish": (i32, [vp, i32, vp, vp]),
    "sg_pipe_stage_direct": (i32, [vp, i32, vp, i64, vp, i64, i32, vp, i64, vp, vp]),
    "sg_relayout_sample_hdr": (i32, [vp, vp, vp, i64, vp]),
    "sg_relayout_sample_compact": (i32, [vp, vp, vp, i64, vp]),
    "sg_copy_async": (i32, [vp, vp, i64, vp]),
    "sg_pipe_release": (i32, [vp, i32, vp]),
    "sg_pipe_copy_stream": (vp, [vp]),
    "sg_pipe_wait": (i32, [vp, i32, vp]),
}

EXPORTED = tuple(_SIGS)
_lib = None


def load():
    """Load (once) and return the CDLL; raise loudly if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build the sm_100a library first "
            "(python -m paper_2303_13775_b200._build). There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    sizes = np.zeros(2, dtype=np.int64)
    lib.sg_struct_sizes(sizes.ctypes.data)
    if sizes[0] != C.sizeof(SgMeta) or sizes[1] != C.sizeof(SgSplitLayout):
        raise RuntimeError(f"ABI mismatch: C sizes {sizes.tolist()} vs ctypes "
                           f"{[C.sizeof(SgMeta), C.sizeof(SgSplitLayout)]}")
    _lib = lib
    return lib


class SplitGNNError(RuntimeError):
    pass


def check(rc, what=""):
    if rc != 0:
        msg = load().sg_last_error().decode(errors="replace")
        if rc == 1:
            raise ValueError(msg or what)
        raise SplitGNNError(f"{what}: {msg}" if what else msg)


def call(name, *args):
    """Invoke a C-ABI entry point and raise on a non-zero status."""
    check(getattr(load(), name)(*args), name)


def ptr(t):
    """Device/host pointer of a torch tensor or numpy array (None -> NULL)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


_RAW_STREAM = None


def stream_ptr(stream=None):
    """cudaStream_t of `stream` or of torch's current stream on the current
    device (read through torch's raw-stream query: building a Stream object
    costs ~3 us per call, and the hot paths call this several times a step)."""
    global _RAW_STREAM
    if stream is not None:
        return stream.cuda_stream
    if _RAW_STREAM is None:
        import torch
        raw, dev = getattr(torch._C, "_cuda_getCurrentRawStream", None), getattr(torch._C, "_cuda_getDevice", None)
        _RAW_STREAM = (lambda: raw(dev())) if raw is not None and dev is not None else \
            (lambda: torch.cuda.current_stream().cuda_stream)
    return _RAW_STREAM()


_STREAM_OBJ = [None, None]  # ((device, raw cudaStream_t), torch Stream)


def current_stream():
    """torch's current Stream object, reused while the current device and its
    raw current stream are unchanged (torch.cuda.current_stream() builds a new
    object per call, ~3 us; Event.record() without a stream calls it)."""
    import torch
    key = (torch._C._cuda_getDevice(), stream_ptr())
    if _STREAM_OBJ[0] != key or _STREAM_OBJ[1] is None:
        _STREAM_OBJ[1] = torch.cuda.current_stream()
        _STREAM_OBJ[0] = key
    return _STREAM_OBJ[1]


def launch_count():
    return int(load().sg_launch_count())
