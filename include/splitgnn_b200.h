/*
 * splitgnn-b200 — C ABI of the B200-native split-parallel GNN training step.
 *
 * The reference (arXiv 2303.13775 desk-scale package, /root/reference) is a
 * pure-Python/NumPy library with no FFI; every entry point below REPLACES the
 * NumPy body of the reference function cited beside it, and is bound from the
 * Python mirror package `paper_2303_13775_b200` through ctypes (see
 * INTEGRATION.md for the binding a maintainer adds on the reference side).
 *
 * Conventions
 *   - plain C types only: device pointers are `void*`/typed pointers into
 *     caller-owned (PyTorch-allocated) CUDA memory, sizes are int64_t;
 *   - every call is asynchronous on `stream` (a cudaStream_t passed as void*)
 *     and never synchronises the host;
 *   - return 0 on success, SG_ERR_ARG (1) for a bad argument, SG_ERR_CUDA (2)
 *     for a CUDA error; sg_last_error() returns the message;
 *   - data-dependent errors found on the device (e.g. a sampled vertex outside
 *     the partition map, scheduler.py:175-178) are reported through
 *     SgMeta.err, which the host reads with the per-iteration count D2H.
 */
#ifndef SPLITGNN_B200_H
#define SPLITGNN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SG_OK 0
#define SG_ERR_ARG 1
#define SG_ERR_CUDA 2

#define SG_MAXL 8  /* max GNN layers */
#define SG_MAXG 16 /* max devices (split parts) */

#define SG_ERR_MISSING_VERTEX 1 /* SgMeta.err bit: scheduler.py:177-178 */

/* sg_split_run flags */
#define SG_SPLIT_DST_GROUPED 1 /* each destination's in-edges are contiguous */
#define SG_SPLIT_ALL_CACHED 2  /* every sampled vertex is cached (load_gids empty) */

/* Per-iteration split descriptor written by sg_split_run into device memory.
 * Counts / offsets of the reference's LocalSplit + ShufflePlan
 * (scheduler.py:24-122). Index conventions: [l] layer 0..L, [l-1] for edge
 * layers 1..L, [s][o] = holder s -> owner o. */
typedef struct SgMeta {
  int32_t L, g, err, dst_grouped;
  int64_t nV[SG_MAXL + 1];   /* |V^l| */
  int64_t nE[SG_MAXL];       /* |E^l| at [l-1] */
  int64_t voff[SG_MAXL + 2]; /* offsets of V^l in the concatenated vertex array */
  int64_t eoff[SG_MAXL + 1]; /* offsets of E^l at [l-1] */
  int32_t n_own[SG_MAXL + 1][SG_MAXG];        /* len(owned_gids[l]) per device */
  int32_t own_off[SG_MAXL + 1][SG_MAXG + 1];  /* exclusive prefix over devices */
  int32_t n_edge[SG_MAXL][SG_MAXG];           /* per-device edges of layer l at [l-1] */
  int32_t edge_off[SG_MAXL][SG_MAXG + 1];
  int32_t n_load[SG_MAXG]; /* len(load_gids) */
  int32_t load_off[SG_MAXG + 1];
  int32_t n_uniq[SG_MAXL + 1];               /* distinct reference vertices at l */
  int32_t n_ref[SG_MAXL + 1][SG_MAXG];       /* len(ref_gids[l]) per holder */
  int32_t ref_off[SG_MAXL + 1][SG_MAXG + 1]; /* == first pair slot of holder */
  int32_t cnt[SG_MAXL + 1][SG_MAXG][SG_MAXG];      /* PlanEntry.count (l,s,o) */
  int32_t pair_off[SG_MAXL + 1][SG_MAXG][SG_MAXG]; /* s-major slot of entry (l,s,o) */
  int32_t recv_off[SG_MAXL + 1][SG_MAXG + 1];      /* owner o's receive base (o-major) */
  int32_t recv_in[SG_MAXL + 1][SG_MAXG][SG_MAXG];  /* offset of sender s inside o's block */
  int32_t npairs[SG_MAXL + 1];                     /* ShufflePlan.pair_count(l) */
} SgMeta;

/* Byte offsets (inside one caller-allocated workspace) of every split array.
 * Produced by sg_split_layout from the sample sizes; mirrored in Python. */
typedef struct SgSplitLayout {
  int64_t total_bytes;
  int32_t L, g;
  int64_t n_vertices;   /* len(PartitionMap.assignment) */
  int64_t nV[SG_MAXL + 1];
  int64_t nE[SG_MAXL];
  int64_t voff[SG_MAXL + 2];
  int64_t eoff[SG_MAXL + 1];
  int64_t pbase[SG_MAXL + 2]; /* per-layer base of pair-indexed arrays */
  int64_t nVtot, nEtot, nPtot;
  int64_t bm_words;           /* bitmap words per layer (padded) */
  int64_t pos_tiles, edge_tiles, pair_tiles;
  /* byte offsets */
  int64_t o_meta;
  int64_t o_keys, o_rank, o_grouped;      /* positions multisplit: nVtot + nV0 */
  int64_t o_ekey, o_egrouped, o_lsrc, o_ldst; /* edges: nEtot */
  int64_t o_pmask;                        /* u32 per position */
  int64_t o_bitmap, o_wpre, o_ctot;       /* gid-order ranking (layers 1..L) */
  int64_t o_uorder;                       /* positions of reference vertices in gid order */
  int64_t o_refrank;                      /* g * nVtot */
  int64_t o_contrib;                      /* g * nVtot, -1 = no contribution */
  int64_t o_pairs, o_pair_hidx, o_sendpos, o_xfer, o_recv_row; /* nPtot each */
  int64_t o_selfrow;                      /* nVtot, aligned with o_grouped */
  int64_t o_rowbeg, o_rowend;             /* per-layer local row space: nVtot + nPtot */
  int64_t o_tiles_pos, o_tiles_edge, o_tiles_pair; /* multisplit tile tables */
  int64_t o_tilebase_pos, o_tilebase_edge, o_tilebase_pair;
  int64_t rbase[SG_MAXL + 2]; /* per-layer base of row-space arrays */
} SgSplitLayout;

/* ---------------------------------------------------------------- library */
const char* sg_last_error(void);
const char* sg_version(void);
unsigned long long sg_launch_count(void); /* kernels launched by this library */
/* Programmatic dependent launch for every library kernel (default on;
 * SG_PDL=0 in the environment disables it at load). */
void sg_set_pdl(int on);
int sg_get_pdl(void);
int sg_device_sm_count(void);
void sg_struct_sizes(int64_t* out /* [sizeof(SgMeta), sizeof(SgSplitLayout)] */);

/* ---------------------------------------------------------------- splitter
 * Replaces split_minibatch (scheduler.py:164-254) including _group_by
 * (:157-161), the cache-filtered load set (:193-203), reference-vertex
 * ordering by gid (:228-238) and the ShufflePlan entries (:244-252). Computes
 * the split of ALL g devices from the replicated sample (each rank of a
 * multi-GPU job runs it on its own copy and keeps its own slice).
 *
 * The layout (sg_split_layout) is computed from CAPACITIES nV/nE; V: int32
 * layer vertices (V^l at offset voff[l]), esrc/edst: int32 per-layer edge
 * positions (E^l at eoff[l-1]). sizes: nullable DEVICE array of the actual
 * sizes [nV_0..nV_L, nE_1..nE_L] (<= capacities) — every kernel reads the
 * actual sizes from device memory, so one captured CUDA graph serves every
 * sample that fits the capacities. asn: uint8 device of each
 * global vertex (PartitionMap.assignment, partition.py:20-52). cache_bits:
 * nullable bitmap of CacheState.global_mask (partition.py:70-75). flags:
 * SG_SPLIT_DST_GROUPED if every layer's edges list each destination's in-edges
 * contiguously (true for sample_minibatch output, sampling.py:148-169);
 * SG_SPLIT_ALL_CACHED if the cache holds every vertex (no host loads). */
int sg_split_layout(int32_t L, int32_t g, const int64_t* nV, const int64_t* nE,
                    int64_t n_vertices, SgSplitLayout* out);
int sg_split_run(void* ws, const SgSplitLayout* lay, const int32_t* V,
                 const int32_t* esrc, const int32_t* edst, const int64_t* sizes,
                 const uint8_t* asn, const uint32_t* cache_bits, int32_t flags,
                 void* stream);

/* Stable LSD radix sort of (key,value) pairs (keys < 2^key_bits), used to
 * build CSR-by-source for the transpose SpMM (engine.py:263-273) and
 * CSR-by-destination for unordered samples. n is read from *n_dev (<= n_max).
 * Workspace from sg_sort_ws_bytes. */
int64_t sg_sort_ws_bytes(int64_t n_max);
int sg_sort_pairs(void* ws, int64_t n_max, const int32_t* n_dev, uint32_t* keys,
                  int32_t* vals, int32_t key_bits, void* stream);

/* Build CSR-by-source of the edges of device d at layers [lmin, L]. Keys are
 * global rows at l-1 (row_base[l] + own_off[l-1][d] + lsrc); on return
 * srcbeg/srcend (indexed by that key space) bound runs of `perm`. val_mode 0:
 * values are global edge slots of the split's grouped edge array; 1: values
 * encode the gradient row each out-edge reads (>= 0 owned row, < 0
 * -(1 + pair slot) of the push-from-owner payload). */
int sg_src_csr(const void* split_ws, const SgSplitLayout* lay, int32_t d,
               int32_t lmin, int32_t val_mode, void* sort_ws, int64_t n_max, int32_t* n_dev,
               uint32_t* keys, int32_t* perm, int32_t* srcbeg, int32_t* srcend,
               int64_t n_rows_total, void* stream);
/* Same for destinations (only needed when the sample is not dst-grouped):
 * writes rowbeg/rowend of the split workspace, with a permutation array. */
int sg_dst_csr(void* split_ws, const SgSplitLayout* lay, int32_t d,
               void* sort_ws, int64_t n_max, int32_t* n_dev, uint32_t* keys,
               int32_t* perm, void* stream);

/* ---------------------------------------------------------------- feature cache
 * Replaces SplitExecutor._load_inputs (engine.py:160-167): layer-0 rows of
 * device d resolve to rows of the GPU-resident partitioned feature cache
 * (cache_slot[gid] >= 0) or of the miss staging area appended after it
 * (miss_base + rank in load_gids). */
int sg_layer0_rows(const void* split_ws, const SgSplitLayout* lay, int32_t d,
                   const int32_t* V, const int32_t* cache_slot, int32_t miss_base,
                   int32_t* src_row0, void* stream);
int sg_gather_rows(const float* table, const int32_t* rows, int64_t n_rows, int32_t width,
                   float* out, void* stream);
/* Cache-miss staging (the host loads of _load_inputs, engine.py:160-167, of
 * the load_gids scheduler.py:193-203 lists): for devices [d0, d1), every
 * layer-0 row on the load list is read from host feature memory mapped into
 * the device address space (host_feats = the device address sg_host_map
 * returns for a row-major [n, feat_dim] fp32 matrix) into table row
 * n_cached + q, q = global load index (the row sg_layer0_rows assigns with
 * miss_base = n_cached). Counts come from the device SgMeta: no host sync,
 * capturable. staging_rows (rows allocated after the cached ones) must be
 * >= the layer-0 capacity. */
int sg_stage_misses(const void* split_ws, const SgSplitLayout* lay, int32_t d0, int32_t d1,
                    const int32_t* V, const float* host_feats, int32_t feat_dim,
                    float* table, int32_t row_stride, int32_t n_cached,
                    int64_t staging_rows, void* stream);
/* Page-lock a caller-owned host range for device access (mapped, read-only
 * hint) and return its device address; sg_host_unmap releases it. */
int sg_host_map(void* host_ptr, int64_t bytes, void** dev_ptr);
int sg_host_unmap(void* host_ptr);

/* Synthetic U[0,1) features (hash of (seed, row, col)), written on the device. */
int sg_fill_uniform(float* out, int64_t rows, int32_t width, uint64_t seed,
                    int64_t row0, void* stream);

/* h_stride (sg_sage_agg_fwd, _perm, sg_sage_fused_fwd, sg_sage_combine_fwd):
 * row stride of h_prev in floats, 0 = w. A layer-1 feature table whose rows
 * are padded to whole 128-byte lines (FeatureStore row_stride) is read in
 * whole lines: measured ~1.4x faster row gathers than 400-byte rows. */
/* ---------------------------------------------------------------- GraphSAGE
 * Forward local aggregation (engine.py:180-195, segment_sum/count
 * models.py:150-175): per local destination row, the sum of h_prev rows over
 * its in-edges and the edge count. Owned rows go to sums[own_off+q], counts;
 * reference rows are PACKED into the layer's pair-slot send buffer (width
 * send_stride >= w+1: sums then count) — the push-to-owner payload. h_prev
 * rows are addressed through `src_row` when non-null (layer 0: feature cache
 * indirection), else by global owned row. */
int sg_sage_agg_fwd(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                    const float* h_prev, const int32_t* src_row, int32_t w, int32_t h_stride,
                    float* sums, float* counts, float* sendbuf, int32_t send_stride,
                    int64_t max_rows, void* stream);
/* As sg_sage_agg_fwd for samples whose edges are not grouped by destination:
 * rowbeg/rowend index `dperm` (from sg_dst_csr). */
int sg_sage_agg_fwd_perm(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                         const float* h_prev, const int32_t* src_row, int32_t w, int32_t h_stride,
                         float* sums,
                         float* counts, float* sendbuf, int32_t send_stride,
                         const int32_t* dperm, int64_t max_rows, void* stream);
/* sg_sage_agg_fwd with the push-to-owner fused into the epilogue (peer
 * transport, one rank per GPU): reference rows go straight into the owners'
 * peer-mapped receive buffers peer_recv[0..g) (receive-slot layout, row stride
 * send_stride) at xfer[pair slot]; dperm may be null. */
int sg_sage_agg_fwd_peer(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                         const float* h_prev, const int32_t* src_row, int32_t w, int32_t h_stride,
                         float* sums, float* counts, const int64_t* peer_recv, int32_t send_stride,
                         const int32_t* dperm, int64_t max_rows, void* stream);
/* Single-device split (g = 1: no reference rows, no remote contributions):
 * aggregation + mean + both GEMVs + bias + ReLU in one kernel
 * (engine.py:180-226 with the exchange vacuous). Also writes mean, counts and
 * the compact self rows hs (n_own x w) the backward pass reads. */
int sg_sage_fused_fwd(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                      const float* h_prev, const int32_t* src_row, int32_t w, int32_t h_stride,
                      int32_t dout,
                      const float* w_self, const float* w_neigh, const float* bias,
                      int32_t final_layer, float* mean, float* counts, float* hs, float* h,
                      int64_t max_rows, void* stream);
/* Single-device split, LAST layer: aggregation + update (no ReLU) +
 * classifier_loss (models.py:287-302) + the layer's row-local backward
 * (engine.py:237-244: d_pre = d_h, weight/bias partials, d_self, d_sums) in
 * one kernel. part_cls gets nblocks x (dout*ncls + ncls + 1) partials in the
 * sg_cls_loss layout, part_lay nblocks x (2*w*dout + dout) in the
 * sg_sage_bwd_rows layout; both are summed by sg_reduce_partials. Also
 * writes mean, counts and h (n_own x dout). */
int sg_sage_final_fused(const void* split_ws, const SgSplitLayout* lay, int32_t d,
                        const float* h_prev, const int32_t* src_row, int32_t w, int32_t dout,
                        int32_t ncls, const float* w_self, const float* w_neigh,
                        const float* bias, const float* w_cls, const float* b_cls,
                        const int32_t* V, const int32_t* labels, float* mean, float* counts,
                        float* h, float* d_self, float* d_sums, float* part_cls,
                        float* part_lay, int32_t nblocks, int64_t max_rows, void* stream);
/* g > 1 owner side of a layer in one kernel: combine the local partial
 * (sums, counts from sg_sage_agg_fwd) with the holders' partials in recv
 * (receive slots, ascending sender: engine.py:197-210), mean, the two GEMVs,
 * bias, ReLU unless final (:212-226). counts is updated to the combined N;
 * mean, hs (self rows, n_own x w) and h are written. recv_stride % 4 == 0. */
int sg_sage_combine_fwd(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                        const float* h_prev, const int32_t* src_row, int32_t w, int32_t h_stride,
                        int32_t dout,
                        const float* w_self, const float* w_neigh, const float* bias,
                        int32_t final_layer, const float* sums, float* counts, const float* recv,
                        int32_t recv_stride, float* mean, float* hs, float* h, int64_t max_rows,
                        void* stream);
/* sg_sage_final_fused for any g: the last layer's combine (as
 * sg_sage_combine_fwd) + update + loss + row-local backward on device d. */
int sg_sage_final_combine(const void* split_ws, const SgSplitLayout* lay, int32_t d,
                          const float* h_prev, const int32_t* src_row, int32_t w, int32_t dout,
                          int32_t ncls, const float* w_self, const float* w_neigh,
                          const float* bias, const float* w_cls, const float* b_cls,
                          const int32_t* V, const int32_t* labels, const float* sums,
                          const float* recv, int32_t recv_stride, float* mean, float* counts,
                          float* h, float* d_self, float* d_sums, float* part_cls,
                          float* part_lay, int32_t nblocks, int64_t max_rows, void* stream);
/* Owner combine + update (engine.py:197-226): adds the holders' partial
 * (sum,count) rows from recvbuf in ascending sender order, mean = S/N,
 * pre = h_self@W_self + mean@W_neigh + b, h = relu(pre) unless final.
 * Writes mean (n_own x w), counts (combined), h (n_own x dout); with hs_out
 * (nullable) it also writes the compact self rows and runs the dense part as
 * the register-tiled FP32 GEMM k_sage_linear. */
int sg_sage_update(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                   const float* h_prev, const int32_t* src_row, int32_t w, int32_t dout,
                   const float* sums, float* counts, const float* recvbuf, int32_t recv_stride,
                   const float* w_self, const float* w_neigh, const float* bias,
                   int32_t final_layer, float* mean, float* h, float* hs_out, int64_t max_rows,
                   void* stream);
/* Backward row pass (engine.py:228-254): d_pre = d_h*[h>0] (or d_h if final);
 * per-block partial sums of h_self^T d_pre, mean^T d_pre and sum(d_pre)
 * (reduced later by sg_reduce_partials, deterministic order); optionally
 * d_self = d_pre W_self^T and d_sums = (d_pre W_neigh^T)/counts.
 * self_compact: h_prev is the compact self-row buffer (hs of
 * sg_sage_fused_fwd) indexed by owned row, instead of the layer input. */
int sg_sage_bwd_rows(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                     const float* h_prev, const int32_t* src_row, int32_t w, int32_t dout,
                     const float* d_h, const float* h, int32_t final_layer,
                     const float* mean, const float* counts,
                     const float* w_self, const float* w_neigh,
                     float* partial, int32_t nblocks, float* d_self, float* d_sums,
                     int32_t self_compact, int64_t max_rows, void* stream);
/* Transposed SpMM of layer l (engine.py:263-273) fused with the row-local
 * backward of layer l-1 (engine.py:237-244): the d_h rows of layer l-1 are
 * formed in shared memory tile by tile (scatter args as sg_sage_scatter_bwd)
 * while the tile's [hs | mean] rows of layer l-1 stream in, then masked by
 * ReLU'(h) and turned into weight-gradient partials (sg_sage_bwd_rows layout,
 * nblocks rows) and, if given, d_self_prev / d_sums_prev of layer l-1.
 * d_h width w in {4, 8, 16, 32}; w_in = layer l-1's input width (% 4 == 0). */
int sg_sage_scatter_bwd_rows(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                             const float* d_self, const float* d_sums, const float* bwd_recv,
                             int32_t recv_stride, const int32_t* enc, const int32_t* srcbeg,
                             const int32_t* srcend, int64_t key_base, const float* hs, int32_t w_in,
                             int32_t w, const float* h, const float* mean, const float* counts,
                             const float* w_self, const float* w_neigh, float* partial,
                             int32_t nblocks, float* d_self_prev, float* d_sums_prev,
                             int64_t max_rows, void* stream);
/* Transpose SpMM (engine.py:263-273): for each owned row u at l-1,
 * d_prev[u] = [u is the self row of v] d_self[v] + sum over out-edges of
 * d_sums_all[dst], where reference destinations read the owners' returned
 * gradients from bwd_recv[sendpos[...]] (push-from-owner payload). */
int sg_sage_scatter_bwd(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                        int32_t w, const float* d_self, const float* d_sums,
                        const float* bwd_recv, int32_t recv_stride,
                        const int32_t* enc, const int32_t* srcbeg, const int32_t* srcend,
                        int64_t key_base, float* d_prev, int64_t max_rows, void* stream);

/* ---------------------------------------------------------------- GAT
 * _gat_forward / _gat_backward (engine.py:280-552), models.py:217-261, with
 * 5 exchange rounds per layer instead of 10 (online-softmax merge + softmax
 * backward identity, see gat.cu). `heads` H >= 1: dout = D = H * d_head
 * (H = 1 is the reference layer; H > 1 concatenates H single-head layers).
 * Per-edge arrays are [edge slot][head] with the split's grouped edge slot
 * (eoff[l-1] + i); per-row scalars are [row][head]. */
int sg_gat_project(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                   const float* h_prev, const int32_t* src_row, int32_t w, int32_t dout,
                   int32_t heads, const float* W, const float* a_src, const float* a_dst,
                   float* z, float* s, float* t, int64_t max_rows, void* stream);
int sg_gat_agg(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d, int32_t dout,
               int32_t heads, float slope, const float* z, const float* s, const float* t,
               const float* t_recv, const int32_t* dperm, float* pre_e, float* loc_m,
               float* loc_s, float* loc_U, float* sendbuf, int32_t send_stride,
               int64_t max_rows, void* stream);
/* sg_gat_agg_fused: one device only -- sg_gat_agg with the owner combine
 * (num = U / den, h, md) and the per-edge alpha (engine.py:380-400) folded
 * into the aggregation epilogue (no holder partials to merge). */
int sg_gat_agg_fused(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t dout, int32_t heads,
                     float slope, const float* z, const float* s, const float* t, const int32_t* dperm, float* pre_e,
                     int32_t final_layer, float* md, float* num, float* h, float* alpha, int64_t max_rows,
                     void* stream);
int sg_gat_combine(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                   int32_t dout, int32_t heads, const float* loc_m, const float* loc_s,
                   const float* loc_U, const float* recv, int32_t recv_stride,
                   int32_t final_layer, float* md, float* num, float* h, int64_t max_rows,
                   void* stream);
int sg_gat_alpha(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                 int32_t heads, float slope, const float* pre_e, const float* md,
                 const float* md_recv, float* alpha, int64_t max_edges, void* stream);
int sg_gat_bwd_rows(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                    int32_t dout, int32_t heads, const float* d_h, const float* num,
                    int32_t final_layer, float* dnc, int64_t max_rows, void* stream);
int sg_gat_bwd_dst(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                   int32_t dout, int32_t heads, float slope, const float* z, const float* alpha,
                   const float* pre_e, const float* dnc, const float* dnc_recv,
                   int32_t recv_stride, const int32_t* dperm, float* d_pre, float* dt_loc,
                   float* sendbuf, int64_t max_rows, void* stream);
int sg_gat_bwd_src(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                   int32_t dout, int32_t heads, const int32_t* perm, const int32_t* srcbeg,
                   const int32_t* srcend, int64_t key_base, const float* alpha, const float* d_pre,
                   const float* dnc, const float* dnc_recv, int32_t dnc_stride,
                   const float* dt_loc, const float* dt_recv, const float* a_src,
                   const float* a_dst, float* d_z, float* ds, float* dt_tot, int64_t max_rows,
                   void* stream);
/* Partial slices (CTAs) sg_gat_bwd_param wants for `rows` rows: the caller
 * sizes `partial` as nblocks x (w*dout + 2*dout) floats with this count. */
int32_t sg_gat_bwd_param_blocks(int32_t w, int32_t dout, int32_t heads, int64_t rows);
int sg_gat_bwd_param(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                     const float* h_prev, const int32_t* src_row, int32_t w, int32_t dout,
                     int32_t heads, const float* z, const float* d_z, const float* ds,
                     const float* dt_tot, const float* W, float* partial, int32_t nblocks,
                     float* d_prev, int64_t max_rows, void* stream);

/* ---------------------------------------------------------------- exchange
 * Pack / transport helpers for the push-to-owner / push-from-owner rounds
 * (engine.py:125-156, scatter_shuffle_forward :591-630). Layer-l pair slots
 * are holder-major (the holders' send buffers back to back); receive slots
 * are owner-major (xfer maps slot -> receive slot). */
int sg_xfer_to_owner(const void* split_ws, const SgSplitLayout* lay, int32_t l,
                     const float* sendbuf, float* recvbuf, int32_t stride, void* stream);
int sg_xfer_from_owner(const void* split_ws, const SgSplitLayout* lay, int32_t l,
                       const float* sendbuf_recv_layout, float* recvbuf_pair_layout,
                       int32_t stride, void* stream);
/* Owner-side pack of owned rows for push-from-owner: out[recv slot] = rows[recv_row]. */
int sg_pack_from_owner(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                       const float* rows, int32_t w, float* out, int32_t stride,
                       int64_t max_slots, void* stream);
/* Holder-side unpack of a push-from-owner payload into ref-aligned rows. */
int sg_unpack_refs(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                   const float* recv_pair_layout, int32_t stride, int32_t w, float* out,
                   int64_t max_rows, void* stream);

/* ---------------------------------------------------------------- loss / optimizer
 * classifier_loss (models.py:287-302) fused: logits, summed softmax-CE,
 * d_h = (softmax-onehot) W^T, per-block partials of W-grad, b-grad and loss. */
int sg_cls_loss(const void* split_ws, const SgSplitLayout* lay, int32_t d,
                const int32_t* V, const int32_t* labels, const float* h, int32_t hid,
                int32_t ncls, const float* w_cls, const float* b_cls, float* d_h,
                float* partial, int32_t nblocks, int64_t max_rows, void* stream);
/* Deterministic reduction of per-block partials: out[k] = sum_b partial[b*n+k]
 * (ascending b). jobs: HOST array of n_jobs quadruples (partial device ptr,
 * nblocks, n, out device ptr), passed to the kernel by value. */
int sg_reduce_partials(const int64_t* jobs, int32_t n_jobs, int64_t max_n, void* stream);
/* split_cost (scheduler.py:257-309) on the device for a packed sample
 * (V, esrc, edst as sg_split_run; nV[0..L], nE[0..L-1] host arrays):
 * counts[(l-1)*g + d] = edges of E^l whose source lives on d, local[l-1] =
 * edges with source and destination on one device, cost_rows = C[v^l] for
 * every position of V^1..V^L (concatenated), cost[l-1] = sum of C over V^l.
 * mask_ws: sum_{l>=1} nV[l] uint32 scratch. *err != 0 when a sampled vertex is
 * outside the map. Integer atomics only (exact). */
int sg_split_cost(const int32_t* V, const int32_t* esrc, const int32_t* edst, const int64_t* nV,
                  const int64_t* nE, int32_t L, const uint8_t* assignment, int64_t n_vertices,
                  int32_t g, uint32_t* mask_ws, int32_t* cost_rows, int64_t* counts,
                  int64_t* local, int64_t* cost, int32_t* err, void* stream);
/* ---- peer-memory transport (one rank per GPU; replaces the NCCL
 * all-to-all-v of engine.py:121-156 with IPC-mapped buffers) ----------------
 * peer_bufs / peer_flags: g device pointers (this rank's own entry included),
 * each a peer's buffer mapped into this process.
 * sg_peer_exchange push=1 (push-to-owner): this rank's pair-slot rows of
 * `local` are written into each owner's buffer at their receive slot.
 * push=0 (push-from-owner): this rank's pair-slot rows of `local` are read
 * from each owner's buffer (packed at receive slots by sg_pack_from_owner).
 * sg_peer_signal stores the current epoch into slot [round][rank] of every
 * peer's flag array; sg_peer_wait blocks the stream until every peer has
 * signalled `round` for the current epoch (*timeout set if a peer vanished);
 * sg_peer_epoch bumps the epoch once per step. */
int sg_peer_rounds(void);
int sg_peer_exchange(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t rank,
                     int32_t push, float* local, int32_t stride, const int64_t* peer_bufs,
                     void* stream);
int sg_peer_signal(const int64_t* peer_flags, int32_t rank, int32_t g, int32_t round,
                   const int32_t* epoch, void* stream);
/* k_peer_wait traps (aborting the CUDA context) after 20 s without a peer
 * signal, after setting *timeout: a lost peer never lets a step continue. */
int sg_peer_wait(const int32_t* my_flags, int32_t rank, int32_t g, int32_t round,
                 const int32_t* epoch, int32_t* timeout, void* stream);
int sg_peer_epoch(int32_t* epoch, void* stream);
/* Gradient all-reduce + SGD over peer memory (allreduce_and_step,
 * engine.py:633-647): stage this rank's n1 = n + 1 floats (gradient + loss
 * slot) into slot (epoch & 1) of its shared slots (2 x slot_stride floats),
 * then, after a signal/wait round, every rank sums all ranks' slots in rank
 * order (identical on every rank), writes the sum to grads_out (optional) and
 * applies params[k] -= scale * sum[k] for k < n. */
int sg_peer_grad_stage(const float* grads, float* my_slots, int64_t n1, int64_t slot_stride,
                       const int32_t* epoch, void* stream);
int sg_peer_allreduce_sgd(const int64_t* peer_slots, int32_t g, int64_t n, int64_t n1,
                          int64_t slot_stride, const int32_t* epoch, float* params, float* grads_out,
                          float scale, void* stream);
/* scale = lr / *num_targets on the device (the replayed sample's target count). */
int sg_peer_allreduce_sgd_nt(const int64_t* peer_slots, int32_t g, int64_t n, int64_t n1,
                             int64_t slot_stride, const int32_t* epoch, float* params, float* grads_out,
                             double lr, const int64_t* num_targets, void* stream);
/* ---- GPU k-hop sampler (sample_minibatch, sampling.py:118-177) ---------------
 * From a device in-CSR (row_offsets int64[n+1], col_indices int32), for
 * device int64 targets[nt]: the packed sample (V^l at voff[l], E^l at
 * eoff_cap[l-1], sizes = [nV_0..nV_L, nE_1..nE_L]) identical to the native
 * host sampler's for the same seed. ws: sg_gpu_sampler_ws_bytes(n, max_dst,
 * max_edges, max fanout) bytes, initialised once with sg_gpu_sampler_ws_init
 * (it keeps a device generation counter, so calls replay inside a CUDA graph).
 * seed_dev (optional): read the seed from device memory (per replay).
 * *err: 1 target out of range, 2/4 edge / vertex capacity exceeded.
 * Fanouts in [0, 64]. */
int64_t sg_gpu_sampler_ws_bytes(int64_t n, int64_t max_dst, int64_t max_edges, int32_t fmax);
int sg_gpu_sampler_ws_init(void* ws, int64_t n, int64_t ws_bytes, void* stream);
int sg_gpu_sample(const int64_t* row_offsets, const int32_t* col_indices, int64_t n,
                  const int64_t* targets, int64_t nt, const int32_t* fanouts, int32_t L, uint64_t seed,
                  const uint64_t* seed_dev, int64_t ws_bytes, const int64_t* voff, const int64_t* eoff_cap,
                  int64_t max_dst,
                  int64_t max_edges, int32_t* V, int32_t* esrc, int32_t* edst, int64_t* sizes, void* ws,
                  int32_t* err, void* stream);
/* ---- balanced k-way partitioning (partition.py:236-349) --------------------
 * Multilevel, on symmetric weighted level graphs (off int64[n+1], nbr int32,
 * wt int32 edge weights, vw int32 vertex weights; level 0 = the input graph
 * symmetrised, weight = arcs u->v + arcs v->u, partition.py:123-136).
 * sg_partition_cut: directed arcs whose endpoints lie in different parts, on
 *   the input in-CSR (cut_size, partition.py:352-355).
 * sg_partition_cut_w: sum of wt over level-graph entries across parts (twice
 *   the directed cut at level 0).
 * sg_partition_sizes: part weights under vw (nullable: unit weights).
 * sg_partition_match_round: one heavy-edge matching round (partition.py:144-175
 *   restated as locally-dominant-edge matching): unmatched vertices (match < 0)
 *   pick the heaviest unmatched neighbour with vw[u] + vw[v] <= wcap (ties by a
 *   pair-symmetric seeded hash); mutual picks are matched. ws >= 4n bytes;
 *   *matched_out accumulates the matched vertices (device).
 * sg_partition_round: one parallel refinement round (partition.py:236-270):
 *   a seeded half of the vertices propose their best strictly positive gain
 *   move (lowest part on ties), admitted per target part in descending gain
 *   within the weight cap; updates part and sizes; ws >= 8n + 8*16*64 + 64
 *   bytes; *moved_out = moves (device).
 * sg_partition_coarse_host (HOST memory, CPU): the coarsest level's initial
 *   partition (partition.py:186-233): greedy region growing + sequential
 *   refinement, best of `restarts` (a feasible partition preferred); writes
 *   part_out[n] and *cut_out (level cut, directed-arc units). */
int sg_partition_cut(const int64_t* row_offsets, const int32_t* col_indices, int64_t n, const int32_t* part,
                     unsigned long long* cut_out, void* stream);
int sg_partition_cut_w(const int64_t* off, const int32_t* nbr, const int32_t* wt, int64_t n, const int32_t* part,
                       unsigned long long* cut_out, void* stream);
int sg_partition_sizes(const int32_t* part, const int32_t* vw, int64_t n, int32_t g, int64_t* sizes, void* stream);
int sg_partition_match_round(const int64_t* off, const int32_t* nbr, const int32_t* wt, const int32_t* vw,
                             int64_t n, int64_t wcap, uint64_t seed, int32_t round, int32_t* match, void* ws,
                             unsigned long long* matched_out, void* stream);
int sg_partition_round(const int64_t* off, const int32_t* nbr, const int32_t* wt, const int32_t* vw, int64_t n,
                       int32_t g, int64_t cap, uint64_t seed, int32_t round, int32_t* part, int64_t* sizes,
                       void* ws, unsigned long long* moved_out, void* stream);
int sg_partition_coarse_host(int64_t n, const int64_t* off, const int32_t* nbr, const int32_t* wt,
                             const int32_t* vw, int32_t g, int64_t cap, uint64_t seed, int32_t restarts,
                             int32_t* part_out, int64_t* cut_out);
/* sg_partition_refine_host (HOST memory, CPU): sequential boundary refinement
 * of one level (partition.py:236-270: overfull parts repaired, then strictly
 * positive gain moves within cap, ascending id, lowest part on ties) for the
 * levels small enough for one core; part updated in place, *cut_out = level cut. */
/* sg_pack_sample (HOST memory, CPU): a sample's arrays (V^0..V^L, E^l sources,
 * E^l destinations; each int32 or int64, elem_bytes 4 / 8) copied as int32 to
 * out + dst_off[i] (words), after an int64 header of the 2L+1 sizes
 * [nV_0..nV_L, nE_1..nE_L]; split over `threads` host threads (0 = all),
 * non-temporal stores (the buffer is read next by the H2D DMA, not a CPU).
 * vrange (nullable) receives [min, max] over the vertex ids V^0..V^L.
 * split_minibatch's staging of the sample (scheduler.py:164). */
int sg_pack_sample(int32_t* out, int32_t L, const int64_t* sizes, const int64_t* dst_off, const void* const* src,
                   const int32_t* elem_bytes, int32_t threads, int64_t* vrange);
/* sg_sampler_fetch_starts (HOST memory, CPU): sg_sampler_fetch plus the
 * per-destination run starts of every layer (layers 1..L back to back, |V^l|
 * ints each) -- the compact form split_minibatch sends instead of the
 * destination lists (sampling.py:118-177 output, edges grouped per
 * destination in ascending order). */
int sg_sampler_fetch_starts(void* h, int32_t* V, int32_t* esrc, int32_t* edst, int32_t* starts);
/* sg_host_params_gather (HOST memory, CPU): SplitExecutor.run's parameter
 * snapshot (engine.py:95-117): k contiguous arrays (elem_bytes 8 = fp64,
 * 4 = fp32) flattened to fp32 in order into out. */
int sg_host_params_gather(int32_t k, const void* const* ptrs, const int64_t* sizes, const int32_t* elem_bytes,
                          float* out);
/* sg_host_sum_sgd (HOST memory, CPU): allreduce_and_step (engine.py:633-647,
 * models.py:95-99) for gradients already on the host. If the k parameter
 * arrays, rounded to fp32, still equal `snapshot` bit for bit (nullable: skip
 * the check): total_out = the g
 * flat fp32 gradients (n each) summed in device order, and every parameter
 * p <- fp32(p - scale * total), the product exact and rounded once (the device
 * kernel's fused multiply-add), written back in the array's element type;
 * *applied = 1. Otherwise nothing is written and *applied = 0. */
int sg_host_sum_sgd(int32_t k, void* const* ptrs, const int64_t* sizes, const int32_t* elem_bytes,
                    const float* snapshot, const float* const* grads, int32_t g, int64_t n, float scale,
                    float* total_out, int32_t* applied);
int sg_partition_refine_host(int64_t n, const int64_t* off, const int32_t* nbr, const int32_t* wt,
                             const int32_t* vw, int32_t g, int64_t cap, int32_t max_passes, int32_t* part,
                             int64_t* cut_out);
/* sg_gat_wgrad_dst: GAT layer-1 weight gradient in one destination-centric
 * pass (engine.py:480-552 regrouped by destination: dW = sum_v A_v^T dn_v +
 * SB (x) a_src + SC (x) a_dst, da_src = SB W, da_dst = SC W with
 * A_v = sum_u alpha_uv h_u, SB = sum dpre_uv h_u, SC = sum_v dt_v h_self(v));
 * replaces sg_gat_bwd_src + sg_gat_bwd_param at layer 1. D = 64, heads in
 * {1, 2, 4}, w % 4 == 0, w <= 128. partial: nblocks slices of w*64 + 128
 * floats [dW | da_src | da_dst]; sg_gat_wgrad_dst_blocks gives nblocks. */
int32_t sg_gat_wgrad_dst_blocks(int64_t rows);
int sg_gat_wgrad_dst(const void* split_ws, const SgSplitLayout* lay, int32_t d, int32_t w, int32_t heads,
                     const float* h0, const int32_t* src_row, const int32_t* dperm, const float* alpha,
                     const float* d_pre, const float* dnc, const float* dnc_recv, int32_t recv_stride,
                     const float* dt_loc, const float* dt_recv, const float* W, const float* a_src,
                     const float* a_dst, float* partial, int32_t nblocks, void* stream);
/* sg_reduce_partials with the SGD step fused (single device, nothing to
 * all-reduce): jobs are 6 int64 per job {partials, nblocks, n, out, param,
 * n_sgd}; the first n_sgd summed columns g also update param: p -= scale*g
 * (ModelParams.sgd_step, models.py:95-99). param = 0 skips the step. */
int sg_reduce_partials_sgd(const int64_t* jobs, int32_t n_jobs, int64_t max_n, float scale,
                           void* stream);
/* As sg_reduce_partials_sgd with scale = lr / *num_targets computed on the
 * device (in double, like the host's lr / len(targets)): a captured step
 * normalises by each replayed sample's own target count (device sizes). */
int sg_reduce_partials_sgd_nt(const int64_t* jobs, int32_t n_jobs, int64_t max_n, double lr,
                              const int64_t* num_targets, void* stream);
/* allreduce_and_step (engine.py:633-647): grads = sum over devices in device
 * order (grad_ptrs: HOST array of n_dev device pointers to flat buffers), then
 * p -= lr/num_targets * grads; grads_out (nullable) receives the sum. */
int sg_sum_sgd(float* params, float* grads_out, const int64_t* grad_ptrs, int32_t n_dev,
               int64_t n, float scale, void* stream);
/* sg_sum_sgd over n1 >= n columns (e.g. the loss slot; only k < n update
 * params) with scale = lr / *num_targets computed on the device: the
 * multi-part single-GPU step captured as one CUDA graph. */
int sg_sum_sgd_nt(float* params, float* grads_out, const int64_t* grad_ptrs, int32_t n_dev,
                  int64_t n, int64_t n1, double lr, const int64_t* num_targets, void* stream);

/* ---------------------------------------------------------------- host-side native code
 * Synthetic block-planted Chung-Lu power-law graph as an
 * in-CSR (graph.py:23-128 layout: col = sources of each destination, sorted
 * within a row). Multithreaded; deterministic in (n, m, blocks, p_local,
 * gamma, seed) whatever the thread count. Caller allocates n+1 / m. */
int sg_gen_powerlaw(int64_t n, int64_t m, int32_t blocks, double p_local, double gamma,
                    uint64_t seed, int32_t threads, int64_t* row_offsets, int32_t* col_indices);
/* Uniform labels in [0, num_classes) (hash of (seed, v)). */
int sg_gen_labels(int64_t n, int32_t num_classes, uint64_t seed, int32_t* out);
/* Host twin of sg_fill_uniform (bit-identical values) for rows row_ids (or
 * row0.. when row_ids is null). */
int sg_fill_uniform_host(float* out, int64_t rows, int32_t width, uint64_t seed, int64_t row0,
                         const int64_t* row_ids);
/* Native k-hop neighbour sampler with sample_minibatch semantics
 * (sampling.py:105-177): self-edge first, up to fanout distinct in-neighbours
 * by partial Fisher-Yates, duplicates and the vertex itself dropped, new
 * vertices appended in first-seen order; ValueError cases (:128-136) return
 * SG_ERR_ARG with the reference's message. Counter-based RNG keyed by
 * (seed, layer, position, draw) so results do not depend on threads. */
void* sg_sampler_create(int64_t n, const int64_t* row_offsets, const int32_t* col_indices);
void sg_sampler_destroy(void* h);
int sg_sampler_run(void* h, const int64_t* targets, int64_t n_targets, const int32_t* fanouts,
                   int32_t L, uint64_t seed, int32_t threads, int64_t* nV_out /* L+1 */,
                   int64_t* nE_out /* L */);
int sg_sampler_fetch(void* h, int32_t* V /* sum nV */, int32_t* esrc, int32_t* edst);

/* Load-balanced transposed SpMM (tspmm.cu): the source-row sums of the
 * SAGE scatter backward (replaces sg_sage_scatter_bwd's row-per-warp loop;
 * engine.py:470-520) and of the GAT source backward (sg_gat_bwd_src;
 * engine.py:430-552), over the CSR-by-source from sg_src_csr (its sorted
 * `keys` and values, built with first layer `lmin`). Work is split into
 * chunks of 32 sorted edges so power-law hub rows do not serialise; rows
 * crossing chunks are combined in chunk order (deterministic). `part` holds
 * sg_tspmm_part_floats(max_edges, width, extra) floats (extra = heads for
 * GAT, 0 for SAGE); max_edges bounds layer l's local edges. Widths: width +
 * extra <= 192. */
int64_t sg_tspmm_part_floats(int64_t max_edges, int32_t width, int32_t extra);
int sg_sage_scatter_bwd_lb(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                           int32_t w, const float* d_self, const float* d_sums, const float* bwd_recv,
                           int32_t recv_stride, const uint32_t* keys, const int32_t* enc,
                           const int32_t* srcbeg, const int32_t* srcend, int64_t key_base, int32_t lmin,
                           float* part, int64_t max_edges, float* d_prev, int64_t max_rows, void* stream);
int sg_gat_bwd_src_lb(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d, int32_t dout,
                      int32_t heads, const uint32_t* keys, const int32_t* perm, const int32_t* srcbeg,
                      const int32_t* srcend, int64_t key_base, int32_t lmin, const float* alpha,
                      const float* d_pre, const float* dnc, const float* dnc_recv, int32_t dnc_stride,
                      const float* dt_loc, const float* dt_recv, const float* a_src, const float* a_dst,
                      float* d_z, float* ds, float* dt_tot, float* part, int64_t max_edges,
                      int64_t max_rows, void* stream);

/* Host->device input pipeline for the captured step; replaces the
 * reference's synchronous per-iteration input load (engine.py:760-790,
 * _load_inputs) with a double-buffered one: sg_pipe_stage copies a pinned
 * packed sample into staging slot `slot` on an internal copy stream (after
 * that slot's previous consumer), then, ordered on `stream`, into the graph's
 * input buffer dev_dst; sg_pipe_finish queues the D2H of the step's loss on
 * `stream`; sg_pipe_wait blocks until it has landed and returns it. */
void* sg_pipe_create(int64_t bytes);
/* bytes (a multiple of 16) of staged input layout + `extra` scratch bytes for
 * the compact form's run starts. */
void* sg_pipe_create2(int64_t bytes, int64_t extra);
/* Compact staging of a destination-grouped sample: H2D of the prefix (header,
 * V, es: prefix_bytes) and of the per-destination run starts (layer by layer,
 * |V^l| ints each), the ed lists rebuilt from them on the copy stream
 * (edge_off[l-1] = capacity offset of E^l, o_ed = word offset of the ed
 * region), then the D2D of full_bytes into dev_dst on `stream`. */
int sg_pipe_stage_compact(void* h, int32_t slot, const void* host_prefix, int64_t prefix_bytes,
                          const void* host_starts, int64_t starts_bytes, int32_t L, const int64_t* edge_off,
                          int64_t o_ed, int64_t full_bytes, void* dev_dst, void* stream);
/* Direct staging for one captured graph per slot: the H2D (and, with run
 * starts, the ed rebuild) lands straight in the slot graph's input buffer on
 * the copy stream, which waits for the previous graph on that slot
 * (sg_pipe_release, recorded after queueing it); no device-to-device copy on
 * the step's critical path. starts_bytes == 0: full layout in host_prefix. */
int sg_pipe_stage_direct(void* h, int32_t slot, const void* host_prefix, int64_t prefix_bytes,
                         const void* host_starts, int64_t starts_bytes, int32_t L, const int64_t* edge_off,
                         int64_t o_ed, void* dev_dst, void* stream);
int sg_pipe_release(void* h, int32_t slot, void* stream);
/* One cudaMemcpyAsync (cudaMemcpyDefault: pinned host / device pointers under
 * UVA) on `stream`: SplitExecutor.run's parameter upload (engine.py:95-117
 * executor inputs), sample load and gradient read-back. */
int sg_copy_async(void* dst, const void* src, int64_t bytes, void* stream);
/* split_minibatch for a sample the native sampler wrote into one pinned
 * buffer [int64 header of the 2L+1 sizes | V^0..V^L | E^l sources | E^l
 * destinations] (scheduler.py:164 entry; replaces sg_pack_sample's host copy):
 * after one H2D of it to `src`, its 3L+2 segments are copied into the capacity
 * layout `dst`, the segment bounds derived on the device from the sample's
 * own int64 sizes header (src[0 .. S) words, S = 2(2L+1)): geo = [L, S, o_V,
 * o_es, o_ed, voff[0..L+1], eoff[0..L]] (host int64, the capacity layout;
 * lengths clamped to it); max_len bounds the longest segment (grid size). */
int sg_relayout_sample_hdr(const int32_t* src, int32_t* dst, const int64_t* geo, int64_t max_len, void* stream);
/* Compact form of sg_relayout_sample_hdr: src = [header | V^0..V^L | E^l
 * sources | per-destination run starts of layers 1..L (|V^l| ints each, first
 * edge of each destination, ascending)]; the E^l destination lists are
 * rebuilt from the starts into the capacity layout (the sampler's edge order:
 * one run per destination). */
int sg_relayout_sample_compact(const int32_t* src, int32_t* dst, const int64_t* geo, int64_t max_len,
                               void* stream);
void* sg_pipe_copy_stream(void* h);
void sg_pipe_destroy(void* h);
int sg_pipe_stage(void* h, int32_t slot, const void* host_src, int64_t bytes, void* dev_dst,
                  void* stream);
int sg_pipe_finish(void* h, int32_t slot, const float* dev_loss, void* stream);
int sg_pipe_wait(void* h, int32_t slot, float* loss_out);

#ifdef __cplusplus
}
#endif
#endif /* SPLITGNN_B200_H */
