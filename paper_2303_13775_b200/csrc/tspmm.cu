// Load-balanced transposed SpMM for the backward pass: the source-row sums
//   SAGE  d_prev[u] = sum_{e: src(e)=u} d_sums[dst(e)] (+ d_self[u] on self rows)
//         (engine.py:_sage_backward scatter, :470-520)
//   GAT   d_z[u]    = sum_{e: src(e)=u} alpha_e * d_num[dst(e)] + ds_u a_src (+ dt_u a_dst)
//         (engine.py:_gat_backward, :430-552)
// over the CSR-by-source (edges sorted by source-row key, sort.cu).
//
// Sampled graphs are power-law: a layer-0 source can have ~1000 out-edges
// while the mean is ~2, so one warp per source row serialises the hub rows
// (measured: 276 us for 344K edges). Positions of the sorted edge array are
// cut into CHUNKS of TC = 32; a row's edges are processed in PIECES that
// never cross a chunk boundary, one warp task per piece:
//   row task      (one per source row): the row's first piece
//                 [beg, min(end, next chunk boundary)) -- for light rows the
//                 whole row, finished straight from registers;
//   continuation  (one per chunk that starts inside a row): the row's piece
//                 inside that chunk.
// Each task is at most 32 edges: one index prefetch, then independent row
// loads. Pieces of rows that span chunks go to part[chunk][slot]; K2 (one
// warp per chunk) finishes each row that STARTS in its chunk and spans out,
// summing the pieces in chunk order. Every sum has a fixed order, so results
// are run-to-run deterministic, with no float atomics.
//
// Partial slot rule: a row's first piece uses slot 0 of its chunk when the
// row starts at the chunk start, else slot 1; continuation pieces use slot 0.
#include <cstring>

#include "common.cuh"

namespace sg {
namespace {

constexpr int TC = 32;       // sorted edge positions per chunk
constexpr int TWARPS = 8;    // warps per block
constexpr unsigned FULL = 0xffffffffu;

struct TsGeom {
  int l, d, lmin, ws;        // ws = shared-memory row stride (>= width + extra, % 4 == 0)
  int64_t key_base;
  const uint32_t* keys;      // sorted row keys
  const int32_t* vals;       // sorted values (SAGE: dst code, GAT: edge slot)
  const int32_t* srcbeg;
  const int32_t* srcend;
  float* part;               // [chunks][2][ws]
};

__device__ __forceinline__ void layer_span(const SgMeta* meta, int l, int d, int lmin, int64_t& p0, int& n) {
  int64_t acc = 0;
  for (int li = lmin - 1; li < l - 1; ++li) acc += meta->n_edge[li][d];
  p0 = acc;
  n = meta->n_edge[l - 1][d];
}

// ---------------------------------------------------------------- policies
struct SagePol {
  static constexpr bool kExtra = false;
  int l, d, w, stride;
  int64_t voff_lm1, voff_l;
  const int32_t* grouped;
  const int32_t* rank;
  const float* d_self;
  const float* d_sums;
  const float* bwd_recv;
  float* d_prev;

  __device__ int width() const { return w; }
  __device__ int extra() const { return 0; }
  __device__ int code_of(const SgMeta*, int val, int& x) const {
    x = 0;
    return val;
  }
  __device__ const float* row(int code) const {
    return code >= 0 ? d_sums + (int64_t)code * w : bwd_recv + (int64_t)(-code - 1) * stride;
  }
  __device__ float scale(int, int) const { return 1.f; }
  __device__ float extra_val(int, int) const { return 0.f; }
  __device__ int64_t self_row(const SgMeta* meta, int64_t U) const {
    const int p = grouped[voff_lm1 + U];
    if (p >= meta->nV[l]) return -1;
    return meta->own_off[l][d] + rank[voff_l + p];
  }
  template <int VEC>
  __device__ void finish_vec(int64_t U, int64_t v, int col, const float* acc, float) const {
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
      if (col + k >= w) break;
      float val = acc[k];
      if (v >= 0) val += d_self[v * w + col + k];
      d_prev[U * w + col + k] = val;
    }
  }
};

struct GatPol {
  static constexpr bool kExtra = true;
  int l, d, dout, heads, g, dnc_stride;
  int64_t voff_lm1, voff_l, pbase_l;
  const int32_t* grouped;
  const int32_t* rank;
  const int32_t* contrib;
  const int32_t* ldst;
  const int32_t* sendpos;
  const float* alpha;
  const float* d_pre;
  const float* dnc;
  const float* dnc_recv;
  const float* dt_loc;
  const float* dt_recv;
  const float* a_src;
  const float* a_dst;
  float* d_z;
  float* ds;
  float* dt_tot;

  __device__ int width() const { return dout; }
  __device__ int extra() const { return heads; }
  __device__ int code_of(const SgMeta* meta, int x, int& xo) const {
    xo = x;
    const int q = ldst[x];
    const int n_own = meta->n_own[l][d];
    if (q < n_own) return meta->own_off[l][d] + q;
    return -1 - sendpos[pbase_l + meta->ref_off[l][d] + (q - n_own)];
  }
  __device__ const float* row(int code) const {
    return code >= 0 ? dnc + (int64_t)code * (dout + heads) : dnc_recv + (int64_t)(-code - 1) * dnc_stride;
  }
  __device__ float scale(int x, int col) const { return alpha[(int64_t)x * heads + col / (dout / heads)]; }
  __device__ float extra_val(int x, int h) const { return d_pre[(int64_t)x * heads + h]; }
  __device__ int64_t self_row(const SgMeta* meta, int64_t U) const {
    const int p = grouped[voff_lm1 + U];
    if (p >= meta->nV[l]) return -1;
    return meta->own_off[l][d] + rank[voff_l + p];
  }
  // the VEC columns col.. lie in one head (d_head % VEC == 0)
  template <int VEC>
  __device__ void finish_vec(int64_t U, int64_t v, int col, const float* acc, float dsv) const {
    const int dh = dout / heads, h = col / dh;
    float dt = 0.f;
    if (v >= 0) {
      dt = dt_loc[v * heads + h];
      const int* cb = contrib + (int64_t)g * voff_l + v * g;
      for (int s = 0; g > 1 && s < g; ++s) {
        const int rs = cb[s];
        if (rs >= 0) dt += dt_recv[(int64_t)rs * heads + h];
      }
    }
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
      if (col + k >= dout) break;
      float val = fmaf(dsv, a_src[col + k], acc[k]);
      if (v >= 0) val = fmaf(dt, a_dst[col + k], val);
      d_z[U * dout + col + k] = val;
    }
    if (col % dh == 0) {
      ds[U * heads + h] = dsv;
      if (v >= 0) dt_tot[v * heads + h] = dt;
    }
  }
};

// ---------------------------------------------------------------- K1: pieces
// A TEAM of LPR lanes (LPR * VEC >= width) takes one task, 32 / LPR teams per
// warp. Round structure is warp-uniform (max piece length over the warp), so
// the team shuffles never diverge; the self-row lookup is issued up front so
// its latency overlaps the edge loads.
template <class P, int VEC, int LPR>
__global__ void __launch_bounds__(256) k_tspmm_pieces(const SgMeta* __restrict__ meta, P pol, TsGeom t) {
  SG_PDL_ENTRY();
  constexpr int TPW = 32 / LPR;  // teams per warp
  const int lane = threadIdx.x & 31, lr = lane % LPR;
  const int W = pol.width(), X = pol.extra();
  const int col = lr * VEC;
  const bool colok = col < W;
  const int dh = X > 0 ? W / X : W;
  const int hl = colok ? col / dh : 0;
  const bool hlead = X > 0 && colok && col % dh == 0;
  int64_t P0;
  int n;
  layer_span(meta, t.l, t.d, t.lmin, P0, n);
  const int n_prev = meta->n_own[t.l - 1][t.d];
  const int prev0 = meta->own_off[t.l - 1][t.d];
  const int nch = (n + TC - 1) / TC;
  const int64_t ntask = (int64_t)n_prev + nch;
  const int64_t team0 = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * TPW;
  const int64_t nteam = (((int64_t)gridDim.x * blockDim.x) >> 5) * TPW;
  const int tw = lane / LPR;
  for (int64_t wbase = team0; wbase < ntask; wbase += nteam) {  // warp-uniform
    const int64_t task = wbase + tw;
    int64_t U = 0, p = 0, chunk = 0, v = -1;
    int cnt = 0, slot = 0;
    bool complete = false, live = false;
    if (task < n_prev) {
      live = true;
      U = prev0 + task;
      v = pol.self_row(meta, U);
      const int64_t key = t.key_base + U;
      const int b = t.srcbeg[key], e = t.srcend[key];
      complete = true;
      if (e > b) {
        chunk = (b - P0) / TC;
        const int64_t B1 = P0 + (chunk + 1) * TC;
        p = b;
        cnt = (int)(min((int64_t)e, B1) - b);
        complete = e <= B1;
        slot = b == P0 + chunk * TC ? 0 : 1;
      }
    } else if (task < ntask) {
      chunk = task - n_prev;
      const int64_t pos = P0 + chunk * TC;
      if (chunk > 0) {
        const uint32_t k = t.keys[pos];
        if (t.keys[pos - 1] == k) {  // chunk starts inside a row: continuation piece
          live = true;
          U = (int64_t)k - t.key_base;
          p = pos;
          cnt = (int)(min((int64_t)t.srcend[k], pos + TC) - pos);
        }
      }
    }
    float acc[VEC];
#pragma unroll
    for (int k = 0; k < VEC; ++k) acc[k] = 0.f;
    float dsv = 0.f;
    const int maxcnt = __reduce_max_sync(FULL, cnt);
    for (int base = 0; base < maxcnt; base += LPR) {
      int code = 0, x = 0;
      if (base + lr < cnt) code = pol.code_of(meta, t.vals[p + base + lr], x);
      const int nb = min(LPR, maxcnt - base);
#pragma unroll 4
      for (int k = 0; k < nb; ++k) {
        const int ck = __shfl_sync(FULL, code, k, LPR);
        const int xk = __shfl_sync(FULL, x, k, LPR);
        if (base + k < cnt) {
          if (colok) {
            const float* r = pol.row(ck) + col;
            const float sc = pol.scale(xk, col);
            if constexpr (VEC >= 4) {
#pragma unroll
              for (int q4 = 0; q4 < VEC / 4; ++q4) {
                const float4 v4 = *reinterpret_cast<const float4*>(r + 4 * q4);
                acc[4 * q4 + 0] = fmaf(sc, v4.x, acc[4 * q4 + 0]);
                acc[4 * q4 + 1] = fmaf(sc, v4.y, acc[4 * q4 + 1]);
                acc[4 * q4 + 2] = fmaf(sc, v4.z, acc[4 * q4 + 2]);
                acc[4 * q4 + 3] = fmaf(sc, v4.w, acc[4 * q4 + 3]);
              }
            } else {
              acc[0] = fmaf(sc, *r, acc[0]);
            }
          }
          if (P::kExtra && hlead) dsv += pol.extra_val(xk, hl);
        }
      }
    }
    // every lane of a head needs its head's ds: take it from the head lead
    const float dsh = P::kExtra ? __shfl_sync(FULL, dsv, (hl * dh) / VEC, LPR) : 0.f;
    if (!live) continue;
    if (complete) {
      if (colok) pol.template finish_vec<VEC>(U, v, col, acc, dsh);
    } else {
      float* dst = t.part + (chunk * 2 + slot) * t.ws;
      if (colok) {
#pragma unroll
        for (int k = 0; k < VEC; ++k)
          if (col + k < W) dst[col + k] = acc[k];
      }
      if (P::kExtra && hlead) dst[W + hl] = dsv;
    }
  }
}

// ---------------------------------------------------------------- K2: rows that span chunks
template <class P, int VEC>
__global__ void __launch_bounds__(256) k_tspmm_spans(const SgMeta* __restrict__ meta, P pol, TsGeom t) {
  SG_PDL_ENTRY();
  extern __shared__ __align__(16) float smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int WS = t.ws, W = pol.width(), X = pol.extra(), WX = W + X;
  float* R = smem + warp * WS;
  int64_t P0;
  int n;
  layer_span(meta, t.l, t.d, t.lmin, P0, n);
  const int nch = (n + TC - 1) / TC;
  for (int c = blockIdx.x * TWARPS + warp; c < nch; c += gridDim.x * TWARPS) {
    const int64_t last = P0 + (int64_t)c * TC + TC - 1;
    if (last + 1 >= P0 + n) continue;
    const uint32_t k = t.keys[last];
    if (t.keys[last + 1] != k) continue;  // nothing spans out of this chunk
    const int b = t.srcbeg[k], e = t.srcend[k];
    if (b < P0 + (int64_t)c * TC) continue;  // started in an earlier chunk: not ours
    const int ce = (int)((e - 1 - P0) / TC);
    const int slot0 = b == P0 + (int64_t)c * TC ? 0 : 1;
    for (int col = lane; col < WX; col += 32) {
      float acc = t.part[((int64_t)c * 2 + slot0) * WS + col];
#pragma unroll 4
      for (int cc = c + 1; cc <= ce; ++cc) acc += t.part[(int64_t)cc * 2 * WS + col];
      R[col] = acc;
    }
    __syncwarp();
    const int64_t U = (int64_t)k - t.key_base;
    const int64_t v = pol.self_row(meta, U);
    const int dh = X > 0 ? W / X : W;
    for (int c4 = lane * VEC; c4 < W; c4 += 32 * VEC)
      pol.template finish_vec<VEC>(U, v, c4, R + c4, X > 0 ? R[W + c4 / dh] : 0.f);
    __syncwarp();
  }
}

template <class P, int VEC, int LPR>
int launch_pieces(const SgMeta* meta, const P& pol, const TsGeom& t, int64_t max_edges, int64_t max_rows,
                  cudaStream_t st) {
  const int64_t chunks = (max_edges + TC - 1) / TC;
  const int64_t tasks = max_rows + chunks;
  if (tasks <= 0) return SG_OK;
  const int64_t warps = div_up(tasks, 32 / LPR);
  ::sg::launch(k_tspmm_pieces<P, VEC, LPR>, clamp_grid(div_up(warps, TWARPS), kSMs * 16), 256, 0, st, meta, pol, t);
  SG_CHECK_LAUNCH("k_tspmm_pieces");
  if (chunks > 0) {
    const size_t smem2 = sizeof(float) * (size_t)TWARPS * t.ws;
    ::sg::launch(k_tspmm_spans<P, VEC>, clamp_grid(div_up(chunks, TWARPS), kSMs * 8), 256, smem2, st, meta, pol, t);
    SG_CHECK_LAUNCH("k_tspmm_spans");
  }
  return SG_OK;
}

// VEC = columns per lane (1, or 4/8/16 = 1/2/4 float4s, all inside one head);
// LPR = smallest power of two with LPR * VEC >= width.
template <class P, int VEC>
int launch_vec(const SgMeta* meta, const P& pol, const TsGeom& t, int width, int64_t max_edges,
               int64_t max_rows, cudaStream_t st) {
  int lanes = 1;
  while (lanes * VEC < width) lanes <<= 1;
  switch (lanes) {
    case 1: return launch_pieces<P, VEC, 1>(meta, pol, t, max_edges, max_rows, st);
    case 2: return launch_pieces<P, VEC, 2>(meta, pol, t, max_edges, max_rows, st);
    case 4: return launch_pieces<P, VEC, 4>(meta, pol, t, max_edges, max_rows, st);
    case 8: return launch_pieces<P, VEC, 8>(meta, pol, t, max_edges, max_rows, st);
    case 16: return launch_pieces<P, VEC, 16>(meta, pol, t, max_edges, max_rows, st);
    case 32: return launch_pieces<P, VEC, 32>(meta, pol, t, max_edges, max_rows, st);
    default:
      set_error("tspmm: width too large for one warp");
      return SG_ERR_ARG;
  }
}

// `unit` = largest column group a lane may own (the head width for GAT, the
// row width for SAGE); aligned rows take 16 columns per lane when possible,
// keeping >= 4 lanes per team.
template <class P>
int launch_tspmm(const SgMeta* meta, const P& pol, const TsGeom& t, bool aligned, int width, int unit,
                 int64_t max_edges, int64_t max_rows, cudaStream_t st) {
  if (aligned) {
    if (unit % 16 == 0 && width >= 64) return launch_vec<P, 16>(meta, pol, t, width, max_edges, max_rows, st);
    if (unit % 8 == 0 && width >= 32) return launch_vec<P, 8>(meta, pol, t, width, max_edges, max_rows, st);
    if (unit % 4 == 0) return launch_vec<P, 4>(meta, pol, t, width, max_edges, max_rows, st);
  }
  return launch_vec<P, 1>(meta, pol, t, width, max_edges, max_rows, st);
}

int ws_cols(int w, int x) { return (w + x + 3) / 4 * 4; }

}  // namespace

extern "C" int64_t sg_tspmm_part_floats(int64_t max_edges, int32_t width, int32_t extra) {
  if (max_edges <= 0) return 0;
  return ((max_edges + TC - 1) / TC) * 2 * (int64_t)ws_cols(width, extra);
}

extern "C" int sg_sage_scatter_bwd_lb(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                                      int32_t w, const float* d_self, const float* d_sums,
                                      const float* bwd_recv, int32_t recv_stride, const uint32_t* keys,
                                      const int32_t* enc, const int32_t* srcbeg, const int32_t* srcend,
                                      int64_t key_base, int32_t lmin, float* part, int64_t max_edges,
                                      float* d_prev, int64_t max_rows, void* stream) {
  SG_REQUIRE(split_ws && lay, "sage_scatter_bwd_lb: null workspace");
  const char* base = (const char*)split_ws;
  const SgSplitLayout& y = *lay;
  SG_REQUIRE(l >= 2 && l <= y.L && d >= 0 && d < y.g && lmin >= 1 && lmin <= l,
             "sage_scatter_bwd_lb: bad layer/device");
  SG_REQUIRE(w >= 1 && ws_cols(w, 0) <= 192, "sage_scatter_bwd_lb: width must be 1..192");
  SG_REQUIRE(keys && enc && srcbeg && srcend && d_prev && (part || max_edges <= 0),
             "sage_scatter_bwd_lb: null pointer");
  SagePol p;
  memset(&p, 0, sizeof(p));
  p.l = l; p.d = d; p.w = w; p.stride = recv_stride;
  p.voff_lm1 = y.voff[l - 1]; p.voff_l = y.voff[l];
  p.grouped = (const int32_t*)(base + y.o_grouped);
  p.rank = (const int32_t*)(base + y.o_rank);
  p.d_self = d_self; p.d_sums = d_sums; p.bwd_recv = bwd_recv; p.d_prev = d_prev;
  TsGeom t{l, d, lmin, ws_cols(w, 0), key_base, keys, enc, srcbeg, srcend, part};
  const bool aligned = w % 4 == 0 && (recv_stride % 4 == 0 || y.g == 1);
  return launch_tspmm((const SgMeta*)(base + y.o_meta), p, t, aligned, w, w, max_edges, max_rows,
                      (cudaStream_t)stream);
}

extern "C" int sg_gat_bwd_src_lb(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                                 int32_t dout, int32_t heads, const uint32_t* keys, const int32_t* perm,
                                 const int32_t* srcbeg, const int32_t* srcend, int64_t key_base, int32_t lmin,
                                 const float* alpha, const float* d_pre, const float* dnc,
                                 const float* dnc_recv, int32_t dnc_stride, const float* dt_loc,
                                 const float* dt_recv, const float* a_src, const float* a_dst, float* d_z,
                                 float* ds, float* dt_tot, float* part, int64_t max_edges, int64_t max_rows,
                                 void* stream) {
  SG_REQUIRE(split_ws && lay, "gat_bwd_src_lb: null workspace");
  const char* base = (const char*)split_ws;
  const SgSplitLayout& y = *lay;
  SG_REQUIRE(l >= 1 && l <= y.L && d >= 0 && d < y.g && lmin >= 1 && lmin <= l,
             "gat_bwd_src_lb: bad layer/device");
  SG_REQUIRE(heads >= 1 && dout % heads == 0, "gat: dout must be a multiple of heads");
  SG_REQUIRE(ws_cols(dout, heads) <= 192, "gat_bwd_src_lb: dout + heads must be <= 192");
  SG_REQUIRE(keys && perm && srcbeg && srcend && d_z && ds && (part || max_edges <= 0),
             "gat_bwd_src_lb: null pointer");
  GatPol p;
  memset(&p, 0, sizeof(p));
  p.l = l; p.d = d; p.dout = dout; p.heads = heads; p.g = y.g; p.dnc_stride = dnc_stride;
  p.voff_lm1 = y.voff[l - 1]; p.voff_l = y.voff[l]; p.pbase_l = y.pbase[l];
  p.grouped = (const int32_t*)(base + y.o_grouped);
  p.rank = (const int32_t*)(base + y.o_rank);
  p.contrib = (const int32_t*)(base + y.o_contrib);
  p.ldst = (const int32_t*)(base + y.o_ldst);
  p.sendpos = (const int32_t*)(base + y.o_sendpos);
  p.alpha = alpha; p.d_pre = d_pre; p.dnc = dnc; p.dnc_recv = dnc_recv;
  p.dt_loc = dt_loc; p.dt_recv = dt_recv; p.a_src = a_src; p.a_dst = a_dst;
  p.d_z = d_z; p.ds = ds; p.dt_tot = dt_tot;
  TsGeom t{l, d, lmin, ws_cols(dout, heads), key_base, keys, perm, srcbeg, srcend, part};
  const int dh = dout / heads;
  const bool aligned = dh % 4 == 0 && (dout + heads) % 4 == 0 && (dnc_stride % 4 == 0 || y.g == 1);
  return launch_tspmm((const SgMeta*)(base + y.o_meta), p, t, aligned, dout, dh, max_edges, max_rows,
                      (cudaStream_t)stream);
}

}  // namespace sg
