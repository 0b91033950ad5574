// Online splitter on the GPU — replaces split_minibatch (scheduler.py:164-254).
//
// All g devices' splits are computed from the replicated sample in ~15
// launches, with no host synchronisation:
//   k_meta_init      header -> SgMeta (zero counts)
//   k_owner_keys     dev = asn[gid] for every position of every layer (:180),
//                    load key (cached ? g : dev) for layer 0 (:193-203)
//   ms_* (positions) stable g-way multisplit per layer = _group_by (:157-161):
//                    local_of_pos (:184-190), owned lists, n_owned, load lists
//   k_edge_keys      source device of each edge (:224-227); cross edges set
//                    bit `s` of the destination's pair mask
//   ms_* (edges)     stable grouping of edges by source device
//   k_ref_bits / k_ref_scan / k_ref_chunks / k_ref_rank
//                    reference vertices ranked by GLOBAL ID (:228-232) via a
//                    popcount-prefix over an n-bit bitmap (no sort)
//   k_pair_count / k_pair_scan / k_pair_scatter
//                    ShufflePlan entries (l,s,o) in gid order (:244-252), the
//                    holder ref rows, send slots, receive slots and the
//                    owner-side combine table
//   k_local_edges    edges_src / edges_dst / self_rows (:233-243) and the
//                    CSR-by-destination runs of every device
// Ordering is stable by construction (warp match/ballot ranks, tiles in
// order), so the integer outputs are bit-identical to the reference.
#include <algorithm>
#include <cstring>

#include "common.cuh"

namespace sg {

namespace {

constexpr int MS_T = 2048;       // multisplit tile (elements)
constexpr int MS_THREADS = 256;  // 8 warps x 8 rounds x 32
constexpr int MS_ROUNDS = MS_T / MS_THREADS;
constexpr int PAIR_T = 256;      // pair tile (1 element / thread)
constexpr int CHUNK_WORDS = 1024;
constexpr int MAXSEG = SG_MAXL + 2;
constexpr int MAXKEY = SG_MAXG + 1;
constexpr int MAXKQ = SG_MAXG * SG_MAXG + SG_MAXG;

struct SegDesc {
  int nseg;
  int nkeys;
  int mode;  // 0: position segments (lengths meta->nV[s], load segment nV[0]); 1: edges (nE[s])
  int64_t beg[MAXSEG + 1];
  int64_t tile_beg[MAXSEG + 1];
};

__device__ __forceinline__ int64_t seg_end(const SegDesc& sd, const SgMeta* meta, int s) {
  int64_t len;
  if (sd.mode == 0) len = (s <= meta->L) ? meta->nV[s] : meta->nV[0];
  else len = meta->nE[s];
  return sd.beg[s] + len;
}

struct MetaHeader {
  int32_t L, g, dst_grouped, pad;
  int64_t nV[SG_MAXL + 1];
  int64_t nE[SG_MAXL];
  int64_t voff[SG_MAXL + 2];
  int64_t eoff[SG_MAXL + 1];
  int64_t rbase[SG_MAXL + 1];  // row-space base of edge layer l at [l-1]
};

__device__ __forceinline__ int seg_of_tile(const SegDesc& sd, int64_t t) {
  int s = 0;
  while (s + 1 < sd.nseg && sd.tile_beg[s + 1] <= t) ++s;
  return s;
}

__device__ __forceinline__ int layer_of(const int64_t* off, int nl, int64_t i) {
  int l = 0;
  while (l + 1 < nl && off[l + 1] <= i) ++l;
  return l;
}

// Header (capacity offsets) + ACTUAL sizes (device array nV[0..L], nE[0..L-1],
// or the capacities when sizes == nullptr) -> SgMeta with zero counts.
__global__ void k_meta_init(MetaHeader h, const int64_t* __restrict__ sizes, SgMeta* meta) {
  SG_PDL_ENTRY();
  int32_t* w = reinterpret_cast<int32_t*>(meta);
  const int nwords = sizeof(SgMeta) / 4;
  for (int i = threadIdx.x; i < nwords; i += blockDim.x) w[i] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    meta->L = h.L;
    meta->g = h.g;
    meta->dst_grouped = h.dst_grouped;
    for (int l = 0; l <= SG_MAXL; ++l) {
      int64_t v = h.nV[l];
      if (sizes && l <= h.L) v = min(v, sizes[l]);
      meta->nV[l] = v;
    }
    for (int l = 0; l < SG_MAXL; ++l) {
      int64_t v = h.nE[l];
      if (sizes && l < h.L) v = min(v, sizes[h.L + 1 + l]);
      meta->nE[l] = v;
    }
    for (int l = 0; l < SG_MAXL + 2; ++l) meta->voff[l] = h.voff[l];
    for (int l = 0; l < SG_MAXL + 1; ++l) meta->eoff[l] = h.eoff[l];
  }
}

// dev of every position; layer-0 load key appended after nVtot.
__global__ void k_owner_keys(const int32_t* __restrict__ V, MetaHeader h, int64_t nVtot,
                             int64_t nV0, const uint8_t* __restrict__ asn, int64_t n_asn,
                             const uint32_t* __restrict__ cache_bits, int g,
                             uint8_t* __restrict__ keys, SgMeta* meta) {
  SG_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nVtot;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int l = layer_of(h.voff, h.L + 1, i);
    if (i - h.voff[l] >= meta->nV[l]) continue;  // capacity padding
    int32_t gid = V[i];
    uint8_t dv = 0;
    if (gid < 0 || gid >= n_asn) {
      atomicOr(&meta->err, SG_ERR_MISSING_VERTEX);
    } else {
      dv = asn[gid];
    }
    keys[i] = dv;
    if (i < nV0) {
      bool cached = cache_bits != nullptr && gid >= 0 && gid < n_asn &&
                    ((cache_bits[gid >> 5] >> (gid & 31)) & 1u);
      keys[nVtot + i] = cached ? (uint8_t)g : dv;
    }
  }
}

// ---- generic stable multisplit (counting sort by small key, per segment) ----

__global__ void __launch_bounds__(MS_THREADS) ms_count(const uint8_t* __restrict__ keys, SegDesc sd,
                                                       const SgMeta* __restrict__ meta,
                                                       int32_t* __restrict__ tilecnt) {
  SG_PDL_ENTRY();
  __shared__ int cnt[MAXKEY];
  const int64_t t = blockIdx.x;
  const int s = seg_of_tile(sd, t);
  const int64_t base = sd.beg[s] + (t - sd.tile_beg[s]) * MS_T;
  const int64_t end = min(base + MS_T, seg_end(sd, meta, s));
  if (threadIdx.x < sd.nkeys) cnt[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t i = base + threadIdx.x; i < end; i += MS_THREADS) atomicAdd(&cnt[keys[i]], 1);
  __syncthreads();
  if (threadIdx.x < sd.nkeys) tilecnt[t * sd.nkeys + threadIdx.x] = cnt[threadIdx.x];
}

// One block per segment: exclusive scan over the segment's tiles for every
// key (warp per key), segment totals and key offsets. mode 0: positions
// (segments 0..L = layers -> n_own/own_off, segment L+1 -> n_load/load_off);
// mode 1: edges (segment l-1 -> n_edge/edge_off).
__global__ void ms_scan(SegDesc sd, const int32_t* __restrict__ tilecnt,
                        int32_t* __restrict__ tilebase, int32_t* __restrict__ keyoff, int mode,
                        SgMeta* meta) {
  SG_PDL_ENTRY();
  __shared__ int tot[MAXKEY];
  const int s = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t0 = sd.tile_beg[s], t1 = sd.tile_beg[s + 1];
  for (int k = warp; k < sd.nkeys; k += blockDim.x >> 5) {
    int run = 0;
    for (int64_t tb = t0; tb < t1; tb += 32) {
      int64_t t = tb + lane;
      int v = (t < t1) ? tilecnt[t * sd.nkeys + k] : 0;
      int inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      if (t < t1) tilebase[t * sd.nkeys + k] = run + inc - v;
      run += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) tot[k] = run;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    const int g = meta->g;
    const int L = meta->L;
    for (int k = 0; k < sd.nkeys; ++k) {
      keyoff[s * sd.nkeys + k] = acc;
      if (mode == 0 && s <= L && k < g) {
        meta->n_own[s][k] = tot[k];
        meta->own_off[s][k] = acc;
      } else if (mode == 0 && s == L + 1 && k < g) {
        meta->n_load[k] = tot[k];
        meta->load_off[k] = acc;
      } else if (mode == 1 && k < g) {
        meta->n_edge[s][k] = tot[k];
        meta->edge_off[s][k] = acc;
      }
      acc += tot[k];
    }
    if (mode == 0 && s <= L) meta->own_off[s][g] = acc;
    if (mode == 0 && s == L + 1) meta->load_off[g] = acc - tot[g];
    if (mode == 1) meta->edge_off[s][g] = acc;
  }
}

__global__ void __launch_bounds__(MS_THREADS) ms_scatter(const uint8_t* __restrict__ keys, SegDesc sd,
                                                         const SgMeta* __restrict__ meta,
                                                         const int32_t* __restrict__ tilebase,
                                                         const int32_t* __restrict__ keyoff,
                                                         int32_t* __restrict__ rank_out,
                                                         int32_t* __restrict__ grouped_out) {
  SG_PDL_ENTRY();
  __shared__ int wcnt[MS_THREADS / 32][MAXKEY];
  __shared__ int wbase[MS_THREADS / 32][MAXKEY];
  const int64_t t = blockIdx.x;
  const int s = seg_of_tile(sd, t);
  const int64_t sbeg = sd.beg[s];
  const int64_t base = sbeg + (t - sd.tile_beg[s]) * MS_T;
  const int64_t end = min(base + MS_T, seg_end(sd, meta, s));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = sd.nkeys;
  for (int k = lane; k < nk; k += 32) wcnt[warp][k] = 0;
  __syncwarp();
  int myk[MS_ROUNDS], myr[MS_ROUNDS];
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int j = 0; j < MS_ROUNDS; ++j) {
    const int64_t idx = base + warp * (32 * MS_ROUNDS) + j * 32 + lane;
    const bool valid = idx < end;
    const int k = valid ? (int)keys[idx] : 255;
    const unsigned peers = __match_any_sync(0xffffffffu, k);
    const int r = __popc(peers & lt);
    const int prior = valid ? wcnt[warp][k] : 0;
    __syncwarp();
    if (valid && r == 0) wcnt[warp][k] = prior + __popc(peers);
    __syncwarp();
    myk[j] = k;
    myr[j] = prior + r;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < nk; k += MS_THREADS) {
    int run = 0;
#pragma unroll
    for (int w = 0; w < MS_THREADS / 32; ++w) {
      wbase[w][k] = run;
      run += wcnt[w][k];
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < MS_ROUNDS; ++j) {
    const int64_t idx = base + warp * (32 * MS_ROUNDS) + j * 32 + lane;
    if (idx < end) {
      const int k = myk[j];
      const int rnk = tilebase[t * nk + k] + wbase[warp][k] + myr[j];
      if (rank_out) rank_out[idx] = rnk;
      grouped_out[sbeg + keyoff[s * nk + k] + rnk] = (int32_t)(idx - sbeg);
    }
  }
}

// ---- edges: source-device key + pair masks ----
__global__ void k_edge_keys(const int32_t* __restrict__ esrc, const int32_t* __restrict__ edst,
                            MetaHeader h, const SgMeta* __restrict__ meta,
                            const uint8_t* __restrict__ keys, uint8_t* __restrict__ ekey,
                            uint32_t* __restrict__ pmask, int32_t* __restrict__ egrouped_identity) {
  SG_PDL_ENTRY();
  const int64_t n = h.eoff[h.L];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int li = layer_of(h.eoff, h.L, e);  // edge layer l = li + 1
    if (e - h.eoff[li] >= meta->nE[li]) continue;  // capacity padding
    const int32_t src = esrc[e], dst = edst[e];
    const uint8_t sd = keys[h.voff[li] + src];
    const uint8_t dd = keys[h.voff[li + 1] + dst];
    ekey[e] = sd;
    if (sd != dd) atomicOr(&pmask[h.voff[li + 1] + dst], 1u << sd);
    if (egrouped_identity) egrouped_identity[e] = (int32_t)(e - h.eoff[li]);
  }
}

// g == 1: one device owns every edge, grouping is the identity.
__global__ void k_single_edge_meta(SgMeta* meta) {
  SG_PDL_ENTRY();
  const int li = threadIdx.x;
  if (li < meta->L) {
    meta->n_edge[li][0] = (int32_t)meta->nE[li];
    meta->edge_off[li][0] = 0;
    meta->edge_off[li][1] = (int32_t)meta->nE[li];
  }
}

// ---- reference vertices in global-id order (bitmap popcount prefix) ----
__global__ void k_ref_bits(const int32_t* __restrict__ V, MetaHeader h,
                           const uint32_t* __restrict__ pmask, uint32_t* __restrict__ bm,
                           int64_t words, int clear) {
  SG_PDL_ENTRY();
  const int64_t b = h.voff[1], e = h.voff[h.L + 1];
  for (int64_t i = b + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (pmask[i] == 0) continue;
    const int l = layer_of(h.voff, h.L + 1, i);
    const int32_t gid = V[i];
    uint32_t* w = &bm[(int64_t)(l - 1) * words + (gid >> 5)];
    if (clear) *w = 0u; else atomicOr(w, 1u << (gid & 31));
  }
}

// Per 1024-word chunk: exclusive popcount prefix of each word + chunk total.
__global__ void __launch_bounds__(256) k_ref_scan(const uint32_t* __restrict__ bm,
                                                  int32_t* __restrict__ wpre,
                                                  int32_t* __restrict__ ctot) {
  SG_PDL_ENTRY();
  __shared__ int wsum[8];
  const int64_t c = blockIdx.x;
  const int64_t w0 = c * CHUNK_WORDS + threadIdx.x * 4;
  uint4 v = *reinterpret_cast<const uint4*>(bm + w0);
  int p0 = __popc(v.x), p1 = __popc(v.y), p2 = __popc(v.z), p3 = __popc(v.w);
  int tsum = p0 + p1 + p2 + p3;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int inc = tsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  int wpref = 0;
  for (int w = 0; w < warp; ++w) wpref += wsum[w];
  int ex = wpref + inc - tsum;
  int4 out = make_int4(ex, ex + p0, ex + p0 + p1, ex + p0 + p1 + p2);
  *reinterpret_cast<int4*>(wpre + w0) = out;
  if (threadIdx.x == 255) ctot[c] = wpref + inc;
}

// Single block: per layer, exclusive prefix of chunk totals (in place) and
// the number of distinct reference vertices.
__global__ void k_ref_chunks(int32_t* __restrict__ ctot, int64_t chunks_per_layer, int L,
                             SgMeta* meta) {
  SG_PDL_ENTRY();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int l = 1 + warp; l <= L; l += blockDim.x >> 5) {
    int32_t* c = ctot + (int64_t)(l - 1) * chunks_per_layer;
    int run = 0;
    for (int64_t b = 0; b < chunks_per_layer; b += 32) {
      int64_t i = b + lane;
      int v = i < chunks_per_layer ? c[i] : 0;
      int inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      if (i < chunks_per_layer) c[i] = run + inc - v;
      run += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) meta->n_uniq[l] = run;
  }
}

__global__ void k_ref_rank(const int32_t* __restrict__ V, MetaHeader h,
                           const uint32_t* __restrict__ pmask, const uint32_t* __restrict__ bm,
                           const int32_t* __restrict__ wpre, const int32_t* __restrict__ cpre,
                           int64_t words, int32_t* __restrict__ uorder) {
  SG_PDL_ENTRY();
  const int64_t b = h.voff[1], e = h.voff[h.L + 1];
  const int64_t cpl = words / CHUNK_WORDS;
  for (int64_t i = b + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (pmask[i] == 0) continue;
    const int l = layer_of(h.voff, h.L + 1, i);
    const int32_t gid = V[i];
    const int64_t wi = (int64_t)(l - 1) * words + (gid >> 5);
    const int r = cpre[(int64_t)(l - 1) * cpl + ((gid >> 5) / CHUNK_WORDS)] + wpre[wi] +
                  __popc(bm[wi] & ((1u << (gid & 31)) - 1u));
    uorder[h.voff[l] + r] = (int32_t)(i - h.voff[l]);
  }
}

// ---- ShufflePlan: (holder s, owner o) entries in gid order ----
struct PairDesc {
  int L, g, kq;
  int64_t voff[SG_MAXL + 2];
  int64_t nV[SG_MAXL + 1];
  int64_t tile_beg[SG_MAXL + 2];  // tile_beg[l] for l = 1..L (index l), tile_beg[L+1] end
  int64_t pbase[SG_MAXL + 2];
};

__device__ __forceinline__ int layer_of_pair_tile(const PairDesc& pd, int64_t t) {
  int l = 1;
  while (l < pd.L && pd.tile_beg[l + 1] <= t) ++l;
  return l;
}

__global__ void __launch_bounds__(PAIR_T) k_pair_count(PairDesc pd, const SgMeta* __restrict__ meta,
                                                       const int32_t* __restrict__ uorder,
                                                       const uint32_t* __restrict__ pmask,
                                                       const uint8_t* __restrict__ keys,
                                                       int32_t* __restrict__ tilecnt) {
  SG_PDL_ENTRY();
  __shared__ int cnt[MAXKQ];
  const int64_t t = blockIdx.x;
  const int l = layer_of_pair_tile(pd, t);
  const int g = pd.g, kq = pd.kq;
  for (int k = threadIdx.x; k < kq; k += PAIR_T) cnt[k] = 0;
  __syncthreads();
  const int64_t r = (t - pd.tile_beg[l]) * PAIR_T + threadIdx.x;
  if (r < meta->n_uniq[l]) {
    const int32_t p = uorder[pd.voff[l] + r];
    const uint32_t m = pmask[pd.voff[l] + p];
    const int o = keys[pd.voff[l] + p];
    for (int s = 0; s < g; ++s)
      if ((m >> s) & 1u) {
        atomicAdd(&cnt[s * g + o], 1);
        atomicAdd(&cnt[g * g + s], 1);
      }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < kq; k += PAIR_T) tilecnt[t * kq + k] = cnt[k];
}

// Single block: per layer, exclusive tile scan per key (warp per key), then the
// plan's count matrix and every derived offset.
__global__ void k_pair_scan(PairDesc pd, const int32_t* __restrict__ tilecnt,
                            int32_t* __restrict__ tilebase, SgMeta* meta) {
  SG_PDL_ENTRY();
  __shared__ int tot[MAXKQ];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = pd.g, kq = pd.kq;
  for (int l = 1; l <= pd.L; ++l) {
    const int64_t t0 = pd.tile_beg[l], t1 = pd.tile_beg[l + 1];
    for (int k = warp; k < kq; k += nw) {
      int run = 0;
      for (int64_t tb = t0; tb < t1; tb += 32) {
        const int64_t t = tb + lane;
        const int v = t < t1 ? tilecnt[t * kq + k] : 0;
        int inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          int y = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += y;
        }
        if (t < t1) tilebase[t * kq + k] = run + inc - v;
        run += __shfl_sync(0xffffffffu, inc, 31);
      }
      if (lane == 0) tot[k] = run;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0;
      for (int s = 0; s < g; ++s) {
        meta->n_ref[l][s] = tot[g * g + s];
        meta->ref_off[l][s] = acc;
        int a2 = acc;
        for (int o = 0; o < g; ++o) {
          meta->cnt[l][s][o] = tot[s * g + o];
          meta->pair_off[l][s][o] = a2;
          a2 += tot[s * g + o];
        }
        acc += tot[g * g + s];
      }
      meta->ref_off[l][g] = acc;
      meta->npairs[l] = acc;
      int racc = 0;
      for (int o = 0; o < g; ++o) {
        meta->recv_off[l][o] = racc;
        int in = 0;
        for (int s = 0; s < g; ++s) {
          meta->recv_in[l][s][o] = in;
          in += tot[s * g + o];
        }
        racc += in;
      }
      meta->recv_off[l][g] = racc;
    }
    __syncthreads();
  }
}

struct PairOut {
  int32_t* pairs;
  int32_t* pair_hidx;
  int32_t* sendpos;
  int32_t* xfer;
  int32_t* recv_row;
  int32_t* refrank;
  int32_t* contrib;
};

__global__ void __launch_bounds__(PAIR_T) k_pair_scatter(PairDesc pd, const SgMeta* __restrict__ meta,
                                                         const int32_t* __restrict__ uorder,
                                                         const uint32_t* __restrict__ pmask,
                                                         const uint8_t* __restrict__ keys,
                                                         const int32_t* __restrict__ rank,
                                                         const int32_t* __restrict__ tilebase,
                                                         PairOut out) {
  SG_PDL_ENTRY();
  __shared__ int wcnt[PAIR_T / 32][MAXKQ];
  __shared__ int wbase[PAIR_T / 32][MAXKQ];
  const int64_t t = blockIdx.x;
  const int l = layer_of_pair_tile(pd, t);
  const int g = pd.g, kq = pd.kq;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = lane; k < kq; k += 32) wcnt[warp][k] = 0;
  __syncwarp();
  const int64_t r = (t - pd.tile_beg[l]) * PAIR_T + threadIdx.x;
  const bool valid = r < meta->n_uniq[l];
  const int32_t p = valid ? uorder[pd.voff[l] + r] : 0;
  const uint32_t m = valid ? pmask[pd.voff[l] + p] : 0u;
  const int o = valid ? (int)keys[pd.voff[l] + p] : 255;
  const unsigned peers = __match_any_sync(0xffffffffu, o);
  const unsigned lt = lanemask_lt();
  for (int s = 0; s < g; ++s) {
    const unsigned bs = __ballot_sync(0xffffffffu, (m >> s) & 1u);
    if (bs == 0) continue;
    const unsigned grp = bs & peers;
    if (((m >> s) & 1u) && (grp & lt) == 0) wcnt[warp][s * g + o] = __popc(grp);
    if (lane == 0) wcnt[warp][g * g + s] = __popc(bs);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < kq; k += PAIR_T) {
    int run = 0;
#pragma unroll
    for (int w = 0; w < PAIR_T / 32; ++w) {
      wbase[w][k] = run;
      run += wcnt[w][k];
    }
  }
  __syncthreads();
  const int64_t pb = pd.pbase[l];
  const int64_t vl = pd.voff[l];
  const int64_t nVl = pd.nV[l];
  const int q = valid ? rank[vl + p] : 0;
  const int orow = valid ? meta->own_off[l][o] + q : 0;
  const int64_t tb = t * kq;
  for (int s = 0; s < g; ++s) {
    const bool has = (m >> s) & 1u;
    const unsigned bs = __ballot_sync(0xffffffffu, has);  // all lanes participate
    if (!has) continue;
    const int kso = s * g + o, ks = g * g + s;
    const int pidx = tilebase[tb + kso] + wbase[warp][kso] + __popc(bs & peers & lt);
    const int rr = tilebase[tb + ks] + wbase[warp][ks] + __popc(bs & lt);
    const int slot = meta->pair_off[l][s][o] + pidx;
    const int rs = meta->recv_off[l][o] + meta->recv_in[l][s][o] + pidx;
    out.pairs[pb + slot] = p;
    out.pair_hidx[pb + slot] = rr;
    out.sendpos[pb + meta->ref_off[l][s] + rr] = slot;
    out.xfer[pb + slot] = rs;
    out.recv_row[pb + rs] = orow;
    out.refrank[(int64_t)g * vl + (int64_t)s * nVl + p] = rr;
    out.contrib[(int64_t)g * vl + (int64_t)orow * g + s] = rs;
  }
}

// ---- per-device local edges, self rows, CSR-by-destination runs ----
struct LocalOut {
  int32_t* lsrc;
  int32_t* ldst;
  int32_t* rowbeg;
  int32_t* rowend;
  int32_t* selfrow;
};

__global__ void k_local_edges(const int32_t* __restrict__ esrc, const int32_t* __restrict__ edst,
                              MetaHeader h, const SgMeta* __restrict__ meta,
                              const uint8_t* __restrict__ keys, const int32_t* __restrict__ rank,
                              const int32_t* __restrict__ grouped,
                              const int32_t* __restrict__ egrouped,
                              const int32_t* __restrict__ refrank, LocalOut out) {
  SG_PDL_ENTRY();
  const int g = h.g;
  const int64_t nE = h.eoff[h.L];
  const int64_t nS = h.voff[h.L + 1] - h.voff[1];  // owned positions of layers 1..L
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < nE + nS;
       x += (int64_t)gridDim.x * blockDim.x) {
    if (x < nE) {
      const int li = layer_of(h.eoff, h.L, x);  // layer l = li+1
      const int l = li + 1;
      const int64_t eo = h.eoff[li];
      const int i = (int)(x - eo);
      if (i >= meta->nE[li]) continue;  // capacity padding
      const int d = find_bucket(meta->edge_off[li], g, i);
      const int e = egrouped[eo + i];
      const int32_t src = esrc[eo + e], dst = edst[eo + e];
      const int64_t vl = h.voff[l];
      out.lsrc[eo + i] = rank[h.voff[l - 1] + src];
      const int od = keys[vl + dst];
      const int nown = meta->n_own[l][d];
      const int q = (od == d) ? rank[vl + dst]
                              : nown + refrank[(int64_t)g * vl + (int64_t)d * h.nV[l] + dst];
      out.ldst[eo + i] = q;
      if (h.dst_grouped) {
        const int ebeg = meta->edge_off[li][d], eend = meta->edge_off[li][d + 1];
        const int64_t R = h.rbase[li] + meta->own_off[l][d] + meta->ref_off[l][d] + q;
        if (i == ebeg || edst[eo + egrouped[eo + i - 1]] != dst) out.rowbeg[R] = i;
        if (i == eend - 1 || edst[eo + egrouped[eo + i + 1]] != dst) out.rowend[R] = i + 1;
      }
    } else {
      const int64_t y = x - nE + h.voff[1];
      const int l = layer_of(h.voff, h.L + 1, y);
      if (y - h.voff[l] >= meta->nV[l]) continue;  // capacity padding
      const int32_t p = grouped[y];
      out.selfrow[y] = rank[h.voff[l - 1] + p];
    }
  }
}

// g == 1 with no partial cache and destination-grouped edges: the split is the
// identity (_group_by with one key keeps everything in order), so one pass
// writes every array the executor reads.
__global__ void k_split_single(const int32_t* __restrict__ V, const int32_t* __restrict__ esrc,
                               const int32_t* __restrict__ edst, MetaHeader h, SgMeta* meta,
                               int64_t n_asn, int all_cached, int32_t* __restrict__ rank,
                               int32_t* __restrict__ grouped, int32_t* __restrict__ egrouped,
                               LocalOut out) {
  SG_PDL_ENTRY();
  const int L = h.L;
  const int64_t nVtot = h.voff[L + 1], nE = h.eoff[L];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int l = 0; l <= L; ++l) {
      meta->n_own[l][0] = (int32_t)meta->nV[l];
      meta->own_off[l][0] = 0;
      meta->own_off[l][1] = (int32_t)meta->nV[l];
    }
    for (int li = 0; li < L; ++li) {
      meta->n_edge[li][0] = (int32_t)meta->nE[li];
      meta->edge_off[li][0] = 0;
      meta->edge_off[li][1] = (int32_t)meta->nE[li];
    }
    const int32_t nl = all_cached ? 0 : (int32_t)meta->nV[0];
    meta->n_load[0] = nl;
    meta->load_off[0] = 0;
    meta->load_off[1] = nl;
  }
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < nVtot + nE;
       x += (int64_t)gridDim.x * blockDim.x) {
    if (x < nVtot) {
      const int l = layer_of(h.voff, L + 1, x);
      const int64_t p = x - h.voff[l];
      if (p >= meta->nV[l]) continue;
      const int32_t gid = V[x];
      if (gid < 0 || gid >= n_asn) atomicOr(&meta->err, SG_ERR_MISSING_VERTEX);
      rank[x] = (int32_t)p;
      grouped[x] = (int32_t)p;
      if (l >= 1) out.selfrow[x] = (int32_t)p;
      if (l == 0 && !all_cached) {
        rank[nVtot + p] = (int32_t)p;
        grouped[nVtot + p] = (int32_t)p;
      }
    } else {
      const int64_t y = x - nVtot;
      const int li = layer_of(h.eoff, L, y);
      const int i = (int)(y - h.eoff[li]);
      if (i >= meta->nE[li]) continue;
      const int32_t src = esrc[y], dst = edst[y];
      egrouped[y] = i;
      out.lsrc[y] = src;
      out.ldst[y] = dst;
      const int64_t R = h.rbase[li] + dst;
      if (i == 0 || edst[y - 1] != dst) out.rowbeg[R] = i;
      if (i == meta->nE[li] - 1 || edst[y + 1] != dst) out.rowend[R] = i + 1;
    }
  }
}

}  // namespace

// ---------------------------------------------------------------- host side

static int64_t align256(int64_t x) { return (x + 255) & ~int64_t(255); }

extern "C" int sg_split_layout(int32_t L, int32_t g, const int64_t* nV, const int64_t* nE,
                               int64_t n_vertices, SgSplitLayout* out) {
  SG_REQUIRE(L >= 1 && L <= SG_MAXL, "split: num_layers must be in [1, 8]");
  SG_REQUIRE(g >= 1 && g <= SG_MAXG, "split: num_devices must be in [1, 16]");
  SG_REQUIRE(n_vertices >= 0 && n_vertices < (int64_t(1) << 31), "split: n_vertices out of range");
  SgSplitLayout y;
  memset(&y, 0, sizeof(y));
  y.L = L;
  y.g = g;
  y.n_vertices = n_vertices;
  y.voff[0] = 0;
  for (int l = 0; l <= L; ++l) {
    SG_REQUIRE(nV[l] >= 0 && nV[l] < (int64_t(1) << 30), "split: layer too large");
    y.nV[l] = nV[l];
    y.voff[l + 1] = y.voff[l] + nV[l];
  }
  y.eoff[0] = 0;
  for (int l = 0; l < L; ++l) {
    SG_REQUIRE(nE[l] >= 0 && nE[l] < (int64_t(1) << 30), "split: layer too large");
    y.nE[l] = nE[l];
    y.eoff[l + 1] = y.eoff[l] + nE[l];
  }
  y.nVtot = y.voff[L + 1];
  y.nEtot = y.eoff[L];
  // pair-indexed arrays: upper bound min(|E^l|, (g-1)|V^l|) per layer
  y.pbase[0] = 0;
  y.pbase[1] = 0;
  for (int l = 1; l <= L; ++l) {
    int64_t P = (g == 1) ? 0 : std::min<int64_t>(nE[l - 1], (int64_t)(g - 1) * nV[l]);
    y.pbase[l + 1] = y.pbase[l] + P;
  }
  y.nPtot = y.pbase[L + 1];
  {
    int64_t acc = 0;
    for (int l = 1; l <= L; ++l) {
      y.rbase[l - 1] = acc;  // indexed by li = l-1
      acc += nV[l] + (y.pbase[l + 1] - y.pbase[l]);
    }
    y.rbase[L] = acc;
  }
  const int64_t rows_total = y.rbase[L];
  int64_t words = (n_vertices + 31) / 32;
  words = ((words + CHUNK_WORDS - 1) / CHUNK_WORDS) * CHUNK_WORDS;
  if (words == 0) words = CHUNK_WORDS;
  y.bm_words = words;
  // tiles
  int64_t pt = 0;
  for (int l = 0; l <= L; ++l) pt += (nV[l] + MS_T - 1) / MS_T;
  pt += (nV[0] + MS_T - 1) / MS_T;
  y.pos_tiles = pt;
  int64_t et = 0;
  for (int l = 0; l < L; ++l) et += (nE[l] + MS_T - 1) / MS_T;
  y.edge_tiles = et;
  int64_t qt = 0;
  for (int l = 1; l <= L; ++l) qt += (nV[l] + PAIR_T - 1) / PAIR_T;
  y.pair_tiles = qt;
  const int64_t kq = (int64_t)g * g + g;

  int64_t o = 0;
  auto take = [&](int64_t bytes) {
    int64_t r = o;
    o += align256(bytes > 0 ? bytes : 1);
    return r;
  };
  y.o_meta = take(sizeof(SgMeta));
  const int64_t npos = y.nVtot + nV[0];
  y.o_keys = take(npos);
  y.o_rank = take(4 * npos);
  y.o_grouped = take(4 * npos);
  y.o_ekey = take(y.nEtot);
  y.o_egrouped = take(4 * y.nEtot);
  y.o_lsrc = take(4 * y.nEtot);
  y.o_ldst = take(4 * y.nEtot);
  y.o_pmask = take(4 * y.nVtot);
  y.o_bitmap = take(4 * words * L);
  y.o_wpre = take(4 * words * L);
  y.o_ctot = take(4 * (words / CHUNK_WORDS) * L);
  y.o_uorder = take(4 * y.nVtot);
  y.o_refrank = take(4 * (int64_t)g * y.nVtot);
  y.o_contrib = take(4 * (int64_t)g * y.nVtot);
  y.o_pairs = take(4 * y.nPtot);
  y.o_pair_hidx = take(4 * y.nPtot);
  y.o_sendpos = take(4 * y.nPtot);
  y.o_xfer = take(4 * y.nPtot);
  y.o_recv_row = take(4 * y.nPtot);
  y.o_selfrow = take(4 * y.nVtot);
  y.o_rowbeg = take(4 * rows_total);
  y.o_rowend = take(4 * rows_total);
  const int64_t nseg_pos = L + 2, nseg_edge = L;
  y.o_tiles_pos = take(4 * (pt * (g + 1)));
  y.o_tilebase_pos = take(4 * (pt * (g + 1) + nseg_pos * (g + 1)));
  y.o_tiles_edge = take(4 * (et * g));
  y.o_tilebase_edge = take(4 * (et * g + nseg_edge * g));
  y.o_tiles_pair = take(4 * (qt * kq));
  y.o_tilebase_pair = take(4 * (qt * kq));
  y.total_bytes = o;
  *out = y;
  return SG_OK;
}

extern "C" int sg_split_run(void* ws, const SgSplitLayout* lay, const int32_t* V,
                            const int32_t* esrc, const int32_t* edst, const int64_t* sizes,
                            const uint8_t* asn, const uint32_t* cache_bits, int32_t flags,
                            void* stream) {
  const int32_t dst_grouped = flags & SG_SPLIT_DST_GROUPED;
  const int all_cached = (flags & SG_SPLIT_ALL_CACHED) ? 1 : 0;
  SG_REQUIRE(ws && lay, "split: null workspace");
  const SgSplitLayout& y = *lay;
  const int L = y.L, g = y.g;
  cudaStream_t st = (cudaStream_t)stream;
  char* base = (char*)ws;
  auto P8 = [&](int64_t o) { return (uint8_t*)(base + o); };
  auto P32 = [&](int64_t o) { return (int32_t*)(base + o); };
  auto U32 = [&](int64_t o) { return (uint32_t*)(base + o); };
  SgMeta* meta = (SgMeta*)(base + y.o_meta);

  MetaHeader h;
  memset(&h, 0, sizeof(h));
  h.L = L;
  h.g = g;
  h.dst_grouped = dst_grouped ? 1 : 0;
  for (int l = 0; l <= SG_MAXL; ++l) h.nV[l] = l <= L ? y.nV[l] : 0;
  for (int l = 0; l < SG_MAXL; ++l) h.nE[l] = l < L ? y.nE[l] : 0;
  for (int l = 0; l < SG_MAXL + 2; ++l) h.voff[l] = l <= L + 1 ? y.voff[l] : y.voff[L + 1];
  for (int l = 0; l < SG_MAXL + 1; ++l) h.eoff[l] = l <= L ? y.eoff[l] : y.eoff[L];
  for (int l = 0; l <= SG_MAXL; ++l) h.rbase[l] = l <= L ? y.rbase[l] : y.rbase[L];

  if (g == 1 && dst_grouped && (cache_bits == nullptr || all_cached)) {
    ::sg::launch(k_meta_init, 1, 256, 0, st, h, sizes, meta);
    SG_CHECK_LAUNCH("k_meta_init");
    LocalOut lo{P32(y.o_lsrc), P32(y.o_ldst), P32(y.o_rowbeg), P32(y.o_rowend), P32(y.o_selfrow)};
    const int64_t tot = y.nVtot + y.nEtot;
    ::sg::launch(k_split_single, clamp_grid(div_up(tot, 256), kSMs * 8), 256, 0, st, V, esrc, edst, h, meta, y.n_vertices, all_cached, P32(y.o_rank), P32(y.o_grouped),
        P32(y.o_egrouped), lo);
    SG_CHECK_LAUNCH("k_split_single");
    return SG_OK;
  }
  // zero-initialised regions: pair masks, gid bitmaps, rows; contrib = -1.
  SG_CUDA(cudaMemsetAsync(base + y.o_pmask, 0, 4 * y.nVtot, st));
  if (g > 1) SG_CUDA(cudaMemsetAsync(base + y.o_bitmap, 0, 4 * y.bm_words * L, st));
  SG_CUDA(cudaMemsetAsync(base + y.o_contrib, 0xff, 4 * (int64_t)g * y.nVtot, st));
  const int64_t rows_total = y.rbase[L];
  if (rows_total > 0) {
    SG_CUDA(cudaMemsetAsync(base + y.o_rowbeg, 0, 4 * rows_total, st));
    SG_CUDA(cudaMemsetAsync(base + y.o_rowend, 0, 4 * rows_total, st));
  }

  ::sg::launch(k_meta_init, 1, 256, 0, st, h, sizes, meta);
  SG_CHECK_LAUNCH("k_meta_init");

  const int64_t nVtot = y.nVtot, nV0 = y.nV[0];
  if (nVtot > 0) {
    ::sg::launch(k_owner_keys, clamp_grid(div_up(nVtot, 256), kSMs * 8), 256, 0, st, V, h, nVtot, nV0, asn, y.n_vertices, cache_bits, g, P8(y.o_keys), meta);
    SG_CHECK_LAUNCH("k_owner_keys");
  }

  // positions multisplit: segments = layers 0..L, then the layer-0 load set
  SegDesc sp;
  memset(&sp, 0, sizeof(sp));
  sp.nseg = L + 2;
  sp.nkeys = g + 1;
  sp.mode = 0;
  {
    int64_t t = 0;
    for (int s = 0; s <= L; ++s) {
      sp.beg[s] = y.voff[s];
      sp.tile_beg[s] = t;
      t += (y.nV[s] + MS_T - 1) / MS_T;
    }
    sp.beg[L + 1] = nVtot;
    sp.tile_beg[L + 1] = t;
    t += (nV0 + MS_T - 1) / MS_T;
    sp.beg[L + 2] = nVtot + nV0;
    sp.tile_beg[L + 2] = t;
  }
  int32_t* tb_pos = P32(y.o_tilebase_pos);
  int32_t* keyoff_pos = tb_pos + y.pos_tiles * (g + 1);
  if (y.pos_tiles > 0) {
    ::sg::launch(ms_count, (int)y.pos_tiles, MS_THREADS, 0, st, P8(y.o_keys), sp, meta, P32(y.o_tiles_pos));
    SG_CHECK_LAUNCH("ms_count(pos)");
  }
  ::sg::launch(ms_scan, sp.nseg, 1024, 0, st, sp, P32(y.o_tiles_pos), tb_pos, keyoff_pos, 0, meta);
  SG_CHECK_LAUNCH("ms_scan(pos)");
  if (y.pos_tiles > 0) {
    ::sg::launch(ms_scatter, (int)y.pos_tiles, MS_THREADS, 0, st, P8(y.o_keys), sp, meta, tb_pos, keyoff_pos,
                                                        P32(y.o_rank), P32(y.o_grouped));
    SG_CHECK_LAUNCH("ms_scatter(pos)");
  }

  // edges: key = source device, pair masks
  const int64_t nEtot = y.nEtot;
  if (nEtot > 0) {
    ::sg::launch(k_edge_keys, clamp_grid(div_up(nEtot, 256), kSMs * 8), 256, 0, st, esrc, edst, h, meta, P8(y.o_keys), P8(y.o_ekey), U32(y.o_pmask),
        g == 1 ? P32(y.o_egrouped) : nullptr);
    SG_CHECK_LAUNCH("k_edge_keys");
  }
  SegDesc se;
  memset(&se, 0, sizeof(se));
  se.nseg = L;
  se.nkeys = g;
  se.mode = 1;
  {
    int64_t t = 0;
    for (int s = 0; s < L; ++s) {
      se.beg[s] = y.eoff[s];
      se.tile_beg[s] = t;
      t += (y.nE[s] + MS_T - 1) / MS_T;
    }
    se.beg[L] = nEtot;
    se.tile_beg[L] = t;
  }
  int32_t* tb_edge = P32(y.o_tilebase_edge);
  int32_t* keyoff_edge = tb_edge + y.edge_tiles * g;
  if (g == 1) {
    ::sg::launch(k_single_edge_meta, 1, 32, 0, st, meta);
    SG_CHECK_LAUNCH("k_single_edge_meta");
  } else if (y.edge_tiles > 0) {
    ::sg::launch(ms_count, (int)y.edge_tiles, MS_THREADS, 0, st, P8(y.o_ekey), se, meta, P32(y.o_tiles_edge));
    SG_CHECK_LAUNCH("ms_count(edge)");
  }
  if (g > 1) {
    ::sg::launch(ms_scan, se.nseg, 1024, 0, st, se, P32(y.o_tiles_edge), tb_edge, keyoff_edge, 1, meta);
    SG_CHECK_LAUNCH("ms_scan(edge)");
  }
  if (g > 1 && y.edge_tiles > 0) {
    ::sg::launch(ms_scatter, (int)y.edge_tiles, MS_THREADS, 0, st, P8(y.o_ekey), se, meta, tb_edge, keyoff_edge,
                                                         nullptr, P32(y.o_egrouped));
    SG_CHECK_LAUNCH("ms_scatter(edge)");
  }

  // reference vertices by gid
  const int64_t words = y.bm_words;
  const int64_t nref_pos = y.voff[L + 1] - y.voff[1];
  if (g > 1 && nref_pos > 0) {
    ::sg::launch(k_ref_bits, clamp_grid(div_up(nref_pos, 256), kSMs * 8), 256, 0, st, V, h, U32(y.o_pmask), U32(y.o_bitmap), words, 0);
    SG_CHECK_LAUNCH("k_ref_bits");
    ::sg::launch(k_ref_scan, (int)((words / CHUNK_WORDS) * L), 256, 0, st, U32(y.o_bitmap), P32(y.o_wpre),
                                                                 P32(y.o_ctot));
    SG_CHECK_LAUNCH("k_ref_scan");
    ::sg::launch(k_ref_chunks, 1, 256, 0, st, P32(y.o_ctot), words / CHUNK_WORDS, L, meta);
    SG_CHECK_LAUNCH("k_ref_chunks");
    ::sg::launch(k_ref_rank, clamp_grid(div_up(nref_pos, 256), kSMs * 8), 256, 0, st, V, h, U32(y.o_pmask), U32(y.o_bitmap), P32(y.o_wpre), P32(y.o_ctot), words,
        P32(y.o_uorder));
    SG_CHECK_LAUNCH("k_ref_rank");
  }

  PairDesc pd;
  memset(&pd, 0, sizeof(pd));
  pd.L = L;
  pd.g = g;
  pd.kq = g * g + g;
  for (int l = 0; l <= L + 1; ++l) pd.voff[l] = y.voff[l];
  for (int l = 0; l <= L; ++l) pd.nV[l] = y.nV[l];
  {
    int64_t t = 0;
    for (int l = 1; l <= L; ++l) {
      pd.tile_beg[l] = t;
      t += (y.nV[l] + PAIR_T - 1) / PAIR_T;
    }
    pd.tile_beg[L + 1] = t;
  }
  for (int l = 0; l <= L + 1; ++l) pd.pbase[l] = y.pbase[l];
  if (g > 1 && y.pair_tiles > 0) {
    ::sg::launch(k_pair_count, (int)y.pair_tiles, PAIR_T, 0, st, pd, meta, P32(y.o_uorder), U32(y.o_pmask),
                                                        P8(y.o_keys), P32(y.o_tiles_pair));
    SG_CHECK_LAUNCH("k_pair_count");
    ::sg::launch(k_pair_scan, 1, 1024, 0, st, pd, P32(y.o_tiles_pair), P32(y.o_tilebase_pair), meta);
    SG_CHECK_LAUNCH("k_pair_scan");
    PairOut po{P32(y.o_pairs), P32(y.o_pair_hidx), P32(y.o_sendpos), P32(y.o_xfer),
               P32(y.o_recv_row), P32(y.o_refrank), P32(y.o_contrib)};
    ::sg::launch(k_pair_scatter, (int)y.pair_tiles, PAIR_T, 0, st, pd, meta, P32(y.o_uorder), U32(y.o_pmask),
                                                          P8(y.o_keys), P32(y.o_rank),
                                                          P32(y.o_tilebase_pair), po);
    SG_CHECK_LAUNCH("k_pair_scatter");
  }

  const int64_t nS = y.voff[L + 1] - y.voff[1];
  if (nEtot + nS > 0) {
    LocalOut lo{P32(y.o_lsrc), P32(y.o_ldst), P32(y.o_rowbeg), P32(y.o_rowend), P32(y.o_selfrow)};
    ::sg::launch(k_local_edges, clamp_grid(div_up(nEtot + nS, 256), kSMs * 8), 256, 0, st, esrc, edst, h, meta, P8(y.o_keys), P32(y.o_rank), P32(y.o_grouped), P32(y.o_egrouped),
        P32(y.o_refrank), lo);
    SG_CHECK_LAUNCH("k_local_edges");
  }
  return SG_OK;
}

}  // namespace sg
