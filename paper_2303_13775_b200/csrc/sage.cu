// GraphSAGE (mean aggregator) forward / backward for one device of a split.
//
//   sg_sage_agg_fwd     local_aggregate (engine.py:180-195): CSR-by-destination
//                       segment-sum SpMM. A row group (LPR lanes, warp for
//                       F=100) first fetches up to LPR edge indices in ONE
//                       round (lane i -> edge i, both index hops in parallel),
//                       then broadcasts them with shuffles and issues all the
//                       source-row loads (128-bit) back to back, 8 in flight.
//                       Reference rows are packed straight into the
//                       push-to-owner send buffer (fused pack epilogue).
//   sg_sage_fused_fwd / sg_sage_combine_fwd
//                       one kernel per layer (k_sage_layer): aggregation (g = 1)
//                       or owner combine (g > 1), mean, and the GEMM from smem
//   sg_sage_update      owner combine in ascending sender order + mean +
//                       h_self@W_self + mean@W_neigh + b + ReLU (:197-226);
//                       FP32 FFMA, weights in smem, each thread a 1x4 output
//                       tile (2 scalar + 2 LDS.128 per 8 FMA).
//   sg_sage_bwd_rows    d_pre, weight/bias gradient partials (deterministic
//                       per-block, 1x4 register tiles), d_self and d_sums
//                       (:228-254).
//   sg_sage_scatter_bwd transpose SpMM over CSR-by-source (:263-276): warp per
//                       source row, 32 out-edges fetched per round and split
//                       over 32/LPR lane groups (hub rows load-balanced inside
//                       the warp), fixed-tree reduction (deterministic);
//                       reference destinations read the owners' returned
//                       gradients from the push-from-owner payload (fused
//                       unpack).
// All arithmetic is FP32 (parity target rel 1e-4 vs the float64 reference).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "dense.cuh"

namespace sg {
namespace {

template <int VEC>
struct VecT;
template <>
struct VecT<4> {
  using T = float4;
  __device__ static float4 zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
  __device__ static float4 ld(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
  __device__ static float4 ld_any(const float* p) { return make_float4(p[0], p[1], p[2], p[3]); }
  __device__ static void add(float4& a, const float4& b) {
    a.x += b.x;
    a.y += b.y;
    a.z += b.z;
    a.w += b.w;
  }
  __device__ static float4 shfl_xor(const float4& v, int o) {
    return make_float4(__shfl_xor_sync(0xffffffffu, v.x, o), __shfl_xor_sync(0xffffffffu, v.y, o),
                       __shfl_xor_sync(0xffffffffu, v.z, o), __shfl_xor_sync(0xffffffffu, v.w, o));
  }
  __device__ static void st(float* p, const float4& v) { *reinterpret_cast<float4*>(p) = v; }
  __device__ static void st_any(float* p, const float4& v) {
    p[0] = v.x;
    p[1] = v.y;
    p[2] = v.z;
    p[3] = v.w;
  }
};
template <>
struct VecT<1> {
  using T = float;
  __device__ static float zero() { return 0.f; }
  __device__ static float ld(const float* p) { return __ldg(p); }
  __device__ static float ld_any(const float* p) { return *p; }
  __device__ static void add(float& a, const float& b) { a += b; }
  __device__ static float shfl_xor(const float& v, int o) { return __shfl_xor_sync(0xffffffffu, v, o); }
  __device__ static void st(float* p, const float& v) { *p = v; }
  __device__ static void st_any(float* p, const float& v) { *p = v; }
};

// ---------------------------------------------------------------- forward SpMM
struct AggArgs {
  int l, d, w, stride;
  int hst;  // row stride of h_prev (>= w; a padded feature table reads whole 128 B lines)
  int64_t eoff_li, rbase_li, pbase_l;
  const int32_t* rowbeg;
  const int32_t* rowend;
  const int32_t* lsrc;
  const int32_t* dperm;
  const int32_t* sendpos;
  const int32_t* src_row;
  const float* h_prev;
  float* sums;
  float* counts;
  float* sendbuf;
  // peer transport (one rank per GPU): reference rows go straight into the
  // owners' mapped receive buffers at xfer[pair slot] (push fused into the
  // aggregation epilogue); peer[0] == 0 -> write sendbuf
  int g;
  const int32_t* xfer;
  struct { int64_t p[SG_MAXG]; } peer;
};

// A row "team" of RL = LPR*EG lanes: LPR lanes cover the row width (VEC floats
// each), EG edge groups take every EG-th in-edge, then a fixed xor-tree adds
// the groups (deterministic). Each round the team fetches RL edge indices at
// once (both index hops in parallel), then issues the row loads back to back.
template <int VEC, int LPR, int EG, int NCH>
__global__ void __launch_bounds__(256) k_sage_agg(const SgMeta* __restrict__ meta, AggArgs a) {
  SG_PDL_ENTRY();
  using V = VecT<VEC>;
  using T = typename V::T;
  constexpr int RL = LPR * EG;
  constexpr int RPW = 32 / RL;
  const int l = a.l, d = a.d, w = a.w;
  const int n_own = meta->n_own[l][d];
  const int R = n_own + meta->n_ref[l][d];
  const int own0 = meta->own_off[l][d], ref0 = meta->ref_off[l][d];
  const int prev0 = meta->own_off[l - 1][d];
  const int64_t rb = a.rbase_li + own0 + ref0;
  const int lane = threadIdx.x & 31;
  const int team = lane / RL, tl = lane % RL;
  const int eg = tl / LPR, lr = tl % LPR;
  const unsigned tmask = (RL == 32) ? 0xffffffffu : (((1u << RL) - 1u) << (team * RL));
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = gw * RPW + team; q < R; q += nw * RPW) {
    const int b = a.rowbeg[rb + q], e = a.rowend[rb + q];
    T acc[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) acc[c] = V::zero();
    for (int jb = b; jb < e; jb += RL) {
      const int j = jb + tl;
      int r = 0;
      if (j < e) {
        const int64_t x = a.dperm ? (int64_t)a.dperm[j] : a.eoff_li + j;
        r = prev0 + a.lsrc[x];
        if (a.src_row) r = a.src_row[r];
      }
      const int cnt = min(RL, e - jb);
      const int rounds = (cnt + EG - 1) / EG;
      int kk = 0;
      for (; kk + 4 <= rounds; kk += 4) {
        int rr[4];
        bool ok[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = (kk + u) * EG + eg;
          rr[u] = __shfl_sync(tmask, r, k < RL ? k : RL - 1, RL);
          ok[u] = k < cnt;
        }
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          const int col = (c * LPR + lr) * VEC;
          if (col < a.hst) {  // whole (padded) rows: full 128 B lines
            T v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = ok[u] ? V::ld(a.h_prev + (int64_t)rr[u] * a.hst + col) : V::zero();
#pragma unroll
            for (int u = 0; u < 4; ++u) V::add(acc[c], v[u]);
          }
        }
      }
      for (; kk < rounds; ++kk) {
        const int k = kk * EG + eg;
        const int r0 = __shfl_sync(tmask, r, k < RL ? k : RL - 1, RL);
        if (k < cnt) {
#pragma unroll
          for (int c = 0; c < NCH; ++c) {
            const int col = (c * LPR + lr) * VEC;
            if (col < a.hst) V::add(acc[c], V::ld(a.h_prev + (int64_t)r0 * a.hst + col));
          }
        }
      }
    }
#pragma unroll
    for (int o = LPR; o < RL; o <<= 1) {
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        if constexpr (VEC == 4) {
          acc[c].x += __shfl_xor_sync(tmask, acc[c].x, o, RL);
          acc[c].y += __shfl_xor_sync(tmask, acc[c].y, o, RL);
          acc[c].z += __shfl_xor_sync(tmask, acc[c].z, o, RL);
          acc[c].w += __shfl_xor_sync(tmask, acc[c].w, o, RL);
        } else {
          acc[c] += __shfl_xor_sync(tmask, acc[c], o, RL);
        }
      }
    }
    if (eg != 0) continue;
    const float cntf = (float)(e - b);
    if (q < n_own) {
      float* out = a.sums + (int64_t)(own0 + q) * w;
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const int col = (c * LPR + lr) * VEC;
        if (col < w) V::st(out + col, acc[c]);
      }
      if (lr == 0) a.counts[own0 + q] = cntf;
    } else {
      const int slot = a.sendpos[a.pbase_l + ref0 + (q - n_own)];
      float* out;
      if (a.peer.p[0]) {  // store over NVLink into the owner's receive slot
        const int rs = a.xfer[slot];
        out = (float*)a.peer.p[find_bucket(meta->recv_off[l], a.g, rs)] + (int64_t)rs * a.stride;
      } else {
        out = a.sendbuf + (int64_t)slot * a.stride;
      }
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const int col = (c * LPR + lr) * VEC;
        if (col < w) {
          if ((a.stride & 3) == 0) V::st(out + col, acc[c]); else V::st_any(out + col, acc[c]);
        }
      }
      if (lr == 0) out[w] = cntf;
    }
  }
}

template <int VEC, int LPR, int EG, int NCH>
int launch_agg(const SgMeta* meta, const AggArgs& a, int64_t max_rows, cudaStream_t st) {
  constexpr int RPB = 8 * (32 / (LPR * EG));  // rows per 256-thread block
  const int grid = clamp_grid(div_up(max_rows, RPB), kSMs * 8);
  ::sg::launch(k_sage_agg<VEC, LPR, EG, NCH>, grid, 256, 0, st, meta, a);
  SG_CHECK_LAUNCH("k_sage_agg");
  return SG_OK;
}

// ---------------------------------------------------------------- one-kernel layer arguments
// Single-device split (no row has remote contributions) or the owner side after
// the push-to-owner round: aggregation (or combine) + update in k_sage_layer.
struct FusedArgs {
  int l, d, w, dout, final_;
  int64_t eoff_li, rbase_li, voff_l;
  const int32_t* rowbeg;
  const int32_t* rowend;
  const int32_t* lsrc;
  const int32_t* selfrow;
  const int32_t* src_row;
  const float* h_prev;
  const float* ws;
  const float* wn;
  const float* bias;
  float* mean;
  float* counts;
  float* hs;
  float* h;
  // combine mode (g > 1, set by sg_sage_combine_fwd): the row's local partial
  // (sums, counts) plus the holders' partials from recv in ascending sender
  // order (engine.py:197-210) replace the aggregation
  const float* sums;
  const float* recv;
  const int32_t* contrib;
  int stride, g;
  int hst;  // row stride of h_prev (k_sage_layer: a padded feature table is read in whole lines)
};


// ---------------------------------------------------------------- tiled dense transforms
// h = act(hs @ W_self + mean @ W_neigh + b) for the owned rows: a register-
// tiled FP32 GEMM ([rows x 2w] @ [2w x dout]). K is staged in chunks of 32,
// transposed in smem so each thread reads its RPT consecutive rows with one
// vector load; each thread owns RPT rows x 4 outputs (RPT*4 FFMA per 2 loads).
struct LinArgs {
  int l, d, w, dout, final_;
  const float* hs;
  const float* mean;
  const float* ws;
  const float* wn;
  const float* bias;
  float* h;
};

// 64-row tiles; the whole K = 2w slice of the tile is staged once (all loads
// in flight), K is split over NS thread slices, each thread owns a 4-row x
// 4-output register tile (2 LDS.128 per 16 FFMA), slices are added in a fixed
// order through shared memory (deterministic).
template <int NQ>
__global__ void __launch_bounds__(256, 3) k_sage_linear(const SgMeta* __restrict__ meta, LinArgs a) {
  SG_PDL_ENTRY();
  constexpr int TM = 32;
  constexpr int TMP = TM + 4;
  constexpr int NT = (TM / 4) * NQ;  // register tiles per K slice
  constexpr int NS = 256 / NT;       // K slices
  extern __shared__ __align__(16) float smem[];
  const int w = a.w, dout = a.dout, K = 2 * w;
  float* W_s = smem;                 // [2w][dout]
  float* A_s = W_s + K * dout;       // [2w][TM+4] transposed
  float* red = A_s + K * TMP;        // [NS][TM][dout]
  {
    // all weight loads in flight before any store (w*dout % 4 == 0)
    constexpr int MW = 4;  // float4 per thread per pass: 2*w*dout/4 <= 2048 (two passes)
    const int nw4 = w * dout / 4;
    for (int pass = 0; pass < 2; ++pass) {
      float4 wb[MW];
#pragma unroll
      for (int u = 0; u < MW; ++u) {
        const int i = threadIdx.x + 256 * (u + MW * pass);
        if (i < 2 * nw4)
          wb[u] = i < nw4 ? reinterpret_cast<const float4*>(a.ws)[i]
                          : reinterpret_cast<const float4*>(a.wn)[i - nw4];
      }
#pragma unroll
      for (int u = 0; u < MW; ++u) {
        const int i = threadIdx.x + 256 * (u + MW * pass);
        if (i < 2 * nw4) reinterpret_cast<float4*>(W_s)[i] = wb[u];
      }
    }
  }
  const int n = meta->n_own[a.l][a.d];
  const int own0 = meta->own_off[a.l][a.d];
  const int tile = threadIdx.x % NT, ks = threadIdx.x / NT;
  const int rt = tile / NQ, jq = tile - rt * NQ;
  const int kchunk = (K + NS - 1) / NS;
  const int kb = ks * kchunk, ke = min(K, kb + kchunk);
  const int w4 = w / 4;
  for (int r0 = blockIdx.x * TM; r0 < n; r0 += gridDim.x * TM) {
    __syncthreads();
    {
      // issue every load of the tile (<= 8 float4 per thread), then store
      // transposed; row index fastest: shift/mask indexing, conflict-free stores
      constexpr int MA = 8;
      const int tot = TM * 2 * w4;
      float4 ab[MA];
#pragma unroll
      for (int u = 0; u < MA; ++u) {
        const int idx = threadIdx.x + 256 * u;
        ab[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (idx < tot) {
          const int r = idx & (TM - 1), q = idx / TM;
          if (r0 + r < n) {
            const int64_t G = own0 + r0 + r;
            ab[u] = q < w4 ? *reinterpret_cast<const float4*>(a.hs + G * w + 4 * q)
                           : *reinterpret_cast<const float4*>(a.mean + G * w + 4 * (q - w4));
          }
        }
      }
#pragma unroll
      for (int u = 0; u < MA; ++u) {
        const int idx = threadIdx.x + 256 * u;
        if (idx < tot) {
          const int r = idx & (TM - 1), q = idx / TM;
          A_s[(4 * q + 0) * TMP + r] = ab[u].x;
          A_s[(4 * q + 1) * TMP + r] = ab[u].y;
          A_s[(4 * q + 2) * TMP + r] = ab[u].z;
          A_s[(4 * q + 3) * TMP + r] = ab[u].w;
        }
      }
    }
    __syncthreads();
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
#pragma unroll 4
    for (int k = kb; k < ke; ++k) {
      const float4 av = *reinterpret_cast<const float4*>(A_s + k * TMP + 4 * rt);
      const float4 wv = *reinterpret_cast<const float4*>(W_s + k * dout + 4 * jq);
      const float ar[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc[i][0] = fmaf(ar[i], wv.x, acc[i][0]);
        acc[i][1] = fmaf(ar[i], wv.y, acc[i][1]);
        acc[i][2] = fmaf(ar[i], wv.z, acc[i][2]);
        acc[i][3] = fmaf(ar[i], wv.w, acc[i][3]);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      *reinterpret_cast<float4*>(red + (ks * TM + 4 * rt + i) * dout + 4 * jq) =
          make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    __syncthreads();
    for (int idx = threadIdx.x; idx < TM * dout; idx += 256) {
      const int r = idx / dout, j = idx - r * dout;
      if (r0 + r >= n) continue;
      float v = a.bias[j];
#pragma unroll
      for (int s2 = 0; s2 < NS; ++s2) v += red[(s2 * TM + r) * dout + j];
      a.h[(int64_t)(own0 + r0 + r) * dout + j] = a.final_ ? v : sg_relu(v);
    }
  }
}

template <int NQ>
int launch_linear_q(const SgMeta* meta, const LinArgs& a, int64_t max_rows, cudaStream_t st) {
  constexpr int TM = 32;
  constexpr int NS = 256 / ((TM / 4) * NQ);
  const size_t smem = sizeof(float) * (2 * (size_t)a.w * a.dout + 2 * (size_t)a.w * (TM + 4) +
                                       (size_t)NS * TM * a.dout);
  if (smem > 227 * 1024) {
    set_error("sage_linear: width too large");
    return SG_ERR_ARG;
  }
  const cudaError_t attr = allow_max_smem<k_sage_linear<NQ>>();
  SG_CUDA(attr);
  const int grid = clamp_grid(div_up(max_rows, TM), kSMs * 8);
  ::sg::launch(k_sage_linear<NQ>, grid, 256, smem, st, meta, a);
  SG_CHECK_LAUNCH("k_sage_linear");
  return SG_OK;
}

// ---------------------------------------------------------------- one-kernel layer (g == 1)
// Aggregation and dense transform in ONE kernel: a 32-row tile's [hs | mean]
// operand never leaves the SM. Each warp aggregates 4 destination rows; per
// row all in-edges' 128-bit row loads (up to UN per lane) are in flight at
// once and the NEXT row's edge indices are fetched while they land (the
// rowbeg -> lsrc -> src_row chain is off the critical path). Rows go
// transposed into smem ([2w][TM+4]) and to global (mean, hs: the backward's
// operands); then the same register-tiled FP32 GEMM as k_sage_linear.
template <int NQ, int UN, int RPW, int MINB>
__global__ void __launch_bounds__(256, MINB) k_sage_layer(const SgMeta* __restrict__ meta, FusedArgs a) {
  // the weight staging below runs before the PDL wait (parameters are not
  // written by the preceding kernel; see k_sage_wgrad)
  constexpr int TM = 8 * RPW;  // rows per tile (RPW per warp)
  constexpr int NT = (TM / 4) * NQ;
  constexpr int NS = 256 / NT;
  extern __shared__ __align__(16) float smem[];
  const int w = a.w, dout = a.dout, K = 2 * w;
  const int l = a.l, d = a.d;
  float* W_s = smem;            // [2w][dout]
  const int KP = K + 4;         // row-major A tile: float4 row stores are conflict-free
  float* A_s = W_s + K * dout;  // [TM][2w+4] (hs | mean); reused as the slice reduction
  for (int i = threadIdx.x; i < w * dout / 4; i += 256) {
    reinterpret_cast<float4*>(W_s)[i] = reinterpret_cast<const float4*>(a.ws)[i];
    reinterpret_cast<float4*>(W_s)[w * dout / 4 + i] = reinterpret_cast<const float4*>(a.wn)[i];
  }
  SG_PDL_ENTRY();
  const int n = meta->n_own[l][d];
  const int own0 = meta->own_off[l][d];
  const int prev0 = meta->own_off[l - 1][d];
  const int64_t rb = a.rbase_li + own0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int col = lane * 4;
  const bool colok = col < w;
  const int hst = a.hst;
  const bool ldok = col < hst;  // padded rows: every lane loads (whole 128 B lines), stores stay < w
  const int tile = threadIdx.x % NT, ks = threadIdx.x / NT;
  const int rt = tile / NQ, jq = tile - rt * NQ;
  const int kchunk = ((K + NS - 1) / NS + 3) & ~3;  // whole float4 steps of K
  const int kb = ks * kchunk, ke = min(K, kb + kchunk);
  auto edge_row = [&](int j) {
    int r = prev0 + a.lsrc[a.eoff_li + j];
    return a.src_row ? a.src_row[r] : r;
  };
  for (int r0 = blockIdx.x * TM; r0 < n; r0 += gridDim.x * TM) {
    // ---- aggregation: warp wid owns tile rows [wid*RPW, wid*RPW + RPW)
    const int q0 = r0 + wid * RPW;
    const bool comb = a.sums != nullptr;
    int be = 0;
    if (!comb && lane < 2 * RPW && q0 + (lane >> 1) < n)
      be = (lane & 1) ? a.rowend[rb + q0 + (lane >> 1)] : a.rowbeg[rb + q0 + (lane >> 1)];
    int b = __shfl_sync(0xffffffffu, be, 0), e = __shfl_sync(0xffffffffu, be, 1);
    int rnext = (!comb && q0 < n && lane < e - b) ? edge_row(b + lane) : 0;
    __syncthreads();  // previous tile's GEMM done with A_s
    for (int i = 0; i < RPW; ++i) {
      const int q = q0 + i;
      if (q >= n) break;  // warp-uniform
      const int rcur = rnext;
      const int bc = b, ec = e;
      const int64_t G = own0 + q;
      int rself = prev0 + a.selfrow[a.voff_l + G];
      if (a.src_row) rself = a.src_row[rself];
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      float4 hv = make_float4(0.f, 0.f, 0.f, 0.f);
      float cntf;
      if (comb) {
        float N = a.counts[G];
        if (colok) {
          acc = *reinterpret_cast<const float4*>(a.sums + G * w + col);
          hv = __ldg(reinterpret_cast<const float4*>(a.h_prev + (int64_t)rself * hst + col));
        }
        const int32_t* cb = a.contrib + (int64_t)a.g * a.voff_l + G * a.g;
        for (int s = 0; s < a.g; ++s) {
          const int rs = cb[s];
          if (rs < 0) continue;
          const float* rrow = a.recv + (int64_t)rs * a.stride;
          if (colok) {
            const float4 t = *reinterpret_cast<const float4*>(rrow + col);
            acc.x += t.x; acc.y += t.y; acc.z += t.z; acc.w += t.w;
          }
          N += rrow[w];
        }
        cntf = N;
      } else {
      // next row's bounds + first index hop, issued before this row's loads
      int nb = 0, ne = 0, lnext = 0;
      if (i + 1 < RPW && q + 1 < n) {
        nb = __shfl_sync(0xffffffffu, be, 2 * (i + 1));
        ne = __shfl_sync(0xffffffffu, be, 2 * (i + 1) + 1);
        if (lane < ne - nb) lnext = prev0 + a.lsrc[a.eoff_li + nb + lane];
      }
      const int cnt0 = min(32, ec - bc);
      for (int kk = 0; kk < cnt0; kk += UN) {
        float4 v[UN];
#pragma unroll
        for (int u = 0; u < UN; ++u) {
          const int k = kk + u;
          const int rr = __shfl_sync(0xffffffffu, rcur, k < 32 ? k : 31);
          v[u] = (k < cnt0 && ldok) ? __ldg(reinterpret_cast<const float4*>(a.h_prev + (int64_t)rr * hst + col))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        if (kk == 0 && colok) hv = __ldg(reinterpret_cast<const float4*>(a.h_prev + (int64_t)rself * hst + col));
#pragma unroll
        for (int u = 0; u < UN; ++u) {
          acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w;
        }
      }
      // rows with more than 32 in-edges: remaining rounds (rare in forward)
      for (int jb = bc + 32; jb < ec; jb += 32) {
        const int rr0 = (jb + lane < ec) ? edge_row(jb + lane) : 0;
        const int cnt = min(32, ec - jb);
        for (int k = 0; k < cnt; ++k) {
          const int rr = __shfl_sync(0xffffffffu, rr0, k);
          if (ldok) {
            const float4 t = __ldg(reinterpret_cast<const float4*>(a.h_prev + (int64_t)rr * hst + col));
            acc.x += t.x; acc.y += t.y; acc.z += t.z; acc.w += t.w;
          }
        }
      }
      if (ec == bc && colok) hv = __ldg(reinterpret_cast<const float4*>(a.h_prev + (int64_t)rself * hst + col));
      // second index hop of the next row, overlapping this row's tail
      if (i + 1 < RPW && q + 1 < n) {
        rnext = (lane < ne - nb) ? (a.src_row ? a.src_row[lnext] : lnext) : 0;
        b = nb;
        e = ne;
      }
      cntf = (float)(ec - bc);
      }
      const float inv = 1.0f / cntf;
      const float4 mn = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
      const int rr = wid * RPW + i;
      if (colok) {
        *reinterpret_cast<float4*>(a.mean + G * w + col) = mn;
        if (a.hs) *reinterpret_cast<float4*>(a.hs + G * w + col) = hv;
        *reinterpret_cast<float4*>(A_s + rr * KP + col) = hv;
        *reinterpret_cast<float4*>(A_s + rr * KP + w + col) = mn;
      }
      if (lane == 0) a.counts[G] = cntf;
    }
    __syncthreads();
    // ---- dense transform from smem (rows past n hold garbage: never stored)
    float acc2[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc2[i][0] = acc2[i][1] = acc2[i][2] = acc2[i][3] = 0.f;
    // 4x4 (rows x K) block of A and 4x4 (K x outputs) block of W per step:
    // 8 LDS.128 per 64 FFMA
    for (int k = kb; k < ke; k += 4) {
      float4 av[4], wv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = *reinterpret_cast<const float4*>(A_s + (4 * rt + i) * KP + k);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) wv[kk] = *reinterpret_cast<const float4*>(W_s + (k + kk) * dout + 4 * jq);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float ar[4] = {av[i].x, av[i].y, av[i].z, av[i].w};
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          acc2[i][0] = fmaf(ar[kk], wv[kk].x, acc2[i][0]);
          acc2[i][1] = fmaf(ar[kk], wv[kk].y, acc2[i][1]);
          acc2[i][2] = fmaf(ar[kk], wv[kk].z, acc2[i][2]);
          acc2[i][3] = fmaf(ar[kk], wv[kk].w, acc2[i][3]);
        }
      }
    }
    __syncthreads();
    float* red = A_s;  // [NS][TM][dout]
#pragma unroll
    for (int i = 0; i < 4; ++i)
      *reinterpret_cast<float4*>(red + (ks * TM + 4 * rt + i) * dout + 4 * jq) =
          make_float4(acc2[i][0], acc2[i][1], acc2[i][2], acc2[i][3]);
    __syncthreads();
    for (int idx = threadIdx.x; idx < TM * dout; idx += 256) {
      const int r = idx / dout, j = idx - r * dout;
      if (r0 + r >= n) continue;
      float v = a.bias[j];
#pragma unroll
      for (int s2 = 0; s2 < NS; ++s2) v += red[(s2 * TM + r) * dout + j];
      a.h[(int64_t)(own0 + r0 + r) * dout + j] = a.final_ ? v : sg_relu(v);
    }
  }
}

template <int NQ, int UN, int RPW, int MINB>
int launch_layer_q(const SgMeta* meta, const FusedArgs& a, int64_t max_rows, cudaStream_t st) {
  constexpr int TM = 8 * RPW;
  constexpr int NS = 256 / ((TM / 4) * NQ);
  const size_t a_floats = std::max<size_t>((size_t)TM * (2 * (size_t)a.w + 4), (size_t)NS * TM * a.dout);
  const size_t smem = sizeof(float) * (2 * (size_t)a.w * a.dout + a_floats);
  if (smem > 227 * 1024) {
    set_error("sage_layer: width too large");
    return SG_ERR_ARG;
  }
  const cudaError_t attr = allow_max_smem<k_sage_layer<NQ, UN, RPW, MINB>>();
  SG_CUDA(attr);
  int per_sm = MINB;
  const size_t by_smem = (228 * 1024) / (smem + 1024);
  if ((int)by_smem < per_sm) per_sm = (int)std::max<size_t>(1, by_smem);
  const int grid = clamp_grid(div_up(max_rows, TM), kSMs * per_sm);
  ::sg::launch(k_sage_layer<NQ, UN, RPW, MINB>, grid, 256, smem, st, meta, a);
  SG_CHECK_LAUNCH("k_sage_layer");
  return SG_OK;
}

template <int UN, int RPW, int MINB>
int launch_layer(const SgMeta* meta, const FusedArgs& a, int64_t max_rows, cudaStream_t st) {
  switch (a.dout / 4) {
    case 1: return launch_layer_q<1, UN, RPW, MINB>(meta, a, max_rows, st);
    case 2: return launch_layer_q<2, UN, RPW, MINB>(meta, a, max_rows, st);
    case 4: return launch_layer_q<4, UN, RPW, MINB>(meta, a, max_rows, st);
    case 8: return launch_layer_q<8, UN, RPW, MINB>(meta, a, max_rows, st);
    default: set_error("sage_layer: dout must be 4, 8, 16 or 32"); return SG_ERR_ARG;
  }
}

int launch_linear(const SgMeta* meta, const LinArgs& a, int64_t max_rows, cudaStream_t st) {
  switch (a.dout / 4) {
    case 1: return launch_linear_q<1>(meta, a, max_rows, st);
    case 2: return launch_linear_q<2>(meta, a, max_rows, st);
    case 4: return launch_linear_q<4>(meta, a, max_rows, st);
    case 8: return launch_linear_q<8>(meta, a, max_rows, st);
    default: set_error("sage_linear: dout must be 4, 8, 16 or 32"); return SG_ERR_ARG;
  }
}

// dispatch on width: VEC=4 needs w%4==0 (16B aligned rows)
int dispatch_agg(const SgMeta* meta, const AggArgs& a, int64_t max_rows, cudaStream_t st) {
  const int w = a.w;
  if (w % 4 == 0) {
    if (w <= 16) return launch_agg<4, 4, 4, 1>(meta, a, max_rows, st);
    if (w <= 32) return launch_agg<4, 8, 4, 1>(meta, a, max_rows, st);
    if (w <= 64) return launch_agg<4, 16, 2, 1>(meta, a, max_rows, st);
    if (w <= 128) return launch_agg<4, 32, 1, 1>(meta, a, max_rows, st);
    if (w <= 256) return launch_agg<4, 32, 1, 2>(meta, a, max_rows, st);
    if (w <= 512) return launch_agg<4, 32, 1, 4>(meta, a, max_rows, st);
  } else {
    if (w <= 8) return launch_agg<1, 8, 4, 1>(meta, a, max_rows, st);
    if (w <= 32) return launch_agg<1, 32, 1, 1>(meta, a, max_rows, st);
    if (w <= 128) return launch_agg<1, 32, 1, 4>(meta, a, max_rows, st);
    if (w <= 512) return launch_agg<1, 32, 1, 16>(meta, a, max_rows, st);
  }
  set_error("sage_agg_fwd: width > 512 unsupported");
  return SG_ERR_ARG;
}

// ---------------------------------------------------------------- update
constexpr int UTR = 32;  // rows per tile

struct UpdArgs {
  int l, d, w, dout, final_, g, stride;
  int64_t voff_l;
  const float* h_prev;
  const int32_t* src_row;
  const int32_t* selfrow;
  const int32_t* contrib;
  const float* sums;
  float* counts;
  const float* recv;
  const float* ws;
  const float* wn;
  const float* bias;
  float* mean;
  float* h;
  float* hs_out;  // when set: write the self rows and leave the GEMM to k_sage_linear
  int no_linear;  // mean / counts (/ hs_out) only: the dense transform runs in dense.cu
};

template <bool Q4>
__global__ void __launch_bounds__(256) k_sage_update(const SgMeta* __restrict__ meta, UpdArgs a) {
  SG_PDL_ENTRY();
  extern __shared__ __align__(16) float smem[];
  const int w = a.w, dout = a.dout, wp = w + 1;
  const int wsz = a.no_linear ? 0 : w * dout;
  float* ws_s = smem;              // [w][dout] (none when no_linear)
  float* wn_s = ws_s + wsz;        // [w][dout]
  float* hs_s = wn_s + wsz;        // [UTR][w+1]
  float* mn_s = hs_s + UTR * wp;   // [UTR][w+1]
  float* n_s = mn_s + UTR * wp;    // [UTR]
  int* prow_s = (int*)(n_s + UTR); // [UTR]
  int* cs_s = prow_s + UTR;        // [UTR][g]
  for (int i = threadIdx.x; i < wsz; i += blockDim.x) {
    ws_s[i] = a.ws[i];
    wn_s[i] = a.wn[i];
  }
  const int l = a.l, d = a.d, g = a.g;
  const int n_own = meta->n_own[l][d];
  const int own0 = meta->own_off[l][d], prev0 = meta->own_off[l - 1][d];
  const int ntiles = (n_own + UTR - 1) / UTR;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    __syncthreads();
    // A1: one thread per row resolves the row's indices (all rows in parallel)
    if (threadIdx.x < UTR) {
      const int rr = threadIdx.x;
      const int q = tile * UTR + rr;
      if (q < n_own) {
        const int G = own0 + q;
        float N = a.counts[G];
        const int* cb = a.contrib + (int64_t)g * a.voff_l + (int64_t)G * g;
        for (int s = 0; g > 1 && s < g; ++s) {  // ascending sender order (engine.py:130-138)
          const int rs = cb[s];
          cs_s[rr * g + s] = rs;
          if (rs >= 0) N += a.recv[(int64_t)rs * a.stride + w];
        }
        int r = prev0 + a.selfrow[a.voff_l + G];
        if (a.src_row) r = a.src_row[r];
        prow_s[rr] = r;
        n_s[rr] = 1.0f / N;  // one division per row; the tile multiplies
        a.counts[G] = N;
      }
    }
    __syncthreads();
    // A2: coalesced tile loads (many independent loads in flight per thread)
    {
      const int nrow = min(UTR, n_own - tile * UTR);
#pragma unroll 4
      for (int idx = threadIdx.x; idx < nrow * w; idx += blockDim.x) {
        const int rr = idx / w, c = idx - rr * w;
        const int64_t G = own0 + tile * UTR + rr;
        float S = a.sums[G * w + c];
        for (int s = 0; g > 1 && s < g; ++s) {
          const int rs = cs_s[rr * g + s];
          if (rs >= 0) S += a.recv[(int64_t)rs * a.stride + c];
        }
        const float mv = S * n_s[rr];
        mn_s[rr * wp + c] = mv;
        a.mean[G * w + c] = mv;
        const float hv = __ldg(a.h_prev + (int64_t)prow_s[rr] * w + c);
        hs_s[rr * wp + c] = hv;
        if (a.hs_out) a.hs_out[G * w + c] = hv;
      }
    }
    __syncthreads();
    if (a.hs_out || a.no_linear) continue;  // dense transform done by k_sage_linear / dense.cu
    if (Q4) {
      const int nq = dout >> 2;
      for (int idx = threadIdx.x; idx < UTR * nq; idx += blockDim.x) {
        const int rr = idx / nq, jq = idx - rr * nq;
        const int q = tile * UTR + rr;
        if (q >= n_own) continue;
        const float* hr = hs_s + rr * wp;
        const float* mr = mn_s + rr * wp;
        // two independent accumulator sets (self / neighbour), 4-way unrolled
        float4 as = *reinterpret_cast<const float4*>(a.bias + 4 * jq);
        float4 an = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
        for (int c = 0; c < w; ++c) {
          const float hv = hr[c], mv = mr[c];
          const float4 s4 = *reinterpret_cast<const float4*>(ws_s + c * dout + 4 * jq);
          const float4 n4 = *reinterpret_cast<const float4*>(wn_s + c * dout + 4 * jq);
          as.x = fmaf(hv, s4.x, as.x);
          as.y = fmaf(hv, s4.y, as.y);
          as.z = fmaf(hv, s4.z, as.z);
          as.w = fmaf(hv, s4.w, as.w);
          an.x = fmaf(mv, n4.x, an.x);
          an.y = fmaf(mv, n4.y, an.y);
          an.z = fmaf(mv, n4.z, an.z);
          an.w = fmaf(mv, n4.w, an.w);
        }
        float4 acc = make_float4(as.x + an.x, as.y + an.y, as.z + an.z, as.w + an.w);
        if (!a.final_) {
          acc.x = sg_relu(acc.x);
          acc.y = sg_relu(acc.y);
          acc.z = sg_relu(acc.z);
          acc.w = sg_relu(acc.w);
        }
        *reinterpret_cast<float4*>(a.h + (int64_t)(own0 + q) * dout + 4 * jq) = acc;
      }
    } else {
      for (int idx = threadIdx.x; idx < UTR * dout; idx += blockDim.x) {
        const int rr = idx / dout, j = idx - rr * dout;
        const int q = tile * UTR + rr;
        if (q >= n_own) continue;
        const float* hr = hs_s + rr * wp;
        const float* mr = mn_s + rr * wp;
        float acc = a.bias[j];
        for (int c = 0; c < w; ++c) acc = fmaf(hr[c], ws_s[c * dout + j], fmaf(mr[c], wn_s[c * dout + j], acc));
        a.h[(int64_t)(own0 + q) * dout + j] = a.final_ ? acc : sg_relu(acc);
      }
    }
  }
}

// ---------------------------------------------------------------- backward rows
constexpr int BTR = 32;
constexpr int BMAXQ = 4;    // float4 slots per thread per weight matrix (w*dout <= 4096)
constexpr int BMAXACC = 16;  // scalar slots (dout % 4 != 0 path)

struct BwdArgs {
  int l, d, w, dout, final_, self_compact;
  int64_t voff_l;
  const float* h_prev;
  const int32_t* src_row;
  const int32_t* selfrow;
  const float* d_h;
  const float* h;
  const float* mean;
  const float* counts;
  const float* ws;
  const float* wn;
  float* partial;
  float* d_self;
  float* d_sums;
  // scatter mode (k_sage_wgrad): d_h of this layer's rows is not read but
  // computed in the tile as the transposed SpMM of layer l+1 (engine.py:263-273)
  const int32_t* sc_enc;
  const int32_t* sc_beg;
  const int32_t* sc_end;
  const int32_t* sc_grouped;
  const int32_t* sc_rank;
  const float* sc_dself;   // layer l+1 d_self (owned rows of l+1)
  const float* sc_dsums;   // layer l+1 d_sums
  const float* sc_recv;    // push-from-owner rows (pair slots), g > 1
  int64_t sc_key_base, sc_voff_src, sc_voff_dst;
  int sc_stride;
};

template <bool Q4>
__global__ void __launch_bounds__(256) k_sage_bwd_rows(const SgMeta* __restrict__ meta, BwdArgs a) {
  SG_PDL_ENTRY();
  extern __shared__ __align__(16) float smem[];
  const int w = a.w, dout = a.dout, wp = w + 1;
  const int wst = Q4 ? dout + 4 : dout + 1;  // padded weight row stride
  const bool need_c = a.d_self != nullptr || a.d_sums != nullptr;
  float* dp_s = smem;                  // [BTR][dout]
  float* ws_s = dp_s + BTR * dout;     // [w][wst] (only if need_c)
  float* wn_s = ws_s + w * wst;
  float* hs_s = wn_s + w * wst;        // [BTR][w+1]
  float* mn_s = hs_s + BTR * wp;       // [BTR][w+1]
  float* cnt_s = mn_s + BTR * wp;      // [BTR]
  int* prow_s = (int*)(cnt_s + BTR);   // [BTR]
  if (need_c) {
    for (int i = threadIdx.x; i < w * dout; i += blockDim.x) {
      const int c = i / dout, j = i - c * dout;
      ws_s[c * wst + j] = a.ws[i];
      wn_s[c * wst + j] = a.wn[i];
    }
  }
  const int l = a.l, d = a.d;
  const int n_own = meta->n_own[l][d];
  const int own0 = meta->own_off[l][d], prev0 = meta->own_off[l - 1][d];
  const int nq = dout >> 2;
  const int nslots = Q4 ? w * nq : w * dout;
  float4 aS4[BMAXQ], aN4[BMAXQ];
  float aS[BMAXACC], aN[BMAXACC];
#pragma unroll
  for (int k = 0; k < BMAXQ; ++k) aS4[k] = aN4[k] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int k = 0; k < BMAXACC; ++k) aS[k] = aN[k] = 0.f;
  float ab = 0.f;
  const int ntiles = (n_own + BTR - 1) / BTR;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    __syncthreads();
    if (threadIdx.x < BTR) {
      const int rr = threadIdx.x;
      const int q = tile * BTR + rr;
      if (q < n_own) {
        const int G = own0 + q;
        int r;
        if (a.self_compact) {
          r = G;  // h_prev is the compact self-row buffer written by the forward
        } else {
          r = prev0 + a.selfrow[a.voff_l + G];
          if (a.src_row) r = a.src_row[r];
        }
        prow_s[rr] = r;
        cnt_s[rr] = 1.0f / a.counts[G];
      } else {
        prow_s[rr] = -1;
        cnt_s[rr] = 1.f;
      }
    }
    for (int idx = threadIdx.x; idx < BTR * dout; idx += blockDim.x) {
      const int rr = idx / dout, j = idx - rr * dout;
      const int q = tile * BTR + rr;
      float v = 0.f;
      if (q < n_own) {
        const int64_t G = own0 + q;
        v = a.d_h[G * dout + j];
        if (!a.final_ && !(a.h[G * dout + j] > 0.f)) v = 0.f;
      }
      dp_s[idx] = v;
    }
    __syncthreads();
#pragma unroll 4
    for (int idx = threadIdx.x; idx < BTR * w; idx += blockDim.x) {
      const int rr = idx / w, c = idx - rr * w;
      const int pr = prow_s[rr];
      float hv = 0.f, mv = 0.f;
      if (pr >= 0) {
        hv = __ldg(a.h_prev + (int64_t)pr * w + c);
        mv = a.mean[(int64_t)(own0 + tile * BTR + rr) * w + c];
      }
      hs_s[rr * wp + c] = hv;
      mn_s[rr * wp + c] = mv;
    }
    __syncthreads();
    if (Q4) {
#pragma unroll
      for (int k = 0; k < BMAXQ; ++k) {
        const int idx = threadIdx.x + 256 * k;
        if (idx < nslots) {
          const int c = idx / nq, jq = idx - c * nq;
          float4 s1 = aS4[k], s2 = aN4[k];
#pragma unroll 8
          for (int rr = 0; rr < BTR; ++rr) {
            const float4 g4 = *reinterpret_cast<const float4*>(dp_s + rr * dout + 4 * jq);
            const float hv = hs_s[rr * wp + c], mv = mn_s[rr * wp + c];
            s1.x = fmaf(hv, g4.x, s1.x);
            s1.y = fmaf(hv, g4.y, s1.y);
            s1.z = fmaf(hv, g4.z, s1.z);
            s1.w = fmaf(hv, g4.w, s1.w);
            s2.x = fmaf(mv, g4.x, s2.x);
            s2.y = fmaf(mv, g4.y, s2.y);
            s2.z = fmaf(mv, g4.z, s2.z);
            s2.w = fmaf(mv, g4.w, s2.w);
          }
          aS4[k] = s1;
          aN4[k] = s2;
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < BMAXACC; ++k) {
        const int idx = threadIdx.x + 256 * k;
        if (idx < nslots) {
          const int c = idx / dout, j = idx - c * dout;
          float s1 = aS[k], s2 = aN[k];
          for (int rr = 0; rr < BTR; ++rr) {
            const float gv = dp_s[rr * dout + j];
            s1 = fmaf(hs_s[rr * wp + c], gv, s1);
            s2 = fmaf(mn_s[rr * wp + c], gv, s2);
          }
          aS[k] = s1;
          aN[k] = s2;
        }
      }
    }
    if (threadIdx.x < dout)
      for (int rr = 0; rr < BTR; ++rr) ab += dp_s[rr * dout + threadIdx.x];
    if (need_c) {
      for (int idx = threadIdx.x; idx < BTR * w; idx += blockDim.x) {
        const int rr = idx / w, c = idx - rr * w;
        const int q = tile * BTR + rr;
        if (q >= n_own) continue;
        const int64_t G = own0 + q;
        float s1 = 0.f, s2 = 0.f;
        if (Q4) {
          for (int jq = 0; jq < nq; ++jq) {
            const float4 g4 = *reinterpret_cast<const float4*>(dp_s + rr * dout + 4 * jq);
            const float4 w1 = *reinterpret_cast<const float4*>(ws_s + c * wst + 4 * jq);
            const float4 w2 = *reinterpret_cast<const float4*>(wn_s + c * wst + 4 * jq);
            s1 = fmaf(g4.x, w1.x, fmaf(g4.y, w1.y, fmaf(g4.z, w1.z, fmaf(g4.w, w1.w, s1))));
            s2 = fmaf(g4.x, w2.x, fmaf(g4.y, w2.y, fmaf(g4.z, w2.z, fmaf(g4.w, w2.w, s2))));
          }
        } else {
          for (int j = 0; j < dout; ++j) {
            const float gv = dp_s[rr * dout + j];
            s1 = fmaf(gv, ws_s[c * wst + j], s1);
            s2 = fmaf(gv, wn_s[c * wst + j], s2);
          }
        }
        if (a.d_self) a.d_self[G * w + c] = s1;
        if (a.d_sums) a.d_sums[G * w + c] = s2 * cnt_s[rr];
      }
    }
  }
  // per-block partial in the parameter layout [dW_self | dW_neigh | db]
  const int nwd = w * dout;
  const int64_t ntot = 2 * (int64_t)nwd + dout;
  float* out = a.partial + (int64_t)blockIdx.x * ntot;
  if (Q4) {
#pragma unroll
    for (int k = 0; k < BMAXQ; ++k) {
      const int idx = threadIdx.x + 256 * k;
      if (idx < nslots) {
        const int c = idx / nq, jq = idx - c * nq;
        *reinterpret_cast<float4*>(out + c * dout + 4 * jq) = aS4[k];
        float* o2 = out + nwd + c * dout + 4 * jq;
        o2[0] = aN4[k].x;
        o2[1] = aN4[k].y;
        o2[2] = aN4[k].z;
        o2[3] = aN4[k].w;
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < BMAXACC; ++k) {
      const int idx = threadIdx.x + 256 * k;
      if (idx < nslots) {
        out[idx] = aS[k];
        out[nwd + idx] = aN[k];
      }
    }
  }
  if (threadIdx.x < dout) out[2 * nwd + threadIdx.x] = ab;
}

// Tiled weight gradients (self-compact forward): dW_self = hs^T d_pre,
// dW_neigh = mean^T d_pre over this block's rows, each thread a 4x4 register
// tile (2 LDS.128 per 16 FFMA), per-block partial in the parameter layout.
// Tiles are double-buffered: the [hs | mean] rows, d_h and (for the ReLU mask)
// h of tile t+1 are copied to shared memory with cp.async while tile t is
// multiplied, so each CTA pays one memory latency, not one per tile.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}

template <int NQ>
__global__ void __launch_bounds__(256, 2) k_sage_wgrad(const SgMeta* __restrict__ meta, BwdArgs a) {
  // prologue before the PDL wait: barrier init and the weight staging read
  // nothing the preceding kernel writes (parameters change only in the step's
  // last kernel, and a graph replay / eager step never overlaps the previous one)
  constexpr int TR = 32;
  extern __shared__ __align__(16) float smem[];
  const int w = a.w, dout = a.dout, K = 2 * w, wst = dout + 4;
  const bool need_c = a.d_self != nullptr || a.d_sums != nullptr;
  // A = [hs plane [TR][w] | mean plane [TR][w]]: a tile of each is contiguous in
  // global memory and lands with ONE bulk copy (byte-counted on bar[s]); d_h,
  // h, counts by cp.async
  const int stage_f = TR * K + 2 * TR * dout + TR;  // A | d_h | h | counts
  float* ws_s = smem;                  // [w][dout+4] (need_c)
  float* wn_s = ws_s + w * wst;
  float* stg = wn_s + w * wst;         // 2 x stage
  uint64_t* bar = reinterpret_cast<uint64_t*>(stg + 2 * stage_f);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar + 1)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (need_c)
    for (int i = threadIdx.x; i < w * dout; i += blockDim.x) {
      const int c = i / dout, j = i - c * dout;
      ws_s[c * wst + j] = a.ws[i];
      wn_s[c * wst + j] = a.wn[i];
    }
  SG_PDL_ENTRY();
  const int n = meta->n_own[a.l][a.d];
  const int own0 = meta->own_off[a.l][a.d];
  const int ncg = K / 4, nslots = ncg * NQ, dq = dout / 4;
  const int ntiles = (n + TR - 1) / TR;
  const bool scat = a.sc_enc != nullptr;
  auto issue = [&](int tile, int s) {
    float* A_s = stg + s * stage_f;
    float* dh_s = A_s + TR * K;
    float* hh_s = dh_s + TR * dout;
    float* cn_s = hh_s + TR * dout;
    const int r0 = tile * TR, nr = min(TR, n - r0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of this stage are done
    if (threadIdx.x == 0) {
      const uint32_t mb = (uint32_t)__cvta_generic_to_shared(bar + s);
      const uint32_t bytes = 4u * (uint32_t)(nr * w);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(2u * bytes) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(A_s)),
                   "l"(a.h_prev + (int64_t)(own0 + r0) * w), "r"(bytes), "r"(mb)
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(A_s + TR * w)),
                   "l"(a.mean + (int64_t)(own0 + r0) * w), "r"(bytes), "r"(mb)
                   : "memory");
    }
    for (int idx = threadIdx.x; idx < (TR - nr) * K / 4; idx += 256) {  // rows past n: zeros (0 * garbage may be NaN)
      const int r = nr + idx / (K / 4), q = idx - (r - nr) * (K / 4);
      float* dst = 4 * q < w ? A_s + r * w + 4 * q : A_s + TR * w + r * w + 4 * q - w;
      *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int idx = threadIdx.x; idx < TR * dq; idx += 256) {
      const int r = idx / dq, q = idx - r * dq;
      if (r0 + r < n) {
        const int64_t G = own0 + r0 + r;
        if (!scat) cp_async16(dh_s + r * dout + 4 * q, a.d_h + G * dout + 4 * q);
        if (!a.final_) cp_async16(hh_s + r * dout + 4 * q, a.h + G * dout + 4 * q);
      } else if (!scat) {
        *reinterpret_cast<float4*>(dh_s + r * dout + 4 * q) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    if (need_c && threadIdx.x < TR && r0 + (int)threadIdx.x < n)
      cp_async4(cn_s + threadIdx.x, a.counts + own0 + r0 + threadIdx.x);
  };
  float acc[2][4][4];
#pragma unroll
  for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[s2][i][0] = acc[s2][i][1] = acc[s2][i][2] = acc[s2][i][3] = 0.f;
  float ab = 0.f;
  if (blockIdx.x < ntiles) issue(blockIdx.x, 0);
  asm volatile("cp.async.commit_group;" ::: "memory");
  int s = 0;
  for (int tile = blockIdx.x, it = 0; tile < ntiles; tile += gridDim.x, s ^= 1, ++it) {
    const int r0 = tile * TR;
    if (tile + (int)gridDim.x < ntiles) issue(tile + gridDim.x, s ^ 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (scat) {
      // d_h rows of the tile = transposed SpMM of layer l+1 while the [hs | mean]
      // tile lands: 4 rows per warp at once, each row's out-edges split over
      // GPR lane groups of LPR lanes (one float4 of the row per lane), fixed
      // xor tree over the groups (deterministic), + d_self on self rows.
      float* dh_w = stg + s * stage_f + TR * K;
      const int LPR = dq, GPR = 8 / dq;  // dout in {4, 8, 16, 32}
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      const int slot = lane / LPR, lr = lane - slot * LPR;
      const int rl = warp * 4 + slot / GPR, grp = slot % GPR;
      const int q = r0 + rl;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      int64_t U = 0;
      if (q < n) {
        U = own0 + q;
        const int b = a.sc_beg[a.sc_key_base + U], e = a.sc_end[a.sc_key_base + U];
        for (int j = b + grp; j < e; j += GPR) {
          const int code = a.sc_enc[j];
          const float* row = code >= 0 ? a.sc_dsums + (int64_t)code * dout
                                       : a.sc_recv + (int64_t)(-code - 1) * a.sc_stride;
          const float4 v = *reinterpret_cast<const float4*>(row + 4 * lr);
          acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
      }
      for (int o = LPR; o < LPR * GPR; o <<= 1) {  // the group bits of the lane
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
        acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
        acc.w += __shfl_xor_sync(0xffffffffu, acc.w, o);
      }
      if (grp == 0) {
        if (q < n) {
          const int p = a.sc_grouped[a.sc_voff_src + U];
          if (p < meta->nV[a.l + 1]) {
            const int64_t v = meta->own_off[a.l + 1][a.d] + a.sc_rank[a.sc_voff_dst + p];
            const float4 sv = *reinterpret_cast<const float4*>(a.sc_dself + v * dout + 4 * lr);
            acc.x = sv.x + acc.x; acc.y = sv.y + acc.y; acc.z = sv.z + acc.z; acc.w = sv.w + acc.w;
          }
        }
        *reinterpret_cast<float4*>(dh_w + rl * dout + 4 * lr) = acc;  // rows past n: zeros
      }
    }
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    sg_mbar_wait((uint32_t)__cvta_generic_to_shared(bar + s), (it >> 1) & 1);  // this stage's bulk copies
    __syncthreads();
    const float* A_s = stg + s * stage_f;
    float* dp_s = const_cast<float*>(A_s) + TR * K;
    const float* hh_s = dp_s + TR * dout;
    const float* cn_s = hh_s + TR * dout;
    if (!a.final_)
      for (int idx = threadIdx.x; idx < TR * dout; idx += 256)
        if (!(hh_s[idx] > 0.f)) dp_s[idx] = 0.f;
    __syncthreads();
#pragma unroll
    for (int s2 = 0; s2 < 2; ++s2) {
      const int slot = threadIdx.x + 256 * s2;
      if (slot < nslots) {
        const int cg = slot / NQ, jg = slot - cg * NQ;
        const float* ab = 4 * cg < w ? A_s + 4 * cg : A_s + TR * w + 4 * cg - w;
#pragma unroll 4
        for (int r = 0; r < TR; ++r) {
          const float4 a4 = *reinterpret_cast<const float4*>(ab + r * w);
          const float4 g4 = *reinterpret_cast<const float4*>(dp_s + r * dout + 4 * jg);
          const float av[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            acc[s2][i][0] = fmaf(av[i], g4.x, acc[s2][i][0]);
            acc[s2][i][1] = fmaf(av[i], g4.y, acc[s2][i][1]);
            acc[s2][i][2] = fmaf(av[i], g4.z, acc[s2][i][2]);
            acc[s2][i][3] = fmaf(av[i], g4.w, acc[s2][i][3]);
          }
        }
      }
    }
    if (threadIdx.x < dout)
      for (int r = 0; r < TR; ++r) ab += dp_s[r * dout + threadIdx.x];
    if (need_c) {
      const int nrow = min(TR, n - r0);
      for (int idx = threadIdx.x; idx < nrow * w; idx += blockDim.x) {
        const int r = idx / w, c = idx - r * w;
        const int64_t G = own0 + r0 + r;
        float s1 = 0.f, s2v = 0.f;
        for (int jq = 0; jq < NQ; ++jq) {
          const float4 g4 = *reinterpret_cast<const float4*>(dp_s + r * dout + 4 * jq);
          const float4 w1 = *reinterpret_cast<const float4*>(ws_s + c * wst + 4 * jq);
          const float4 w2 = *reinterpret_cast<const float4*>(wn_s + c * wst + 4 * jq);
          s1 = fmaf(g4.x, w1.x, fmaf(g4.y, w1.y, fmaf(g4.z, w1.z, fmaf(g4.w, w1.w, s1))));
          s2v = fmaf(g4.x, w2.x, fmaf(g4.y, w2.y, fmaf(g4.z, w2.z, fmaf(g4.w, w2.w, s2v))));
        }
        if (a.d_self) a.d_self[G * w + c] = s1;
        if (a.d_sums) a.d_sums[G * w + c] = s2v / cn_s[r];
      }
    }
    __syncthreads();  // buffer s is refilled next iteration
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  const int nwd = w * dout;
  float* out = a.partial + (int64_t)blockIdx.x * (2 * (int64_t)nwd + dout);
#pragma unroll
  for (int s2 = 0; s2 < 2; ++s2) {
    const int slot = threadIdx.x + 256 * s2;
    if (slot < nslots) {
      const int cg = slot / NQ, jg = slot - cg * NQ;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int c = 4 * cg + i;
        float* o = (c < w ? out + c * dout : out + nwd + (c - w) * dout) + 4 * jg;
        *reinterpret_cast<float4*>(o) = make_float4(acc[s2][i][0], acc[s2][i][1], acc[s2][i][2], acc[s2][i][3]);
      }
    }
  }
  if (threadIdx.x < dout) out[2 * nwd + threadIdx.x] = ab;
}

// ---------------------------------------------------------------- scatter (transpose SpMM)
struct ScatArgs {
  int l, d, w, stride;
  int64_t voff_lm1, voff_l, key_base;
  const int32_t* grouped;
  const int32_t* rank;
  const int32_t* enc;  // sorted out-edges: >=0 owned dst row, <0 -(1+pair slot)
  const int32_t* srcbeg;
  const int32_t* srcend;
  const float* d_self;
  const float* d_sums;
  const float* bwd_recv;
  float* d_prev;
};

template <int VEC, int LPR, int NCH>
__global__ void __launch_bounds__(256) k_sage_scatter(const SgMeta* __restrict__ meta, ScatArgs a) {
  SG_PDL_ENTRY();
  using V = VecT<VEC>;
  using T = typename V::T;
  constexpr int NG = 32 / LPR;  // lane groups per warp, each takes every NG-th edge
  const int l = a.l, d = a.d, w = a.w;
  const int n_prev = meta->n_own[l - 1][d];
  const int prev0 = meta->own_off[l - 1][d];
  const int own0 = meta->own_off[l][d];
  const int64_t nVl = meta->nV[l];
  const int lane = threadIdx.x & 31;
  const int gi = lane / LPR, lr = lane % LPR;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = gw; u < n_prev; u += nw) {
    const int64_t U = prev0 + u;
    T acc[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) acc[c] = V::zero();
    const int b = a.srcbeg[a.key_base + U], e = a.srcend[a.key_base + U];
    for (int jb = b; jb < e; jb += 32) {
      const int j = jb + lane;
      const int my = j < e ? a.enc[j] : 0;
      const int cnt = min(32, e - jb);
      const int rounds = (cnt + NG - 1) / NG;
      for (int kk = 0; kk < rounds; ++kk) {
        const int k = kk * NG + gi;
        const int code = __shfl_sync(0xffffffffu, my, k < 32 ? k : 31);
        if (k < cnt) {
          const bool own = code >= 0;
          const float* row = own ? a.d_sums + (int64_t)code * w
                                 : a.bwd_recv + (int64_t)(-code - 1) * a.stride;
#pragma unroll
          for (int c = 0; c < NCH; ++c) {
            const int col = (c * LPR + lr) * VEC;
            if (col < w) {
              if (own || (a.stride & 3) == 0) V::add(acc[c], V::ld(row + col));
              else V::add(acc[c], V::ld_any(row + col));
            }
          }
        }
      }
    }
    // fixed-order tree over the lane groups (deterministic)
#pragma unroll
    for (int o = LPR; o < 32; o <<= 1) {
#pragma unroll
      for (int c = 0; c < NCH; ++c) V::add(acc[c], V::shfl_xor(acc[c], o));
    }
    if (gi == 0) {
      const int p = a.grouped[a.voff_lm1 + U];
      float* out = a.d_prev + U * w;
      if (p < nVl) {
        const int64_t v = own0 + a.rank[a.voff_l + p];
        const float* sr = a.d_self + v * w;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          const int col = (c * LPR + lr) * VEC;
          if (col < w) {
            T s = V::ld(sr + col);
            V::add(s, acc[c]);
            acc[c] = s;
          }
        }
      }
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const int col = (c * LPR + lr) * VEC;
        if (col < w) V::st(out + col, acc[c]);
      }
    }
  }
}

// Narrow rows (w <= 4 LPR floats): one LPR-lane group per source row, 32/LPR
// rows per warp. Most source rows have a handful of out-edges (C2 layer 2:
// 40K edges over 27K rows), so a warp per row idled most lanes through a
// chain of dependent loads; here each group walks its row's out-edges in
// order, four row loads in flight. Rows with more than SC_HEAVY out-edges
// (power-law hubs) are summed by the whole warp afterwards, as in
// k_sage_scatter (lane groups take every (32/LPR)-th edge, fixed xor tree).
constexpr int SC_HEAVY = 12;

template <int LPR>
__global__ void __launch_bounds__(256) k_sage_scatter_grp(const SgMeta* __restrict__ meta, ScatArgs a) {
  SG_PDL_ENTRY();
  constexpr int RW = 32 / LPR;
  const int l = a.l, d = a.d, w = a.w;
  const int n_prev = meta->n_own[l - 1][d];
  const int prev0 = meta->own_off[l - 1][d];
  const int own0 = meta->own_off[l][d];
  const int64_t nVl = meta->nV[l];
  const int lane = threadIdx.x & 31;
  const int gi = lane / LPR, lr = lane % LPR;
  const int col = lr * 4;
  const bool colok = col < w;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  auto row_of = [&](int code) -> const float* {
    return code >= 0 ? a.d_sums + (int64_t)code * w : a.bwd_recv + (int64_t)(-code - 1) * a.stride;
  };
  auto load = [&](int code) -> float4 {
    const float* row = row_of(code);
    if (code >= 0 || (a.stride & 3) == 0) return __ldg(reinterpret_cast<const float4*>(row + col));
    return make_float4(row[col], row[col + 1], row[col + 2], row[col + 3]);
  };
  for (int64_t u0 = gw * RW; u0 < n_prev; u0 += nw * RW) {
    const int64_t u = u0 + gi;
    const bool valid = u < n_prev;
    const int64_t U = prev0 + u;
    int b = 0, e = 0, p = (int)nVl;
    if (valid) {
      b = a.srcbeg[a.key_base + U];
      e = a.srcend[a.key_base + U];
      p = a.grouped[a.voff_lm1 + U];
    }
    const int64_t v = (valid && p < nVl) ? own0 + a.rank[a.voff_l + p] : -1;
    const bool heavy = e - b > SC_HEAVY;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (valid && !heavy) {
      for (int j = b; j < e; j += 4) {
        int code[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) code[t] = j + t < e ? a.enc[j + t] : 0;
        float4 x[4];
#pragma unroll
        for (int t = 0; t < 4; ++t)
          x[t] = (j + t < e && colok) ? load(code[t]) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          acc.x += x[t].x; acc.y += x[t].y; acc.z += x[t].z; acc.w += x[t].w;
        }
      }
    }
    unsigned hm = __ballot_sync(0xffffffffu, valid && heavy && lr == 0);
    while (hm) {
      const int owner = __ffs(hm) - 1;
      hm &= hm - 1;
      const int hb = __shfl_sync(0xffffffffu, b, owner), he = __shfl_sync(0xffffffffu, e, owner);
      // 32 edges per chunk: every round's row load issued before any add,
      // the next chunk's edge codes fetched while this chunk's rows land
      float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
      int my = hb + lane < he ? a.enc[hb + lane] : 0;
      for (int jb = hb; jb < he; jb += 32) {
        const int cnt = min(32, he - jb);
        const int nxt = jb + 32 + lane < he ? a.enc[jb + 32 + lane] : 0;
        float4 x[LPR];
#pragma unroll
        for (int kk = 0; kk < LPR; ++kk) {  // LPR rounds of RW lane groups cover 32 edges
          const int k = kk * RW + gi;
          const int code = __shfl_sync(0xffffffffu, my, k);
          x[kk] = (k < cnt && colok) ? load(code) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int kk = 0; kk < LPR; ++kk) {
          t.x += x[kk].x; t.y += x[kk].y; t.z += x[kk].z; t.w += x[kk].w;
        }
        my = nxt;
      }
#pragma unroll
      for (int o = LPR; o < 32; o <<= 1) {
        t.x += __shfl_xor_sync(0xffffffffu, t.x, o);
        t.y += __shfl_xor_sync(0xffffffffu, t.y, o);
        t.z += __shfl_xor_sync(0xffffffffu, t.z, o);
        t.w += __shfl_xor_sync(0xffffffffu, t.w, o);
      }
      if (gi == owner / LPR) acc = t;
    }
    if (valid && colok) {
      if (v >= 0) {
        float4 s = __ldg(reinterpret_cast<const float4*>(a.d_self + v * w + col));
        s.x += acc.x; s.y += acc.y; s.z += acc.z; s.w += acc.w;
        acc = s;
      }
      *reinterpret_cast<float4*>(a.d_prev + U * w + col) = acc;
    }
  }
}

template <int LPR>
int launch_scat_grp(const SgMeta* meta, const ScatArgs& a, int64_t max_rows, cudaStream_t st) {
  const int grid = clamp_grid(div_up(max_rows, 8 * (32 / LPR)), kSMs * 8);
  ::sg::launch(k_sage_scatter_grp<LPR>, grid, 256, 0, st, meta, a);
  SG_CHECK_LAUNCH("k_sage_scatter_grp");
  return SG_OK;
}

template <int VEC, int LPR, int NCH>
int launch_scat(const SgMeta* meta, const ScatArgs& a, int64_t max_rows, cudaStream_t st) {
  const int grid = clamp_grid(div_up(max_rows, 8), kSMs * 8);
  ::sg::launch(k_sage_scatter<VEC, LPR, NCH>, grid, 256, 0, st, meta, a);
  SG_CHECK_LAUNCH("k_sage_scatter");
  return SG_OK;
}

int dispatch_scat(const SgMeta* meta, const ScatArgs& a, int64_t max_rows, cudaStream_t st) {
  const int w = a.w;
  if (w % 4 == 0 && w <= 32 && std::getenv("SG_SCATTER_WARP") == nullptr) {
    if (w <= 4) return launch_scat_grp<1>(meta, a, max_rows, st);
    if (w <= 8) return launch_scat_grp<2>(meta, a, max_rows, st);
    if (w <= 16) return launch_scat_grp<4>(meta, a, max_rows, st);
    return launch_scat_grp<8>(meta, a, max_rows, st);
  }
  if (w % 4 == 0) {
    if (w <= 16) return launch_scat<4, 4, 1>(meta, a, max_rows, st);
    if (w <= 32) return launch_scat<4, 8, 1>(meta, a, max_rows, st);
    if (w <= 64) return launch_scat<4, 16, 1>(meta, a, max_rows, st);
    if (w <= 128) return launch_scat<4, 32, 1>(meta, a, max_rows, st);
    if (w <= 512) return launch_scat<4, 32, 4>(meta, a, max_rows, st);
  } else {
    if (w <= 8) return launch_scat<1, 8, 1>(meta, a, max_rows, st);
    if (w <= 32) return launch_scat<1, 32, 1>(meta, a, max_rows, st);
    if (w <= 128) return launch_scat<1, 32, 4>(meta, a, max_rows, st);
    if (w <= 512) return launch_scat<1, 32, 16>(meta, a, max_rows, st);
  }
  set_error("sage_scatter_bwd: width > 512 unsupported");
  return SG_ERR_ARG;
}

}  // namespace

#define SPLIT_PTRS                                                     \
  const char* base = (const char*)split_ws;                           \
  const SgSplitLayout& y = *lay;                                       \
  const SgMeta* meta = (const SgMeta*)(base + y.o_meta);               \
  auto I32 = [&](int64_t o) { return (const int32_t*)(base + o); };

static int agg_common(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                      const float* h_prev, const int32_t* src_row, int32_t w, int32_t h_stride, float* sums,
                      float* counts, float* sendbuf, int32_t send_stride, const int32_t* dperm,
                      int64_t max_rows, void* stream, const int64_t* peer_recv = nullptr) {
  SG_REQUIRE(split_ws && lay, "sage_agg_fwd: null workspace");
  SPLIT_PTRS
  SG_REQUIRE(l >= 1 && l <= y.L && d >= 0 && d < y.g, "sage_agg_fwd: bad layer/device");
  SG_REQUIRE(send_stride >= w + 1 || y.g == 1, "sage_agg_fwd: send stride < w+1");
  if (max_rows <= 0) return SG_OK;
  AggArgs a;
  memset(&a, 0, sizeof(a));
  a.l = l;
  a.d = d;
  a.w = w;
  a.stride = send_stride;
  a.eoff_li = y.eoff[l - 1];
  a.rbase_li = y.rbase[l - 1];
  a.pbase_l = y.pbase[l];
  a.rowbeg = I32(y.o_rowbeg);
  a.rowend = I32(y.o_rowend);
  a.lsrc = I32(y.o_lsrc);
  a.dperm = dperm;
  a.sendpos = I32(y.o_sendpos);
  a.src_row = src_row;
  a.h_prev = h_prev;
  a.hst = h_stride > 0 ? h_stride : w;
  a.sums = sums;
  a.counts = counts;
  a.sendbuf = sendbuf;
  a.g = y.g;
  if (peer_recv) {
    SG_REQUIRE(y.g > 1, "sage_agg_fwd_peer: needs g > 1");
    a.xfer = I32(y.o_xfer) + y.pbase[l];
    for (int i = 0; i < y.g; ++i) a.peer.p[i] = peer_recv[i];
    SG_REQUIRE(a.peer.p[0] != 0, "sage_agg_fwd_peer: null peer buffer");
  }
  return dispatch_agg(meta, a, max_rows, (cudaStream_t)stream);
}

// sg_sage_agg_fwd with the push-to-owner fused into the epilogue: reference
// rows are stored straight into the owners' receive buffers (peer_recv: the g
// peer-mapped receive buffers of this round, receive-slot layout, row stride
// send_stride) instead of a local send buffer. dperm may be null.
extern "C" int sg_sage_agg_fwd_peer(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                                    const float* h_prev, const int32_t* src_row, int32_t w, int32_t h_stride,
                                    float* sums, float* counts, const int64_t* peer_recv, int32_t send_stride,
                                    const int32_t* dperm, int64_t max_rows, void* stream) {
  SG_REQUIRE(peer_recv, "sage_agg_fwd_peer: null peer table");
  return agg_common(split_ws, lay, l, d, h_prev, src_row, w, h_stride, sums, counts, nullptr, send_stride, dperm,
                    max_rows, stream, peer_recv);
}

extern "C" int sg_sage_agg_fwd(const void* split_ws, const SgSplitLayout* lay, int32_t l,
                               int32_t d, const float* h_prev, const int32_t* src_row, int32_t w,
                               int32_t h_stride, float* sums, float* counts, float* sendbuf,
                               int32_t send_stride, int64_t max_rows, void* stream) {
  return agg_common(split_ws, lay, l, d, h_prev, src_row, w, h_stride, sums, counts, sendbuf, send_stride,
                    nullptr, max_rows, stream);
}

extern "C" int sg_sage_agg_fwd_perm(const void* split_ws, const SgSplitLayout* lay, int32_t l,
                                    int32_t d, const float* h_prev, const int32_t* src_row,
                                    int32_t w, int32_t h_stride, float* sums, float* counts,
                                    float* sendbuf, int32_t send_stride, const int32_t* dperm,
                                    int64_t max_rows, void* stream) {
  return agg_common(split_ws, lay, l, d, h_prev, src_row, w, h_stride, sums, counts, sendbuf, send_stride,
                    dperm, max_rows, stream);
}

extern "C" int sg_sage_fused_fwd(const void* split_ws, const SgSplitLayout* lay, int32_t l,
                                 int32_t d, const float* h_prev, const int32_t* src_row, int32_t w,
                                 int32_t h_stride, int32_t dout, const float* w_self, const float* w_neigh,
                                 const float* bias, int32_t final_layer, float* mean, float* counts,
                                 float* hs, float* h, int64_t max_rows, void* stream) {
  SG_REQUIRE(split_ws && lay, "sage_fused_fwd: null workspace");
  SPLIT_PTRS
  SG_REQUIRE(y.g == 1, "sage_fused_fwd: single-device split only (no remote contributions)");
  SG_REQUIRE(l >= 1 && l <= y.L && d == 0, "sage_fused_fwd: bad layer/device");
  SG_REQUIRE(w % 4 == 0 && w <= 128 && (dout == 4 || dout == 8 || dout == 16 || dout == 32),
             "sage_fused_fwd: needs w % 4 == 0, w <= 128, dout in {4, 8, 16, 32}");
  if (max_rows <= 0) return SG_OK;
  FusedArgs a;
  memset(&a, 0, sizeof(a));
  a.l = l; a.d = d; a.w = w; a.dout = dout; a.final_ = final_layer;
  a.eoff_li = y.eoff[l - 1]; a.rbase_li = y.rbase[l - 1]; a.voff_l = y.voff[l];
  a.rowbeg = I32(y.o_rowbeg); a.rowend = I32(y.o_rowend); a.lsrc = I32(y.o_lsrc);
  a.selfrow = I32(y.o_selfrow); a.src_row = src_row; a.h_prev = h_prev;
  a.mean = mean; a.counts = counts; a.hs = hs;
  a.ws = w_self; a.wn = w_neigh; a.bias = bias; a.h = h;
  a.hst = h_stride > 0 ? h_stride : w;
  SG_REQUIRE(a.hst >= w && a.hst % 4 == 0 && a.hst <= 128 && (a.hst == w || w > 64),
             "sage_fused_fwd: h_stride must be a multiple of 4, >= w, <= 128 (padded rows need w > 64)");
  cudaStream_t st = (cudaStream_t)stream;
  // one kernel for every width (8 loads in flight per lane, 8-row tiles: one
  // row per warp, 4 CTAs/SM; measured best of UN 8/16 x RPW 1/2/4 x 2..8
  // CTAs/SM; for narrow rows level with aggregation + a separate GEMM)
  return launch_layer<8, 1, 4>(meta, a, max_rows, st);
}

extern "C" int sg_sage_combine_fwd(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                                   const float* h_prev, const int32_t* src_row, int32_t w, int32_t h_stride,
                                   int32_t dout,
                                   const float* w_self, const float* w_neigh, const float* bias,
                                   int32_t final_layer, const float* sums, float* counts, const float* recv,
                                   int32_t recv_stride, float* mean, float* hs, float* h, int64_t max_rows,
                                   void* stream) {
  SG_REQUIRE(split_ws && lay && sums && counts, "sage_combine_fwd: null argument");
  SPLIT_PTRS
  SG_REQUIRE(l >= 1 && l <= y.L && d >= 0 && d < y.g, "sage_combine_fwd: bad layer/device");
  SG_REQUIRE(w % 4 == 0 && w <= 128 && (dout == 4 || dout == 8 || dout == 16 || dout == 32),
             "sage_combine_fwd: needs w % 4 == 0, w <= 128, dout in {4, 8, 16, 32}");
  SG_REQUIRE(y.g == 1 || (recv && recv_stride % 4 == 0 && recv_stride >= w + 1),
             "sage_combine_fwd: recv stride must be a multiple of 4 and >= w + 1");
  if (max_rows <= 0) return SG_OK;
  FusedArgs a;
  memset(&a, 0, sizeof(a));
  a.l = l; a.d = d; a.w = w; a.dout = dout; a.final_ = final_layer;
  a.eoff_li = y.eoff[l - 1]; a.rbase_li = y.rbase[l - 1]; a.voff_l = y.voff[l];
  a.selfrow = I32(y.o_selfrow); a.src_row = src_row; a.h_prev = h_prev;
  a.mean = mean; a.counts = counts; a.hs = hs;
  a.ws = w_self; a.wn = w_neigh; a.bias = bias; a.h = h;
  a.sums = sums; a.recv = recv; a.contrib = I32(y.o_contrib); a.stride = recv_stride; a.g = y.g > 1 ? y.g : 0;
  a.hst = h_stride > 0 ? h_stride : w;
  SG_REQUIRE(a.hst >= w && a.hst % 4 == 0 && a.hst <= 128, "sage_combine_fwd: bad h_stride");
  return launch_layer<8, 1, 4>(meta, a, max_rows, (cudaStream_t)stream);
}

extern "C" int sg_sage_update(const void* split_ws, const SgSplitLayout* lay, int32_t l,
                              int32_t d, const float* h_prev, const int32_t* src_row, int32_t w,
                              int32_t dout, const float* sums, float* counts,
                              const float* recvbuf, int32_t recv_stride, const float* w_self,
                              const float* w_neigh, const float* bias, int32_t final_layer,
                              float* mean, float* h, float* hs_out, int64_t max_rows,
                              void* stream) {
  SG_REQUIRE(split_ws && lay, "sage_update: null workspace");
  SPLIT_PTRS
  SG_REQUIRE(l >= 1 && l <= y.L && d >= 0 && d < y.g, "sage_update: bad layer/device");
  SG_REQUIRE(dout >= 1 && w >= 1, "sage_update: dout/w out of range");
  SG_REQUIRE(y.g <= 32, "sage_update: g > 32");
  if (max_rows <= 0) return SG_OK;
  const size_t smem_fast = sizeof(float) * (2 * (size_t)w * dout + 2 * (size_t)UTR * (w + 1) +
                                            (size_t)UTR * (2 + y.g));
  if (dout > 256 || smem_fast > 227 * 1024) {
    // wide layer: mean / counts (/ self rows) here, then h = act(hs Ws + b + mean Wn)
    UpdArgs u;
    memset(&u, 0, sizeof(u));
    u.l = l; u.d = d; u.w = w; u.dout = dout; u.final_ = final_layer; u.g = y.g; u.stride = recv_stride;
    u.voff_l = y.voff[l]; u.h_prev = h_prev; u.src_row = src_row; u.selfrow = I32(y.o_selfrow);
    u.contrib = I32(y.o_contrib); u.sums = sums; u.counts = counts; u.recv = recvbuf;
    u.mean = mean; u.h = h; u.hs_out = hs_out; u.no_linear = 1;
    const size_t sm = sizeof(float) * (2 * (size_t)UTR * (w + 1) + (size_t)UTR * (2 + y.g));
    SG_REQUIRE(sm <= 227 * 1024, "sage_update: input width too large for shared memory");
    cudaStream_t st = (cudaStream_t)stream;
    const int grid = clamp_grid(div_up(max_rows, UTR), kSMs * 3);
    SG_CUDA(allow_max_smem<k_sage_update<false>>());
    ::sg::launch(k_sage_update<false>, grid, 256, sm, st, meta, u);
    SG_CHECK_LAUNCH("k_sage_update(mean)");
    GemmArgs g1;
    memset(&g1, 0, sizeof(g1));
    g1.R_dev = &meta->n_own[l][d];
    g1.K = w; g1.N = dout;
    if (hs_out) {
      g1.A = hs_out; g1.ar.mode = 0; g1.ar.base_dev = &meta->own_off[l][d];
    } else {
      g1.A = h_prev; g1.ar.mode = 2; g1.ar.base_dev = &meta->own_off[l][d];
      g1.ar.selfrow = I32(y.o_selfrow); g1.ar.prev0_dev = &meta->own_off[l - 1][d];
      g1.ar.voff_l = y.voff[l]; g1.ar.map = src_row;
    }
    g1.lda = w; g1.B = w_self; g1.ldb = dout; g1.C = h; g1.ldc = dout;
    g1.c_base_dev = &meta->own_off[l][d]; g1.bias = bias;
    int rc = dense_gemm_rows(g1, max_rows, st);
    if (rc) return rc;
    GemmArgs g2 = g1;
    memset(&g2.ar, 0, sizeof(g2.ar));
    g2.A = mean; g2.ar.mode = 0; g2.ar.base_dev = &meta->own_off[l][d];
    g2.B = w_neigh; g2.bias = nullptr; g2.accum = 1; g2.relu = final_layer ? 0 : 1;
    return dense_gemm_rows(g2, max_rows, st);
  }
  UpdArgs a;
  memset(&a, 0, sizeof(a));
  a.l = l;
  a.d = d;
  a.w = w;
  a.dout = dout;
  a.final_ = final_layer;
  a.g = y.g;
  a.stride = recv_stride;
  a.voff_l = y.voff[l];
  a.h_prev = h_prev;
  a.src_row = src_row;
  a.selfrow = I32(y.o_selfrow);
  a.contrib = I32(y.o_contrib);
  a.sums = sums;
  a.counts = counts;
  a.recv = recvbuf;
  a.ws = w_self;
  a.wn = w_neigh;
  a.bias = bias;
  a.mean = mean;
  a.h = h;
  const bool tiled = hs_out != nullptr && w % 4 == 0 &&
                     (dout == 4 || dout == 8 || dout == 16 || dout == 32);
  a.hs_out = tiled ? hs_out : nullptr;
  const size_t smem = sizeof(float) * (2 * (size_t)w * dout + 2 * (size_t)UTR * (w + 1) +
                                       (size_t)UTR * (2 + y.g));
  SG_REQUIRE(smem <= 227 * 1024, "sage_update: width too large for shared memory");
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = clamp_grid(div_up(max_rows, UTR), kSMs * 3);
  if (dout % 4 == 0) {
    SG_CUDA(allow_max_smem<k_sage_update<true>>());
    ::sg::launch(k_sage_update<true>, grid, 256, smem, st, meta, a);
  } else {
    SG_CUDA(allow_max_smem<k_sage_update<false>>());
    ::sg::launch(k_sage_update<false>, grid, 256, smem, st, meta, a);
  }
  SG_CHECK_LAUNCH("k_sage_update");
  if (tiled) {
    LinArgs la{l, d, w, dout, final_layer, hs_out, mean, w_self, w_neigh, bias, h};
    return launch_linear(meta, la, max_rows, st);
  }
  return SG_OK;
}

extern "C" int sg_sage_bwd_rows(const void* split_ws, const SgSplitLayout* lay, int32_t l,
                                int32_t d, const float* h_prev, const int32_t* src_row, int32_t w,
                                int32_t dout, const float* d_h, const float* h,
                                int32_t final_layer, const float* mean, const float* counts,
                                const float* w_self, const float* w_neigh, float* partial,
                                int32_t nblocks, float* d_self, float* d_sums, int32_t self_compact,
                                int64_t max_rows, void* stream) {
  SG_REQUIRE(split_ws && lay, "sage_bwd_rows: null workspace");
  SPLIT_PTRS
  SG_REQUIRE(l >= 1 && l <= y.L && d >= 0 && d < y.g, "sage_bwd_rows: bad layer/device");
  SG_REQUIRE(dout >= 1 && w >= 1, "sage_bwd_rows: dout/w out of range");
  SG_REQUIRE(nblocks >= 1, "sage_bwd_rows: nblocks >= 1");
  const bool q4 = dout % 4 == 0;
  const bool fits = dout <= 32 && (q4 ? (int64_t)w * (dout / 4) <= 256 * BMAXQ
                                      : (int64_t)w * dout <= 256 * BMAXACC);
  if (!fits) {
    // wide layer: per-split weight-gradient partials [dW_self | dW_neigh | db]
    // and the input gradients as dense GEMMs (dense.cu); d_pre = d_h * ReLU'(h)
    cudaStream_t st = (cudaStream_t)stream;
    const int32_t* own = &meta->own_off[l][d];
    const float* gmask = final_layer ? nullptr : h;
    TnArgs t;
    memset(&t, 0, sizeof(t));
    t.R_dev = &meta->n_own[l][d];
    t.K = w; t.N = dout; t.lda = w;
    if (self_compact) {
      t.A = h_prev; t.ar.mode = 0; t.ar.base_dev = own;
    } else {
      t.A = h_prev; t.ar.mode = 2; t.ar.base_dev = own; t.ar.selfrow = I32(y.o_selfrow);
      t.ar.prev0_dev = &meta->own_off[l - 1][d]; t.ar.voff_l = y.voff[l]; t.ar.map = src_row;
    }
    t.G = d_h; t.ldg = dout; t.g_base_dev = own; t.gmask = gmask;
    t.P = partial; t.pstride = 2 * (int64_t)w * dout + dout; t.p_off = 0; t.nsplit = nblocks;
    int rc = dense_gemm_tn_partial(t, st);
    if (rc) return rc;
    TnArgs t2 = t;
    memset(&t2.ar, 0, sizeof(t2.ar));
    t2.A = mean; t2.ar.mode = 0; t2.ar.base_dev = own; t2.ones = 1; t2.p_off = (int64_t)w * dout;
    rc = dense_gemm_tn_partial(t2, st);
    if (rc) return rc;
    for (int which = 0; which < 2; ++which) {
      float* out = which == 0 ? d_self : d_sums;
      if (!out) continue;
      GemmArgs g;
      memset(&g, 0, sizeof(g));
      g.R_dev = &meta->n_own[l][d];
      g.K = dout; g.N = w;
      g.A = d_h; g.lda = dout; g.ar.mode = 0; g.ar.base_dev = own;
      g.amask = gmask; g.lda_mask = dout;
      g.B = which == 0 ? w_self : w_neigh; g.ldb = dout; g.bt = 1;
      g.C = out; g.ldc = w; g.c_base_dev = own;
      g.rdiv = which == 0 ? nullptr : counts;
      rc = dense_gemm_rows(g, max_rows, st);
      if (rc) return rc;
    }
    return SG_OK;
  }
  (void)max_rows;
  BwdArgs a;
  memset(&a, 0, sizeof(a));
  a.l = l;
  a.d = d;
  a.w = w;
  a.dout = dout;
  a.final_ = final_layer;
  a.self_compact = self_compact;
  a.voff_l = y.voff[l];
  a.h_prev = h_prev;
  a.src_row = src_row;
  a.selfrow = I32(y.o_selfrow);
  a.d_h = d_h;
  a.h = h;
  a.mean = mean;
  a.counts = counts;
  a.ws = w_self;
  a.wn = w_neigh;
  a.partial = partial;
  a.d_self = d_self;
  a.d_sums = d_sums;
  if (self_compact && q4 && w % 4 == 0 && dout <= 32 && 2 * w * (dout / 4) <= 4 * 512) {
    const size_t sm2 = sizeof(float) * (2 * (32 * (size_t)(2 * w + 4) + 2 * 32 * (size_t)dout + 32) +
                                        2 * (size_t)w * (dout + 4)) + 16;
    SG_REQUIRE(sm2 <= 227 * 1024, "sage_wgrad: width too large for shared memory");
    cudaStream_t st2 = (cudaStream_t)stream;
    cudaError_t attr = cudaSuccess;
    switch (dout / 4) {
      case 1: attr = allow_max_smem<k_sage_wgrad<1>>(); SG_CUDA(attr); ::sg::launch(k_sage_wgrad<1>, nblocks, 256, sm2, st2, meta, a); break;
      case 2: attr = allow_max_smem<k_sage_wgrad<2>>(); SG_CUDA(attr); ::sg::launch(k_sage_wgrad<2>, nblocks, 256, sm2, st2, meta, a); break;
      case 4: attr = allow_max_smem<k_sage_wgrad<4>>(); SG_CUDA(attr); ::sg::launch(k_sage_wgrad<4>, nblocks, 256, sm2, st2, meta, a); break;
      default: attr = allow_max_smem<k_sage_wgrad<8>>(); SG_CUDA(attr); ::sg::launch(k_sage_wgrad<8>, nblocks, 256, sm2, st2, meta, a); break;
    }
    SG_CHECK_LAUNCH("k_sage_wgrad");
    return SG_OK;
  }
  const int wst = q4 ? dout + 4 : dout + 1;
  const size_t smem = sizeof(float) * ((size_t)BTR * dout + 2 * (size_t)w * wst +
                                       2 * (size_t)BTR * (w + 1) + 2 * BTR);
  SG_REQUIRE(smem <= 227 * 1024, "sage_bwd_rows: width too large for shared memory");
  cudaStream_t st = (cudaStream_t)stream;
  if (q4) {
    SG_CUDA(allow_max_smem<k_sage_bwd_rows<true>>());
    ::sg::launch(k_sage_bwd_rows<true>, nblocks, 256, smem, st, meta, a);
  } else {
    SG_CUDA(allow_max_smem<k_sage_bwd_rows<false>>());
    ::sg::launch(k_sage_bwd_rows<false>, nblocks, 256, smem, st, meta, a);
  }
  SG_CHECK_LAUNCH("k_sage_bwd_rows");
  return SG_OK;
}

// Transposed SpMM of layer l (d_prev rows of layer l-1, engine.py:263-273) fused
// with the row-local backward of layer l-1 (engine.py:237-244): k_sage_wgrad in
// scatter mode. hs / mean / counts / h are layer l-1's (self-compact forward).
extern "C" int sg_sage_scatter_bwd_rows(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                                        const float* d_self, const float* d_sums, const float* bwd_recv,
                                        int32_t recv_stride, const int32_t* enc, const int32_t* srcbeg,
                                        const int32_t* srcend, int64_t key_base, const float* hs, int32_t w_in,
                                        int32_t w, const float* h, const float* mean, const float* counts,
                                        const float* w_self, const float* w_neigh, float* partial,
                                        int32_t nblocks, float* d_self_prev, float* d_sums_prev,
                                        int64_t max_rows, void* stream) {
  SG_REQUIRE(split_ws && lay && enc && srcbeg && srcend && hs && h && mean, "sage_scatter_bwd_rows: null argument");
  SPLIT_PTRS
  SG_REQUIRE(l >= 2 && l <= y.L && d >= 0 && d < y.g, "sage_scatter_bwd_rows: bad layer/device");
  SG_REQUIRE(nblocks >= 1, "sage_scatter_bwd_rows: nblocks >= 1");
  SG_REQUIRE((w == 4 || w == 8 || w == 16 || w == 32) && w_in % 4 == 0 && 2 * w_in * (w / 4) <= 4 * 512,
             "sage_scatter_bwd_rows: needs d_h width in {4, 8, 16, 32} and a tiled input width");
  SG_REQUIRE(y.g == 1 || (bwd_recv && recv_stride % 4 == 0), "sage_scatter_bwd_rows: recv stride % 4 != 0");
  (void)max_rows;
  BwdArgs a;
  memset(&a, 0, sizeof(a));
  a.l = l - 1; a.d = d; a.w = w_in; a.dout = w; a.final_ = 0; a.self_compact = 1;
  a.voff_l = y.voff[l - 1]; a.h_prev = hs; a.selfrow = I32(y.o_selfrow);
  a.h = h; a.mean = mean; a.counts = counts; a.ws = w_self; a.wn = w_neigh;
  a.partial = partial; a.d_self = d_self_prev; a.d_sums = d_sums_prev;
  a.sc_enc = enc; a.sc_beg = srcbeg; a.sc_end = srcend; a.sc_grouped = I32(y.o_grouped);
  a.sc_rank = I32(y.o_rank); a.sc_dself = d_self; a.sc_dsums = d_sums; a.sc_recv = bwd_recv;
  a.sc_key_base = key_base; a.sc_voff_src = y.voff[l - 1]; a.sc_voff_dst = y.voff[l]; a.sc_stride = recv_stride;
  const size_t sm2 = sizeof(float) * (2 * (32 * (size_t)(2 * w_in + 4) + 2 * 32 * (size_t)w + 32) +
                                      2 * (size_t)w_in * (w + 4));
  SG_REQUIRE(sm2 <= 227 * 1024, "sage_scatter_bwd_rows: width too large for shared memory");
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t attr = cudaSuccess;
  switch (w / 4) {
    case 1: attr = allow_max_smem<k_sage_wgrad<1>>(); SG_CUDA(attr); ::sg::launch(k_sage_wgrad<1>, nblocks, 256, sm2, st, meta, a); break;
    case 2: attr = allow_max_smem<k_sage_wgrad<2>>(); SG_CUDA(attr); ::sg::launch(k_sage_wgrad<2>, nblocks, 256, sm2, st, meta, a); break;
    case 4: attr = allow_max_smem<k_sage_wgrad<4>>(); SG_CUDA(attr); ::sg::launch(k_sage_wgrad<4>, nblocks, 256, sm2, st, meta, a); break;
    default: attr = allow_max_smem<k_sage_wgrad<8>>(); SG_CUDA(attr); ::sg::launch(k_sage_wgrad<8>, nblocks, 256, sm2, st, meta, a); break;
  }
  SG_CHECK_LAUNCH("k_sage_wgrad(scatter)");
  return SG_OK;
}

extern "C" int sg_sage_scatter_bwd(const void* split_ws, const SgSplitLayout* lay, int32_t l,
                                   int32_t d, int32_t w, const float* d_self, const float* d_sums,
                                   const float* bwd_recv, int32_t recv_stride,
                                   const int32_t* enc, const int32_t* srcbeg,
                                   const int32_t* srcend, int64_t key_base, float* d_prev,
                                   int64_t max_rows, void* stream) {
  SG_REQUIRE(split_ws && lay, "sage_scatter_bwd: null workspace");
  SPLIT_PTRS
  SG_REQUIRE(l >= 1 && l <= y.L && d >= 0 && d < y.g, "sage_scatter_bwd: bad layer/device");
  if (max_rows <= 0) return SG_OK;
  ScatArgs a;
  memset(&a, 0, sizeof(a));
  a.l = l;
  a.d = d;
  a.w = w;
  a.stride = recv_stride;
  a.voff_lm1 = y.voff[l - 1];
  a.voff_l = y.voff[l];
  a.key_base = key_base;
  a.grouped = I32(y.o_grouped);
  a.rank = I32(y.o_rank);
  a.enc = enc;
  a.srcbeg = srcbeg;
  a.srcend = srcend;
  a.d_self = d_self;
  a.d_sums = d_sums;
  a.bwd_recv = bwd_recv;
  a.d_prev = d_prev;
  return dispatch_scat(meta, a, max_rows, (cudaStream_t)stream);
}

}  // namespace sg
