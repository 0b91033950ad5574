// GraphSAGE (mean aggregator) forward / backward for one device of a split.
//
//   sg_sage_agg_fwd     local_aggregate (engine.py:180-195): CSR-by-destination
//                       segment-sum SpMM, warp (or sub-warp) per destination
//                       row, 128-bit loads, 4 source rows in flight per lane
//                       group; reference rows are packed straight into the
//                       push-to-owner send buffer (fused pack epilogue).
//   sg_sage_update      owner combine in ascending sender order + mean +
//                       h_self@W_self + mean@W_neigh + b + ReLU (:197-226),
//                       FP32 FFMA with both weight matrices staged in smem.
//   sg_sage_bwd_rows    d_pre, weight/bias gradient partials (deterministic
//                       per-block), d_self and d_sums (:228-254).
//   sg_sage_scatter_bwd transpose SpMM over CSR-by-source (:263-276) reading
//                       reference destinations from the push-from-owner
//                       payload (fused unpack).
// All arithmetic is FP32 (parity target rel 1e-4 vs the float64 reference).
#include <cstring>

#include "common.cuh"

namespace sg {
namespace {

struct AggArgs {
  int l, d, w, stride;
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
};

template <int VEC>
struct VecT;
template <>
struct VecT<4> {
  using T = float4;
  __device__ static float4 zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
  __device__ static float4 ld(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
  __device__ static void add(float4& a, const float4& b) {
    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
  }
  __device__ static void st(float* p, const float4& v) { *reinterpret_cast<float4*>(p) = v; }
  __device__ static void st_any(float* p, const float4& v) { p[0] = v.x; p[1] = v.y; p[2] = v.z; p[3] = v.w; }
};
template <>
struct VecT<1> {
  using T = float;
  __device__ static float zero() { return 0.f; }
  __device__ static float ld(const float* p) { return __ldg(p); }
  __device__ static void add(float& a, const float& b) { a += b; }
  __device__ static void st(float* p, const float& v) { *p = v; }
  __device__ static void st_any(float* p, const float& v) { *p = v; }
};

// Warp-or-subwarp per destination row. LPR lanes per row, each lane owns NCH
// chunks of VEC consecutive columns: col = (ch*LPR + lane_in_row)*VEC.
template <int VEC, int LPR, int NCH>
__global__ void __launch_bounds__(256) k_sage_agg(const SgMeta* __restrict__ meta, AggArgs a) {
  using V = VecT<VEC>;
  using T = typename V::T;
  constexpr int RPW = 32 / LPR;
  const int l = a.l, d = a.d, w = a.w;
  const int n_own = meta->n_own[l][d];
  const int R = n_own + meta->n_ref[l][d];
  const int own0 = meta->own_off[l][d], ref0 = meta->ref_off[l][d];
  const int prev0 = meta->own_off[l - 1][d];
  const int64_t rb = a.rbase_li + own0 + ref0;
  const int lane = threadIdx.x & 31;
  const int sub = lane / LPR, lr = lane % LPR;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = gw * RPW + sub; q < R; q += nw * RPW) {
    const int b = a.rowbeg[rb + q], e = a.rowend[rb + q];
    T acc[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) acc[c] = V::zero();
    auto rowptr = [&](int j) -> const float* {
      const int64_t x = a.dperm ? (int64_t)a.dperm[j] : a.eoff_li + j;
      int r = prev0 + a.lsrc[x];
      if (a.src_row) r = a.src_row[r];
      return a.h_prev + (int64_t)r * w;
    };
    int j = b;
    for (; j + 4 <= e; j += 4) {
      const float* p0 = rowptr(j);
      const float* p1 = rowptr(j + 1);
      const float* p2 = rowptr(j + 2);
      const float* p3 = rowptr(j + 3);
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const int col = (c * LPR + lr) * VEC;
        if (col < w) {
          T v0 = V::ld(p0 + col), v1 = V::ld(p1 + col), v2 = V::ld(p2 + col), v3 = V::ld(p3 + col);
          V::add(acc[c], v0);
          V::add(acc[c], v1);
          V::add(acc[c], v2);
          V::add(acc[c], v3);
        }
      }
    }
    for (; j < e; ++j) {
      const float* p0 = rowptr(j);
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const int col = (c * LPR + lr) * VEC;
        if (col < w) V::add(acc[c], V::ld(p0 + col));
      }
    }
    const float cnt = (float)(e - b);
    if (q < n_own) {
      float* out = a.sums + (int64_t)(own0 + q) * w;
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const int col = (c * LPR + lr) * VEC;
        if (col < w) V::st(out + col, acc[c]);
      }
      if (lr == 0) a.counts[own0 + q] = cnt;
    } else {
      const int slot = a.sendpos[a.pbase_l + ref0 + (q - n_own)];
      float* out = a.sendbuf + (int64_t)slot * a.stride;
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const int col = (c * LPR + lr) * VEC;
        if (col < w) {
          if ((a.stride & 3) == 0) V::st(out + col, acc[c]); else V::st_any(out + col, acc[c]);
        }
      }
      if (lr == 0) out[w] = cnt;
    }
  }
}

template <int VEC, int LPR, int NCH>
int launch_agg(const SgMeta* meta, const AggArgs& a, int64_t max_rows, cudaStream_t st) {
  constexpr int RPB = 8 * (32 / LPR);  // rows per 256-thread block
  const int grid = clamp_grid(div_up(max_rows, RPB), kSMs * 16);
  k_sage_agg<VEC, LPR, NCH><<<grid, 256, 0, st>>>(meta, a);
  SG_CHECK_LAUNCH("k_sage_agg");
  return SG_OK;
}

// dispatch on width: VEC=4 needs w%4==0 (16B aligned rows)
int dispatch_agg(const SgMeta* meta, const AggArgs& a, int64_t max_rows, cudaStream_t st) {
  const int w = a.w;
  if (w % 4 == 0) {
    if (w <= 16) return launch_agg<4, 4, 1>(meta, a, max_rows, st);
    if (w <= 32) return launch_agg<4, 8, 1>(meta, a, max_rows, st);
    if (w <= 64) return launch_agg<4, 16, 1>(meta, a, max_rows, st);
    if (w <= 128) return launch_agg<4, 32, 1>(meta, a, max_rows, st);
    if (w <= 256) return launch_agg<4, 32, 2>(meta, a, max_rows, st);
    if (w <= 512) return launch_agg<4, 32, 4>(meta, a, max_rows, st);
  } else {
    if (w <= 8) return launch_agg<1, 8, 1>(meta, a, max_rows, st);
    if (w <= 32) return launch_agg<1, 32, 1>(meta, a, max_rows, st);
    if (w <= 128) return launch_agg<1, 32, 4>(meta, a, max_rows, st);
    if (w <= 512) return launch_agg<1, 32, 16>(meta, a, max_rows, st);
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
};

__global__ void __launch_bounds__(256) k_sage_update(const SgMeta* __restrict__ meta, UpdArgs a) {
  extern __shared__ float smem[];
  const int w = a.w, dout = a.dout, wp = w + 1;
  float* ws_s = smem;                 // [w][dout]
  float* wn_s = ws_s + w * dout;      // [w][dout]
  float* hs_s = wn_s + w * dout;      // [UTR][w+1]
  float* mn_s = hs_s + UTR * wp;      // [UTR][w+1]
  for (int i = threadIdx.x; i < w * dout; i += blockDim.x) {
    ws_s[i] = a.ws[i];
    wn_s[i] = a.wn[i];
  }
  const int l = a.l, d = a.d, g = a.g;
  const int n_own = meta->n_own[l][d];
  const int own0 = meta->own_off[l][d], prev0 = meta->own_off[l - 1][d];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = (n_own + UTR - 1) / UTR;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    __syncthreads();
    for (int rr = warp; rr < UTR; rr += 8) {
      const int q = tile * UTR + rr;
      if (q >= n_own) continue;
      const int G = own0 + q;
      float N = a.counts[G];
      const int* cb = a.contrib + (int64_t)g * a.voff_l + (int64_t)G * g;
      int rs[SG_MAXG];
#pragma unroll
      for (int s = 0; s < SG_MAXG; ++s) rs[s] = s < g ? cb[s] : -1;
#pragma unroll
      for (int s = 0; s < SG_MAXG; ++s)
        if (rs[s] >= 0) N += a.recv[(int64_t)rs[s] * a.stride + w];
      int r = prev0 + a.selfrow[a.voff_l + G];
      if (a.src_row) r = a.src_row[r];
      const float* hrow = a.h_prev + (int64_t)r * w;
      for (int c = lane; c < w; c += 32) {
        float S = a.sums[(int64_t)G * w + c];
#pragma unroll
        for (int s = 0; s < SG_MAXG; ++s)
          if (rs[s] >= 0) S += a.recv[(int64_t)rs[s] * a.stride + c];
        const float m = S / N;
        mn_s[rr * wp + c] = m;
        a.mean[(int64_t)G * w + c] = m;
        hs_s[rr * wp + c] = __ldg(hrow + c);
      }
      if (lane == 0) a.counts[G] = N;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < UTR * dout; idx += blockDim.x) {
      const int rr = idx / dout, j = idx - rr * dout;
      const int q = tile * UTR + rr;
      if (q >= n_own) continue;
      const float* hr = hs_s + rr * wp;
      const float* mr = mn_s + rr * wp;
      float acc = a.bias[j];
      for (int c = 0; c < w; ++c) acc = fmaf(hr[c], ws_s[c * dout + j], fmaf(mr[c], wn_s[c * dout + j], acc));
      a.h[(int64_t)(own0 + q) * dout + j] = a.final_ ? acc : fmaxf(acc, 0.f);
    }
  }
}

// ---------------------------------------------------------------- backward rows
constexpr int BTR = 32;
constexpr int MAXACC = 16;  // per thread per weight matrix: w*dout <= 4096

struct BwdArgs {
  int l, d, w, dout, final_;
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
};

__global__ void __launch_bounds__(256) k_sage_bwd_rows(const SgMeta* __restrict__ meta, BwdArgs a) {
  extern __shared__ float smem[];
  const int w = a.w, dout = a.dout, wp = w + 1, dp1 = dout + 1;
  const bool need_c = a.d_self != nullptr || a.d_sums != nullptr;
  float* dp_s = smem;                       // [BTR][dout]
  float* hs_s = dp_s + BTR * dout;          // [BTR][w+1]
  float* mn_s = hs_s + BTR * wp;            // [BTR][w+1]
  float* ws_s = mn_s + BTR * wp;            // [w][dout+1] (only if need_c)
  float* wn_s = ws_s + w * dp1;
  float* inv_s = wn_s + w * dp1;            // [BTR]
  if (need_c) {
    for (int i = threadIdx.x; i < w * dout; i += blockDim.x) {
      const int c = i / dout, j = i - c * dout;
      ws_s[c * dp1 + j] = a.ws[i];
      wn_s[c * dp1 + j] = a.wn[i];
    }
  }
  const int l = a.l, d = a.d;
  const int n_own = meta->n_own[l][d];
  const int own0 = meta->own_off[l][d], prev0 = meta->own_off[l - 1][d];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwd = w * dout;
  float aS[MAXACC], aN[MAXACC], ab = 0.f;
#pragma unroll
  for (int k = 0; k < MAXACC; ++k) aS[k] = aN[k] = 0.f;
  const int ntiles = (n_own + BTR - 1) / BTR;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    __syncthreads();
    for (int rr = warp; rr < BTR; rr += 8) {
      const int q = tile * BTR + rr;
      const bool valid = q < n_own;
      const int G = own0 + q;
      for (int j = lane; j < dout; j += 32) {
        float v = 0.f;
        if (valid) {
          v = a.d_h[(int64_t)G * dout + j];
          if (!a.final_ && !(a.h[(int64_t)G * dout + j] > 0.f)) v = 0.f;
        }
        dp_s[rr * dout + j] = v;
      }
      if (valid) {
        int r = prev0 + a.selfrow[a.voff_l + G];
        if (a.src_row) r = a.src_row[r];
        const float* hrow = a.h_prev + (int64_t)r * w;
        const float* mrow = a.mean + (int64_t)G * w;
        for (int c = lane; c < w; c += 32) {
          hs_s[rr * wp + c] = __ldg(hrow + c);
          mn_s[rr * wp + c] = mrow[c];
        }
        if (lane == 0) inv_s[rr] = a.counts[G];
      } else {
        for (int c = lane; c < w; c += 32) hs_s[rr * wp + c] = mn_s[rr * wp + c] = 0.f;
        if (lane == 0) inv_s[rr] = 1.f;
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < MAXACC; ++k) {
      const int idx = threadIdx.x + 256 * k;
      if (idx < nwd) {
        const int c = idx / dout, j = idx - c * dout;
        float s1 = aS[k], s2 = aN[k];
        for (int rr = 0; rr < BTR; ++rr) {
          const float g = dp_s[rr * dout + j];
          s1 = fmaf(hs_s[rr * wp + c], g, s1);
          s2 = fmaf(mn_s[rr * wp + c], g, s2);
        }
        aS[k] = s1;
        aN[k] = s2;
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
        for (int j = 0; j < dout; ++j) {
          const float g = dp_s[rr * dout + j];
          s1 = fmaf(g, ws_s[c * dp1 + j], s1);
          s2 = fmaf(g, wn_s[c * dp1 + j], s2);
        }
        if (a.d_self) a.d_self[G * w + c] = s1;
        if (a.d_sums) a.d_sums[G * w + c] = s2 / inv_s[rr];
      }
    }
  }
  const int64_t ntot = 2 * (int64_t)nwd + dout;
  float* out = a.partial + (int64_t)blockIdx.x * ntot;
#pragma unroll
  for (int k = 0; k < MAXACC; ++k) {
    const int idx = threadIdx.x + 256 * k;
    if (idx < nwd) {
      out[idx] = aS[k];
      out[nwd + idx] = aN[k];
    }
  }
  if (threadIdx.x < dout) out[2 * nwd + threadIdx.x] = ab;
}

// ---------------------------------------------------------------- scatter (transpose SpMM)
struct ScatArgs {
  int l, d, w, stride;
  int64_t voff_lm1, voff_l, pbase_l, key_base;
  int64_t nV_l;
  const int32_t* grouped;
  const int32_t* rank;
  const int32_t* ldst;
  const int32_t* sendpos;
  const int32_t* perm;
  const int32_t* srcbeg;
  const int32_t* srcend;
  const float* d_self;
  const float* d_sums;
  const float* bwd_recv;
  float* d_prev;
};

template <int VEC, int LPR, int NCH>
__global__ void __launch_bounds__(256) k_sage_scatter(const SgMeta* __restrict__ meta, ScatArgs a) {
  using V = VecT<VEC>;
  using T = typename V::T;
  constexpr int RPW = 32 / LPR;
  const int l = a.l, d = a.d, w = a.w;
  const int n_prev = meta->n_own[l - 1][d];
  const int prev0 = meta->own_off[l - 1][d];
  const int own0 = meta->own_off[l][d], n_own = meta->n_own[l][d], ref0 = meta->ref_off[l][d];
  const int lane = threadIdx.x & 31;
  const int sub = lane / LPR, lr = lane % LPR;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = gw * RPW + sub; u < n_prev; u += nw * RPW) {
    const int64_t U = prev0 + u;
    T acc[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) acc[c] = V::zero();
    const int p = a.grouped[a.voff_lm1 + U];
    if (p < a.nV_l) {
      const int64_t v = own0 + a.rank[a.voff_l + p];
      const float* sr = a.d_self + v * w;
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const int col = (c * LPR + lr) * VEC;
        if (col < w) acc[c] = V::ld(sr + col);
      }
    }
    const int b = a.srcbeg[a.key_base + U], e = a.srcend[a.key_base + U];
    for (int j = b; j < e; ++j) {
      const int x = a.perm[j];
      const int q = a.ldst[x];
      const float* row;
      if (q < n_own) {
        row = a.d_sums + (int64_t)(own0 + q) * w;
      } else {
        const int slot = a.sendpos[a.pbase_l + ref0 + (q - n_own)];
        row = a.bwd_recv + (int64_t)slot * a.stride;
      }
      const bool vec_ok = q < n_own || (a.stride & 3) == 0;
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const int col = (c * LPR + lr) * VEC;
        if (col < w) {
          if (vec_ok) {
            V::add(acc[c], V::ld(row + col));
          } else {
            T t;
            float* tp = reinterpret_cast<float*>(&t);
#pragma unroll
            for (int v = 0; v < VEC; ++v) tp[v] = row[col + v];
            V::add(acc[c], t);
          }
        }
      }
    }
    float* out = a.d_prev + U * w;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const int col = (c * LPR + lr) * VEC;
      if (col < w) V::st(out + col, acc[c]);
    }
  }
}

template <int VEC, int LPR, int NCH>
int launch_scat(const SgMeta* meta, const ScatArgs& a, int64_t max_rows, cudaStream_t st) {
  constexpr int RPB = 8 * (32 / LPR);
  const int grid = clamp_grid(div_up(max_rows, RPB), kSMs * 16);
  k_sage_scatter<VEC, LPR, NCH><<<grid, 256, 0, st>>>(meta, a);
  SG_CHECK_LAUNCH("k_sage_scatter");
  return SG_OK;
}

int dispatch_scat(const SgMeta* meta, const ScatArgs& a, int64_t max_rows, cudaStream_t st) {
  const int w = a.w;
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

extern "C" int sg_sage_agg_fwd(const void* split_ws, const SgSplitLayout* lay, int32_t l,
                               int32_t d, const float* h_prev, const int32_t* src_row, int32_t w,
                               float* sums, float* counts, float* sendbuf, int32_t send_stride,
                               int64_t max_rows, void* stream) {
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
  a.dperm = nullptr;
  a.sendpos = I32(y.o_sendpos);
  a.src_row = src_row;
  a.h_prev = h_prev;
  a.sums = sums;
  a.counts = counts;
  a.sendbuf = sendbuf;
  return dispatch_agg(meta, a, max_rows, (cudaStream_t)stream);
}

extern "C" int sg_sage_agg_fwd_perm(const void* split_ws, const SgSplitLayout* lay, int32_t l,
                                    int32_t d, const float* h_prev, const int32_t* src_row,
                                    int32_t w, float* sums, float* counts, float* sendbuf,
                                    int32_t send_stride, const int32_t* dperm, int64_t max_rows,
                                    void* stream) {
  SG_REQUIRE(split_ws && lay, "sage_agg_fwd: null workspace");
  SPLIT_PTRS
  SG_REQUIRE(l >= 1 && l <= y.L && d >= 0 && d < y.g, "sage_agg_fwd: bad layer/device");
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
  a.sums = sums;
  a.counts = counts;
  a.sendbuf = sendbuf;
  return dispatch_agg(meta, a, max_rows, (cudaStream_t)stream);
}

extern "C" int sg_sage_update(const void* split_ws, const SgSplitLayout* lay, int32_t l,
                              int32_t d, const float* h_prev, const int32_t* src_row, int32_t w,
                              int32_t dout, const float* sums, float* counts,
                              const float* recvbuf, int32_t recv_stride, const float* w_self,
                              const float* w_neigh, const float* bias, int32_t final_layer,
                              float* mean, float* h, int64_t max_rows, void* stream) {
  SG_REQUIRE(split_ws && lay, "sage_update: null workspace");
  SPLIT_PTRS
  SG_REQUIRE(l >= 1 && l <= y.L && d >= 0 && d < y.g, "sage_update: bad layer/device");
  SG_REQUIRE(dout >= 1 && dout <= 256, "sage_update: dout out of range");
  if (max_rows <= 0) return SG_OK;
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
  const size_t smem = sizeof(float) * (2 * (size_t)w * dout + 2 * (size_t)UTR * (w + 1));
  SG_REQUIRE(smem <= 227 * 1024, "sage_update: width too large for shared memory");
  cudaStream_t st = (cudaStream_t)stream;
  if (smem > 48 * 1024)
    SG_CUDA(cudaFuncSetAttribute(k_sage_update, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
  const int grid = clamp_grid(div_up(max_rows, UTR), kSMs * 4);
  k_sage_update<<<grid, 256, smem, st>>>(meta, a);
  SG_CHECK_LAUNCH("k_sage_update");
  return SG_OK;
}

extern "C" int sg_sage_bwd_rows(const void* split_ws, const SgSplitLayout* lay, int32_t l,
                                int32_t d, const float* h_prev, const int32_t* src_row, int32_t w,
                                int32_t dout, const float* d_h, const float* h,
                                int32_t final_layer, const float* mean, const float* counts,
                                const float* w_self, const float* w_neigh, float* partial,
                                int32_t nblocks, float* d_self, float* d_sums, int64_t max_rows,
                                void* stream) {
  SG_REQUIRE(split_ws && lay, "sage_bwd_rows: null workspace");
  SPLIT_PTRS
  SG_REQUIRE(l >= 1 && l <= y.L && d >= 0 && d < y.g, "sage_bwd_rows: bad layer/device");
  SG_REQUIRE(dout >= 1 && dout <= 32, "sage_bwd_rows: dout must be <= 32");
  SG_REQUIRE((int64_t)w * dout <= 256 * MAXACC, "sage_bwd_rows: w*dout > 4096 unsupported");
  SG_REQUIRE(nblocks >= 1, "sage_bwd_rows: nblocks >= 1");
  (void)max_rows;
  BwdArgs a;
  memset(&a, 0, sizeof(a));
  a.l = l;
  a.d = d;
  a.w = w;
  a.dout = dout;
  a.final_ = final_layer;
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
  const size_t smem =
      sizeof(float) * ((size_t)BTR * dout + 2 * (size_t)BTR * (w + 1) + 2 * (size_t)w * (dout + 1) + BTR);
  SG_REQUIRE(smem <= 227 * 1024, "sage_bwd_rows: width too large for shared memory");
  cudaStream_t st = (cudaStream_t)stream;
  if (smem > 48 * 1024)
    SG_CUDA(cudaFuncSetAttribute(k_sage_bwd_rows, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
  k_sage_bwd_rows<<<nblocks, 256, smem, st>>>(meta, a);
  SG_CHECK_LAUNCH("k_sage_bwd_rows");
  return SG_OK;
}

extern "C" int sg_sage_scatter_bwd(const void* split_ws, const SgSplitLayout* lay, int32_t l,
                                   int32_t d, int32_t w, const float* d_self, const float* d_sums,
                                   const float* bwd_recv, int32_t recv_stride,
                                   const int32_t* perm, const int32_t* srcbeg,
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
  a.pbase_l = y.pbase[l];
  a.key_base = key_base;
  a.nV_l = y.nV[l];
  a.grouped = I32(y.o_grouped);
  a.rank = I32(y.o_rank);
  a.ldst = I32(y.o_ldst);
  a.sendpos = I32(y.o_sendpos);
  a.perm = perm;
  a.srcbeg = srcbeg;
  a.srcend = srcend;
  a.d_self = d_self;
  a.d_sums = d_sums;
  a.bwd_recv = bwd_recv;
  a.d_prev = d_prev;
  return dispatch_scat(meta, a, max_rows, (cudaStream_t)stream);
}

}  // namespace sg
