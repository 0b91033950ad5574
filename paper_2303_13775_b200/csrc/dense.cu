// Generic register-tiled FP32 GEMMs for layer widths outside the fused
// fast paths (sage.cu / gat.cu handle the common shapes: SAGE hidden <= 32,
// GAT D <= 128). The reference accepts any hidden size (config.py:91-92);
// these kernels make every SAGE / GAT layer and the classifier work for any
// width, with the same fixed-order (deterministic) reductions:
//
//   gemm_rows        C[r, n]  = epi( sum_k A(r, k) B(k, n) )
//                    A rows gathered (identity / index map / SAGE self row),
//                    optionally masked by ReLU'(h); B row-major [K x N] or
//                    transposed [N x K]; epilogue: accumulate, per-row
//                    1/count scale, bias, ReLU.
//   gemm_tn_partial  P[s][k, n] = sum_{r in split s} A(r, k) G(r, n)
//                    per-split partials of a weight gradient (fixed row
//                    order), optional virtual ones-column (bias gradient),
//                    summed later by sg_reduce_partials in split order.
//
// 64 x 64 output tile per block, 256 threads with 4 x 4 register tiles,
// K staged 16 at a time through shared memory (transposed for broadcast).
#include <cstddef>
#include <cstring>

#include "dense.cuh"

namespace sg {

namespace {

constexpr int GM = 64, GN = 64, GK = 16, GP = 4;

__device__ __forceinline__ int64_t dense_row(const DenseRows& d, int64_t base, int64_t prev0, int64_t r) {
  const int64_t i = base + d.add + r;
  if (d.mode == 0) return i;
  if (d.mode == 1) return d.map[i];
  int64_t p = prev0 + d.selfrow[d.voff_l + i];
  if (d.map) p = d.map[p];
  return p;
}

__device__ __forceinline__ int64_t dev_or0(const int32_t* p) { return p ? (int64_t)*p : 0; }

__global__ void __launch_bounds__(256) k_gemm_rows(GemmArgs a) {
  SG_PDL_ENTRY();
  __shared__ __align__(16) float As[GK][GM + GP];
  __shared__ __align__(16) float Bs[GK][GN + GP];
  __shared__ int64_t arow[GM];
  const int R = *a.R_dev;
  const int64_t abase = dev_or0(a.ar.base_dev), aprev = dev_or0(a.ar.prev0_dev);
  const int64_t cbase = dev_or0(a.c_base_dev);
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const int n0 = blockIdx.y * GN;
  for (int m0 = blockIdx.x * GM; m0 < R; m0 += gridDim.x * GM) {
    __syncthreads();
    if (tid < GM) arow[tid] = m0 + tid < R ? dense_row(a.ar, abase, aprev, m0 + tid) : -1;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
    for (int k0 = 0; k0 < a.K; k0 += GK) {
      __syncthreads();
      // A tile: 64 rows x 16 k, 4 elements per thread (k fastest -> coalesced)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int idx = tid + 256 * u, rr = idx >> 4, kk = idx & 15;
        const int64_t pr = arow[rr];
        const int k = k0 + kk;
        float v = 0.f;
        if (pr >= 0 && k < a.K) {
          v = a.A[pr * a.lda + k];
          if (a.amask && !(a.amask[(cbase + m0 + rr) * a.lda_mask + k] > 0.f)) v = 0.f;
        }
        As[kk][rr] = v;
      }
      // B tile: 16 k x 64 n
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int idx = tid + 256 * u;
        int kk, nn;
        if (a.bt) {
          kk = idx & 15;
          nn = idx >> 4;
        } else {
          kk = idx >> 6;
          nn = idx & 63;
        }
        const int k = k0 + kk, n = n0 + nn;
        float v = 0.f;
        if (k < a.K && n < a.N) v = a.bt ? a.B[(int64_t)n * a.ldb + k] : a.B[(int64_t)k * a.ldb + n];
        Bs[kk][nn] = v;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < GK; ++kk) {
        const float4 av = *reinterpret_cast<const float4*>(&As[kk][4 * ty]);
        const float4 bv = *reinterpret_cast<const float4*>(&Bs[kk][4 * tx]);
        const float ar[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          acc[i][0] = fmaf(ar[i], bv.x, acc[i][0]);
          acc[i][1] = fmaf(ar[i], bv.y, acc[i][1]);
          acc[i][2] = fmaf(ar[i], bv.z, acc[i][2]);
          acc[i][3] = fmaf(ar[i], bv.w, acc[i][3]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = m0 + 4 * ty + i;
      if (r >= R) continue;
      const int64_t cr = cbase + r;
      const float sc = a.rdiv ? 1.f / a.rdiv[cr] : 1.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int n = n0 + 4 * tx + j;
        if (n >= a.N) continue;
        float v = acc[i][j] * sc;
        float* cp = a.C + cr * a.ldc + n;
        if (a.accum) v += *cp;
        if (a.bias) v += a.bias[n];
        if (a.relu) v = sg_relu(v);
        *cp = v;
      }
    }
  }
}


// P[s][p_off + k * N + n] over split s's rows (ascending); grid (tiles, nsplit)
__global__ void __launch_bounds__(256) k_gemm_tn_partial(TnArgs a) {
  SG_PDL_ENTRY();
  constexpr int GR = 16;
  __shared__ __align__(16) float As[GR][GM + GP];
  __shared__ __align__(16) float Gs[GR][GN + GP];
  __shared__ int64_t arow[GR];
  const int R = *a.R_dev;
  const int64_t abase = dev_or0(a.ar.base_dev), aprev = dev_or0(a.ar.prev0_dev);
  const int64_t gbase = dev_or0(a.g_base_dev);
  const int Ke = a.K + (a.ones ? 1 : 0);
  const int tiles_n = (a.N + GN - 1) / GN;
  const int k0 = (blockIdx.x / tiles_n) * GM, n0 = (blockIdx.x % tiles_n) * GN;
  const int s = blockIdx.y;
  const int per = (R + a.nsplit - 1) / a.nsplit;
  const int rb = s * per, re = min(R, rb + per);
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
  for (int r0 = rb; r0 < re; r0 += GR) {
    __syncthreads();
    if (tid < GR) arow[tid] = r0 + tid < re ? dense_row(a.ar, abase, aprev, r0 + tid) : -1;
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int idx = tid + 256 * u, rr = idx >> 6, kk = idx & 63;
      const int64_t pr = arow[rr];
      const int k = k0 + kk;
      float v = 0.f;
      if (pr >= 0 && k < Ke) v = k < a.K ? a.A[pr * a.lda + k] : 1.f;
      As[rr][kk] = v;
      const int n = n0 + kk;
      float gv = 0.f;
      if (r0 + rr < re && n < a.N) {
        const int64_t gr = (gbase + r0 + rr) * a.ldg + n;
        gv = a.G[gr];
        if (a.gmask && !(a.gmask[gr] > 0.f)) gv = 0.f;
      }
      Gs[rr][kk] = gv;
    }
    __syncthreads();
#pragma unroll
    for (int rr = 0; rr < GR; ++rr) {
      const float4 av = *reinterpret_cast<const float4*>(&As[rr][4 * ty]);
      const float4 gv = *reinterpret_cast<const float4*>(&Gs[rr][4 * tx]);
      const float ar[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc[i][0] = fmaf(ar[i], gv.x, acc[i][0]);
        acc[i][1] = fmaf(ar[i], gv.y, acc[i][1]);
        acc[i][2] = fmaf(ar[i], gv.z, acc[i][2]);
        acc[i][3] = fmaf(ar[i], gv.w, acc[i][3]);
      }
    }
  }
  float* out = a.P + (int64_t)s * a.pstride + a.p_off;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = k0 + 4 * ty + i;
    if (k >= Ke) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + 4 * tx + j;
      if (n < a.N) out[(int64_t)k * a.N + n] = acc[i][j];
    }
  }
}

}  // namespace

int dense_gemm_rows(const GemmArgs& a, int64_t max_rows, cudaStream_t st) {
  if (max_rows <= 0 || a.N <= 0) return SG_OK;
  SG_REQUIRE(a.K >= 0 && a.A && a.B && a.C && a.R_dev, "gemm_rows: bad arguments");
  const int gx = clamp_grid(div_up(max_rows, GM), kSMs * 4);
  dim3 grid(gx, (unsigned)div_up(a.N, GN));
  ::sg::launch(k_gemm_rows, grid, 256, 0, st, a);
  SG_CHECK_LAUNCH("k_gemm_rows");
  return SG_OK;
}

int dense_gemm_tn_partial(const TnArgs& a, cudaStream_t st) {
  SG_REQUIRE(a.nsplit >= 1 && a.A && a.G && a.P && a.R_dev, "gemm_tn_partial: bad arguments");
  const int Ke = a.K + (a.ones ? 1 : 0);
  if (Ke <= 0 || a.N <= 0) return SG_OK;
  dim3 grid((unsigned)(div_up(Ke, GM) * div_up(a.N, GN)), (unsigned)a.nsplit);
  ::sg::launch(k_gemm_tn_partial, grid, 256, 0, st, a);
  SG_CHECK_LAUNCH("k_gemm_tn_partial");
  return SG_OK;
}

}  // namespace sg
