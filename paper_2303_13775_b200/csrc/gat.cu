// GAT forward/backward for one device of a split — replaces _gat_forward /
// _gat_backward (engine.py:280-552) and the layer math of models.py:217-261.
// H heads are computed together (H = 1 is the reference's single-head layer;
// H > 1 is the concatenation of H single-head layers on the same input,
// SURVEY §8(a) row 11): z = h W with W = [W_1 | ... | W_H], per-head scores,
// per-head softmax, outputs concatenated, input gradients summed.
//
// The reference runs 10 barrier exchange rounds per layer (test_engine.py:
// 376-384). Here they are 5, with identical mathematics:
//   forward   from_owner t (w H)              t_v = z_v.a_dst per head
//             to_owner (U, m, s) (w D+2H)      ONLINE-SOFTMAX partials: local max
//                                              m, s = sum e^(e-m), U = sum e^(e-m) z_u;
//                                              the owner merges with rescaling
//             from_owner (m, den) (w 2H)       global stabiliser + denominator, so
//                                              every holder materialises alpha
//   backward  from_owner (d_num, c) (w D+H)    c_v = d_num_v . num_v per head; the
//                                              softmax backward identity
//                                              d_e = alpha_e (d_num_v.z_u - c_v)
//                                              replaces the dd to/from rounds
//             to_owner dt (w H)
//   (SURVEY §7 hard part 5; verified there to 1e-15 in float64.)
// Per-edge arrays hold H values per edge ([edge][head]); per-row scalars H
// values per row ([row][head]); D = H * d_head.
#include <cstring>
#include <type_traits>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "dense.cuh"

namespace sg {
namespace {

__device__ __forceinline__ float leaky(float x, float slope) { return x > 0.f ? x : slope * x; }

template <int VEC>
struct V4;
template <>
struct V4<4> {
  using T = float4;
  __device__ static T zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
  __device__ static T ld(const float* p) { return *reinterpret_cast<const float4*>(p); }
  __device__ static T ld_any(const float* p) { return make_float4(p[0], p[1], p[2], p[3]); }
  __device__ static void st(float* p, T v) { *reinterpret_cast<float4*>(p) = v; }
  __device__ static void st_any(float* p, T v) { p[0] = v.x; p[1] = v.y; p[2] = v.z; p[3] = v.w; }
  __device__ static T axpby(float a, T x, float b, T y) {
    return make_float4(fmaf(a, x.x, b * y.x), fmaf(a, x.y, b * y.y), fmaf(a, x.z, b * y.z), fmaf(a, x.w, b * y.w));
  }
  __device__ static void fma_(T& acc, float a, T x) {
    acc.x = fmaf(a, x.x, acc.x); acc.y = fmaf(a, x.y, acc.y); acc.z = fmaf(a, x.z, acc.z); acc.w = fmaf(a, x.w, acc.w);
  }
  __device__ static float dot(T x, T y) { return fmaf(x.x, y.x, fmaf(x.y, y.y, fmaf(x.z, y.z, x.w * y.w))); }
  __device__ static T shfl_xor(unsigned m, T v, int o, int w) {
    return make_float4(__shfl_xor_sync(m, v.x, o, w), __shfl_xor_sync(m, v.y, o, w),
                       __shfl_xor_sync(m, v.z, o, w), __shfl_xor_sync(m, v.w, o, w));
  }
  __device__ static void add(T& a, T b) { a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w; }
  __device__ static T div(T x, float s) { return make_float4(x.x / s, x.y / s, x.z / s, x.w / s); }
  __device__ static T relu(T x) { return make_float4(sg_relu(x.x), sg_relu(x.y), sg_relu(x.z), sg_relu(x.w)); }
};
template <>
struct V4<1> {
  using T = float;
  __device__ static T zero() { return 0.f; }
  __device__ static T ld(const float* p) { return *p; }
  __device__ static T ld_any(const float* p) { return *p; }
  __device__ static void st(float* p, T v) { *p = v; }
  __device__ static void st_any(float* p, T v) { *p = v; }
  __device__ static T axpby(float a, T x, float b, T y) { return fmaf(a, x, b * y); }
  __device__ static void fma_(T& acc, float a, T x) { acc = fmaf(a, x, acc); }
  __device__ static float dot(T x, T y) { return x * y; }
  __device__ static T shfl_xor(unsigned m, T v, int o, int w) { return __shfl_xor_sync(m, v, o, w); }
  __device__ static void add(T& a, T b) { a += b; }
  __device__ static T div(T x, float s) { return x / s; }
  __device__ static T relu(T x) { return sg_relu(x); }
};

// ---------------------------------------------------------------- projection
constexpr int PTR = 32;

struct ProjArgs {
  int l, d, w, dout, heads;
  int64_t voff_lm1, voff_l;
  const float* h_prev;
  const int32_t* src_row;
  const int32_t* grouped;
  const int32_t* rank;
  const float* W;
  const float* a_src;
  const float* a_dst;
  float* z;
  float* s;  // [row][head]
  float* t;  // [owned row at l][head]
};

template <bool Q4>
__global__ void __launch_bounds__(256) k_gat_project(const SgMeta* __restrict__ meta, ProjArgs a) {
  SG_PDL_ENTRY();
  extern __shared__ __align__(16) float smem[];
  const int w = a.w, dout = a.dout, wp = w + 1, dp = dout + 1, H = a.heads, dh = dout / H;
  float* W_s = smem;               // [w][dout]
  float* h_s = W_s + w * dout;     // [PTR][w+1]
  float* z_s = h_s + PTR * wp;     // [PTR][dout+1]
  int* prow_s = (int*)(z_s + PTR * dp);
  for (int i = threadIdx.x; i < w * dout; i += blockDim.x) W_s[i] = a.W[i];
  const int l = a.l, d = a.d;
  const int n = meta->n_own[l - 1][d];
  const int own0 = meta->own_off[l - 1][d];
  const int ownl = meta->own_off[l][d];
  const int64_t nVl = meta->nV[l];
  const int ntiles = (n + PTR - 1) / PTR;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    __syncthreads();
    if (threadIdx.x < PTR) {
      const int q = tile * PTR + threadIdx.x;
      int r = -1;
      if (q < n) {
        r = own0 + q;
        if (a.src_row) r = a.src_row[r];
      }
      prow_s[threadIdx.x] = r;
    }
    __syncthreads();
    const int nrow = min(PTR, n - tile * PTR);
#pragma unroll 4
    for (int idx = threadIdx.x; idx < nrow * w; idx += blockDim.x) {
      const int rr = idx / w, c = idx - rr * w;
      h_s[rr * wp + c] = __ldg(a.h_prev + (int64_t)prow_s[rr] * w + c);
    }
    __syncthreads();
    if (Q4) {
      const int nq = dout >> 2;
      for (int idx = threadIdx.x; idx < nrow * nq; idx += blockDim.x) {
        const int rr = idx / nq, jq = idx - rr * nq;
        const float* hr = h_s + rr * wp;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
        for (int c = 0; c < w; ++c) {
          const float hv = hr[c];
          const float4 w4 = *reinterpret_cast<const float4*>(W_s + c * dout + 4 * jq);
          acc.x = fmaf(hv, w4.x, acc.x);
          acc.y = fmaf(hv, w4.y, acc.y);
          acc.z = fmaf(hv, w4.z, acc.z);
          acc.w = fmaf(hv, w4.w, acc.w);
        }
        *reinterpret_cast<float4*>(a.z + (int64_t)(own0 + tile * PTR + rr) * dout + 4 * jq) = acc;
        float* zr = z_s + rr * dp + 4 * jq;
        zr[0] = acc.x;
        zr[1] = acc.y;
        zr[2] = acc.z;
        zr[3] = acc.w;
      }
    } else {
      for (int idx = threadIdx.x; idx < nrow * dout; idx += blockDim.x) {
        const int rr = idx / dout, j = idx - rr * dout;
        const float* hr = h_s + rr * wp;
        float acc = 0.f;
        for (int c = 0; c < w; ++c) acc = fmaf(hr[c], W_s[c * dout + j], acc);
        a.z[(int64_t)(own0 + tile * PTR + rr) * dout + j] = acc;
        z_s[rr * dp + j] = acc;
      }
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < nrow * H; idx += blockDim.x) {
      const int rr = idx / H, hh = idx - rr * H;
      const int G = own0 + tile * PTR + rr;
      const float* zr = z_s + rr * dp + hh * dh;
      float sv = 0.f;
      for (int j = 0; j < dh; ++j) sv = fmaf(zr[j], a.a_src[hh * dh + j], sv);
      a.s[(int64_t)G * H + hh] = sv;
      const int p = a.grouped[a.voff_lm1 + G];
      if (p < nVl) {  // self row of owned v at layer l
        float tv = 0.f;
        for (int j = 0; j < dh; ++j) tv = fmaf(zr[j], a.a_dst[hh * dh + j], tv);
        a.t[(int64_t)(ownl + a.rank[a.voff_l + p]) * H + hh] = tv;
      }
    }
  }
}

// ---------------------------------------------------------------- tensor-core projection
// z = h W on the tensor pipe with FP32-level accuracy: 3xTF32 (x = hi + lo,
// split_tf32; x*y ~= lo*hi + hi*lo + hi*hi, the dropped lo*lo term is
// ~2^-20 relative) on warp-level mma.sync m16n8k8 (HMMA), FP32
// accumulation. A 32-row tile of gathered rows sits row-major in smem
// (pitch K+4: conflict-free fragment loads), W in FP32 (pitch D+8), both
// split into hi/lo as the fragments are loaded. Warp (mb, cg): rows 16mb..16mb+15, columns cg*D/4 ...
// Then the per-head scores exactly as the FFMA kernel.
// x = hi + lo, both exactly TF32: hi = x rounded to TF32 (add half a TF32 ulp
// to the magnitude, clear the low 13 mantissa bits), lo = (x - hi) (exact in
// FP32, |lo| <= 2^-11 |x|) rounded to TF32 the same way; the dropped part is
// <= 2^-11 |lo| <= 2^-22 |x| with no systematic sign. Four integer/FP
// instructions instead of two multi-instruction cvt.rna.tf32 sequences
// (sm_100a has no single-op form). Passing lo unrounded (the tensor pipe then
// drops its low bits) doubled the roundoff seen in gradients that cancel to
// zero analytically.
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
  hi = (__float_as_uint(x) + 0x1000u) & 0xffffe000u;
  lo = (__float_as_uint(x - __uint_as_float(hi)) + 0x1000u) & 0xffffe000u;
}
__device__ __forceinline__ void mma_tf32(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void cp_async16g(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

template <int NT8>  // n8 tiles per warp: D = 32 * NT8
__global__ void __launch_bounds__(256) k_gat_project_mma(const SgMeta* __restrict__ meta, ProjArgs a) {
  SG_PDL_ENTRY();
  constexpr int TM = 32;
  constexpr int D = 32 * NT8, DP = D + 8;
  extern __shared__ __align__(16) float smem[];
  const int w = a.w, H = a.heads, dh = D / H;
  const int KPAD = (w + 7) & ~7, KP = KPAD + 4;
  float* W_s = smem;                   // [KPAD][DP] fp32 (hi/lo split at use)
  float* A_s = W_s + KPAD * DP;        // [2][TM][KP] double-buffered gathered rows
  float* red = A_s + 2 * TM * KP;      // [TM][D]
  int* prow = reinterpret_cast<int*>(red + TM * D);  // [2][TM]
  for (int i = threadIdx.x; i < KPAD * D; i += 256) {
    const int k = i / D, jj = i - k * D;
    W_s[k * DP + jj] = k < w ? a.W[k * D + jj] : 0.f;
  }
  for (int i = threadIdx.x; i < 2 * TM * (KP - w); i += 256) {  // K padding columns stay zero
    const int r = i / (KP - w), c = w + (i - r * (KP - w));
    A_s[r * KP + c] = 0.f;
  }
  const int l = a.l, d = a.d;
  const int n = meta->n_own[l - 1][d];
  const int own0 = meta->own_off[l - 1][d];
  const int ownl = meta->own_off[l][d];
  const int64_t nVl = meta->nV[l];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int mb = warp >> 2, cg = warp & 3;
  const int w4 = w / 4;
  const int G = gridDim.x;
  auto src_of = [&](int tile) {  // gathered row of this thread's tile row (threads < TM)
    const int r = tile * TM + (int)threadIdx.x;
    if (r >= n) return -1;
    const int pr = own0 + r;
    return a.src_row ? a.src_row[pr] : pr;
  };
  auto issue = [&](int tile, int buf) {
    float* Ab = A_s + buf * TM * KP;
    const int* pb = prow + buf * TM;
    for (int idx = threadIdx.x; idx < TM * w4; idx += 256) {
      const int r = idx / w4, q = idx - r * w4;
      if (pb[r] >= 0 && tile * TM < n) cp_async16g(Ab + r * KP + 4 * q, a.h_prev + (int64_t)pb[r] * w + 4 * q);
      else *reinterpret_cast<float4*>(Ab + r * KP + 4 * q) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int tile = blockIdx.x;
  if (threadIdx.x < TM) prow[threadIdx.x] = src_of(tile);
  int pnext = (threadIdx.x < TM) ? src_of(tile + G) : -1;
  __syncthreads();
  issue(tile, 0);
  for (int k = 0; tile < (n + TM - 1) / TM; ++k, tile += G) {
    const int buf = k & 1;
    if (threadIdx.x < TM) prow[(buf ^ 1) * TM + threadIdx.x] = pnext;
    __syncthreads();  // prow of the next tile visible; A_s[buf ^ 1] free
    issue(tile + G, buf ^ 1);
    if (threadIdx.x < TM) pnext = src_of(tile + 2 * G);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    const int r0 = tile * TM;
    float acc[NT8][4];
#pragma unroll
    for (int jj = 0; jj < NT8; ++jj) acc[jj][0] = acc[jj][1] = acc[jj][2] = acc[jj][3] = 0.f;
    const float* Ar = A_s + buf * TM * KP + (16 * mb + g) * KP;
    for (int k0 = 0; k0 < KPAD; k0 += 8) {
      const float x[4] = {Ar[k0 + t], Ar[8 * KP + k0 + t], Ar[k0 + t + 4], Ar[8 * KP + k0 + t + 4]};
      uint32_t ah[4], al[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        split_tf32(x[u], ah[u], al[u]);
      }
#pragma unroll
      for (int jj = 0; jj < NT8; ++jj) {
        const int n0 = cg * (D / 4) + 8 * jj;
        const float w0 = W_s[(k0 + t) * DP + n0 + g], w1 = W_s[(k0 + t + 4) * DP + n0 + g];
        uint32_t bh0, bh1, bl0, bl1;
        split_tf32(w0, bh0, bl0);
        split_tf32(w1, bh1, bl1);
        mma_tf32(acc[jj], al, bh0, bh1);
        mma_tf32(acc[jj], ah, bl0, bl1);
        mma_tf32(acc[jj], ah, bh0, bh1);
      }
    }
#pragma unroll
    for (int jj = 0; jj < NT8; ++jj) {
      const int n0 = cg * (D / 4) + 8 * jj;
      const int ra = 16 * mb + g;
      red[ra * D + n0 + 2 * t] = acc[jj][0];
      red[ra * D + n0 + 2 * t + 1] = acc[jj][1];
      red[(ra + 8) * D + n0 + 2 * t] = acc[jj][2];
      red[(ra + 8) * D + n0 + 2 * t + 1] = acc[jj][3];
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < TM * D / 4; idx += 256) {
      const int r = idx / (D / 4), q = idx - r * (D / 4);
      if (r0 + r < n)
        reinterpret_cast<float4*>(a.z + (int64_t)(own0 + r0 + r) * D)[q] = reinterpret_cast<const float4*>(red + r * D)[q];
    }
    // scores s = z.a_src per head; t = z.a_dst on self rows
    for (int idx = threadIdx.x; idx < TM * H; idx += 256) {
      const int r = idx / H, hh = idx - r * H;
      if (r0 + r >= n) continue;
      const int G2 = own0 + r0 + r;
      const float* zr = red + r * D + hh * dh;
      float sv = 0.f;
      for (int jj = 0; jj < dh; ++jj) sv = fmaf(zr[jj], a.a_src[hh * dh + jj], sv);
      a.s[(int64_t)G2 * H + hh] = sv;
      const int p = a.grouped[a.voff_lm1 + G2];
      if (p < nVl) {
        float tv = 0.f;
        for (int jj = 0; jj < dh; ++jj) tv = fmaf(zr[jj], a.a_dst[hh * dh + jj], tv);
        a.t[(int64_t)(ownl + a.rank[a.voff_l + p]) * H + hh] = tv;
      }
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// ---------------------------------------------------------------- tcgen05 projection
// z = h W on the 5th-generation tensor cores (tcgen05.mma kind::tf32, FP32
// accumulator in TMEM), 3xTF32 for FP32-level accuracy: per k-step of 8 the
// elected thread issues lo(A) hi(B) + hi(A) lo(B) + hi(A) hi(B) into the same
// accumulator. Tile = 128 gathered rows x D = 64 outputs x K = w (<= 104,
// padded to 8). Operands sit in shared memory in the canonical K-major
// SWIZZLE_NONE layout: 16-byte chunk c of row m at c * LBO + (m / 8) * 128 +
// (m % 8) * 16 (core matrices of 8 rows x 16 B, SBO = 128 B, LBO = rows * 16 B).
// Pipeline per tile: the next tile's rows are gathered by the bulk-copy engine
// (one cp.async.bulk per 4w-byte row into a row-major raw buffer, completion
// counted in bytes on an mbarrier: the LSU stays free for the epilogue) while
// this tile's MMAs run and its epilogue drains TMEM; the raw tile is then split
// into the canonical hi (x rounded to TF32) and lo = x - hi planes.
// Epilogue: warp w reads TMEM lanes 32 (w % 4).. (rows) and columns
// 32 (w / 4).. (tcgen05.ld 32x32b.x32), writes z and the per-head scores.
namespace tc5 {
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
constexpr int M = 128, N = 64, KMAX = 104, CH = KMAX / 4;  // 26 chunks of 16 B
constexpr int A_BYTES = CH * M * 16, B_BYTES = CH * N * 16;
constexpr int LBO_A = M * 16, LBO_B = N * 16, SBO = 128;
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
constexpr size_t SMEM = 3 * (size_t)A_BYTES + 2 * (size_t)B_BYTES + 2 * 64 * 4 + M * 4 + 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(SBO >> 4) << 32) |
         (1ull << 46);  // version 1 (sm_100), base offset 0, SWIZZLE_NONE
}
__device__ __forceinline__ void mma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(IDESC), "r"(acc));
}
}  // namespace tc5

template <int DH>  // head width (divides 32: a thread's 32 accumulator columns hold whole heads)
__global__ void __launch_bounds__(256, 1) k_gat_project_tc(const SgMeta* __restrict__ meta, ProjArgs a) {
  using namespace tc5;
  // TMEM allocation, barrier init and the W hi/lo planes run before the PDL
  // wait: they read only parameters and the split's counts, which the
  // preceding kernel does not write
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* A_raw = smem_raw;
  unsigned char* A_hi = A_raw + A_BYTES;
  unsigned char* A_lo = A_hi + A_BYTES;
  unsigned char* B_hi = A_lo + A_BYTES;
  unsigned char* B_lo = B_hi + B_BYTES;
  float* av_s = reinterpret_cast<float*>(B_lo + B_BYTES);  // a_src[64] | a_dst[64]
  int* hrow_s = reinterpret_cast<int*>(av_s + 128);         // [M] gathered rows of the next tile
  uint64_t* mbar = reinterpret_cast<uint64_t*>(hrow_s + M);  // [0] MMA done, [1] gather landed
  uint32_t* tmem_s = reinterpret_cast<uint32_t*>(mbar + 2);
  const int w = a.w, H = N / DH, wc = w / 4;
  const int kc = ((w + 7) & ~7) / 4;  // 16-byte chunks per row incl. K padding (even)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int l = a.l, d = a.d;
  const int n = meta->n_own[l - 1][d];
  const int own0 = meta->own_off[l - 1][d];
  const int ownl = meta->own_off[l][d];
  const int64_t nVl = meta->nV[l];
  const int ntiles = (n + M - 1) / M;
  const int G = gridDim.x;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_s)), "n"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mbar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mbar + 1)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // B = W^T split into hi / lo planes (K padding zero), attention vectors, raw K padding
#pragma unroll 4
  for (int i = tid; i < (N / 4) * kc * 4; i += 256) {  // coalesced float4 reads of W rows
    const int k = i / (N / 4), nq = i - k * (N / 4);
    const float4 x = k < w ? *reinterpret_cast<const float4*>(a.W + k * N + 4 * nq) : make_float4(0.f, 0.f, 0.f, 0.f);
    const float xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int nn = 4 * nq + u;
      uint32_t hi, lo;
      split_tf32(xv[u], hi, lo);
      const int off = (k >> 2) * LBO_B + (nn >> 3) * SBO + (nn & 7) * 16 + (k & 3) * 4;
      *reinterpret_cast<uint32_t*>(B_hi + off) = hi;
      *reinterpret_cast<uint32_t*>(B_lo + off) = lo;
    }
  }
  for (int i = tid; i < N; i += 256) {
    av_s[i] = a.a_src[i];
    av_s[64 + i] = a.a_dst[i];
  }
  SG_PDL_ENTRY();
  auto hrow_of = [&](int tile, int m) {
    const int r = tile * M + m;
    if (tile >= ntiles || r >= n) return -1;
    return a.src_row ? a.src_row[own0 + r] : own0 + r;
  };
  const uint32_t rowbytes = 4u * (uint32_t)w;
  auto expect = [&](int tile) {  // tid 0: the bytes the tile's row copies will deliver
    if (tile >= ntiles) return;
    const uint32_t bytes = rowbytes * (uint32_t)min(M, n - tile * M);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar + 1)), "r"(bytes)
                 : "memory");
  };
  auto issue = [&](int tile) {  // thread m < M: one bulk copy of row m (hrow_s) into A_raw
    if (tile >= ntiles || tid >= M) return;
    unsigned char* dst = A_raw + tid * rowbytes;
    const int hr = hrow_s[tid];
    if (hr >= 0) {
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(dst)),
                   "l"(a.h_prev + (int64_t)hr * w), "r"(rowbytes), "r"(smem_u32(mbar + 1))
                   : "memory");
    } else {
      for (int c = 0; c < wc; ++c) reinterpret_cast<float4*>(dst)[c] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  auto wait_bar = [&](uint64_t* bar, uint32_t ph) {
    const uint32_t mb = smem_u32(bar);
    uint32_t done = 0;
    const uint64_t t0 = globaltimer_ns();
    while (!done) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
          : "=r"(done)
          : "r"(mb), "r"(ph)
          : "memory");
      if (!done && globaltimer_ns() - t0 > 2000000000ull) __trap();  // never hang the device on a lost arrival
    }
  };
  if (tid < M) hrow_s[tid] = hrow_of(blockIdx.x, tid);
  if (tid == 0) expect(blockIdx.x);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_s;
  issue(blockIdx.x);
  const int row = tid & (M - 1), ch = tid >> 7;  // epilogue: TMEM lane = row, columns 32 ch ..
  for (int k = 0, tile = blockIdx.x; tile < ntiles; ++k, tile += G) {
    const int r0 = tile * M;
    // this thread's epilogue row: its self-row target (grouped -> rank) resolved early
    const int gr = r0 + row < n ? a.grouped[a.voff_lm1 + own0 + r0 + row] : -1;
    wait_bar(mbar + 1, k & 1);  // the bulk copies of this tile's rows landed
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();  // (and the zero-filled rows); the previous tile's TMEM reads are done
    for (int i = tid; i < M * kc; i += 256) {
      // 8 consecutive threads: one core matrix (rows m..m+7 of chunk c, 128
      // contiguous bytes of each plane); raw reads at row pitch 4w (w % 4 == 0)
      // hit distinct bank groups
      const int rest = i >> 3, c = rest % kc, m = (rest / kc) * 8 + (i & 7);
      const int off = c * LBO_A + (m >> 3) * SBO + (m & 7) * 16;
      const float4 x = c < wc ? *reinterpret_cast<const float4*>(A_raw + m * rowbytes + 16 * c)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
      uint32_t h0, h1, h2, h3, l0, l1, l2, l3;
      split_tf32(x.x, h0, l0);
      split_tf32(x.y, h1, l1);
      split_tf32(x.z, h2, l2);
      split_tf32(x.w, h3, l3);
      *reinterpret_cast<uint4*>(A_hi + off) = make_uint4(h0, h1, h2, h3);
      *reinterpret_cast<uint4*>(A_lo + off) = make_uint4(l0, l1, l2, l3);
    }
    if (tid < M) hrow_s[tid] = hrow_of(tile + G, tid);
    if (tid == 0) expect(tile + G);
    const int trow = (gr >= 0 && gr < nVl) ? ownl + a.rank[a.voff_l + gr] : -1;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> tensor core
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t ah = smem_u32(A_hi), al = smem_u32(A_lo), bh = smem_u32(B_hi), bl = smem_u32(B_lo);
      for (int s2 = 0; s2 < kc / 2; ++s2) {
        const uint32_t oa = 2 * s2 * LBO_A, ob = 2 * s2 * LBO_B;
        mma(tmem, desc(al + oa, LBO_A), desc(bh + ob, LBO_B), s2 > 0);
        mma(tmem, desc(ah + oa, LBO_A), desc(bl + ob, LBO_B), 1);
        mma(tmem, desc(ah + oa, LBO_A), desc(bh + ob, LBO_B), 1);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(mbar))
                   : "memory");
    }
    issue(tile + G);  // raw buffer is free: the split is done (fence.proxy.async above)
    wait_bar(mbar, k & 1);  // the accumulator
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t v[32];
    {
      const uint32_t taddr = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + 32 * ch;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
            "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
            "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    }
    if (r0 + row < n) {
      const int64_t G2 = own0 + r0 + row;
      float4* zr = reinterpret_cast<float4*>(a.z + G2 * N + 32 * ch);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        zr[q] = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                            __uint_as_float(v[4 * q + 3]));
#pragma unroll
      for (int h0 = 0; h0 < 32; h0 += DH) {  // heads inside this thread's 32 columns (static indices:
        const int hh = (32 * ch + h0) / DH;  // the accumulator stays in registers)
        float sv = 0.f, tv = 0.f;
#pragma unroll
        for (int j = 0; j < DH; ++j) {
          const float zv = __uint_as_float(v[h0 + j]);
          sv = fmaf(zv, av_s[32 * ch + h0 + j], sv);
          tv = fmaf(zv, av_s[64 + 32 * ch + h0 + j], tv);
        }
        a.s[G2 * H + hh] = sv;
        if (trow >= 0) a.t[(int64_t)trow * H + hh] = tv;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(64));
}

// TM = 32 rows per tile; NT = 8 * NQ register tiles (4 rows x 4 outputs),
// NS = 256 / NT K-slices (NQ <= 32 -> D <= 128).
template <int NQ>
__global__ void __launch_bounds__(256) k_gat_project_tiled(const SgMeta* __restrict__ meta, ProjArgs a) {
  SG_PDL_ENTRY();
  constexpr int TM = 32, TMP = TM + 4;
  constexpr int NT = (TM / 4) * NQ;
  constexpr int NS = 256 / NT;
  extern __shared__ __align__(16) float smem[];
  const int w = a.w, D = a.dout, H = a.heads, dh = D / H;
  float* W_s = smem;               // [w][D]
  float* A_s = W_s + w * D;        // [w][TM+4] transposed
  float* red = A_s + w * TMP;      // [NS][TM][D]
  int* prow = (int*)(red + NS * TM * D);
  for (int i = threadIdx.x; i < w * D / 4; i += 256)
    reinterpret_cast<float4*>(W_s)[i] = reinterpret_cast<const float4*>(a.W)[i];
  const int l = a.l, d = a.d;
  const int n = meta->n_own[l - 1][d];
  const int own0 = meta->own_off[l - 1][d];
  const int ownl = meta->own_off[l][d];
  const int64_t nVl = meta->nV[l];
  const int tile = threadIdx.x % NT, ks = threadIdx.x / NT;
  const int rt = tile / NQ, jq = tile - rt * NQ;
  const int kchunk = (w + NS - 1) / NS;
  const int kb = ks * kchunk, ke = min(w, kb + kchunk);
  const int w4 = w / 4;
  for (int r0 = blockIdx.x * TM; r0 < n; r0 += gridDim.x * TM) {
    __syncthreads();
    if (threadIdx.x < TM) {
      const int r = r0 + threadIdx.x;
      int pr = -1;
      if (r < n) {
        pr = own0 + r;
        if (a.src_row) pr = a.src_row[pr];
      }
      prow[threadIdx.x] = pr;
    }
    __syncthreads();
    {
      constexpr int MA = 4;  // TM * w4 / 256 <= 4 for w <= 128
      float4 ab[MA];
#pragma unroll
      for (int u = 0; u < MA; ++u) {
        const int idx = threadIdx.x + 256 * u;
        ab[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (idx < TM * w4) {
          const int r = idx & (TM - 1), q = idx / TM;
          if (prow[r] >= 0) ab[u] = __ldg(reinterpret_cast<const float4*>(a.h_prev + (int64_t)prow[r] * w) + q);
        }
      }
#pragma unroll
      for (int u = 0; u < MA; ++u) {
        const int idx = threadIdx.x + 256 * u;
        if (idx < TM * w4) {
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
      const float4 wv = *reinterpret_cast<const float4*>(W_s + k * D + 4 * jq);
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
      *reinterpret_cast<float4*>(red + (ks * TM + 4 * rt + i) * D + 4 * jq) =
          make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    __syncthreads();
    // z = sum of the K slices (fixed order); slice 0 keeps the total for the epilogue
    for (int idx = threadIdx.x; idx < TM * D; idx += 256) {
      const int r = idx / D, j = idx - r * D;
      float v = 0.f;
#pragma unroll
      for (int s2 = 0; s2 < NS; ++s2) v += red[(s2 * TM + r) * D + j];
      red[r * D + j] = v;
      if (r0 + r < n) a.z[(int64_t)(own0 + r0 + r) * D + j] = v;
    }
    __syncthreads();
    // scores s = z.a_src per head; t = z.a_dst on self rows
    for (int idx = threadIdx.x; idx < TM * H; idx += 256) {
      const int r = idx / H, hh = idx - r * H;
      if (r0 + r >= n) continue;
      const int G = own0 + r0 + r;
      const float* zr = red + r * D + hh * dh;
      float sv = 0.f;
      for (int j = 0; j < dh; ++j) sv = fmaf(zr[j], a.a_src[hh * dh + j], sv);
      a.s[(int64_t)G * H + hh] = sv;
      const int p = a.grouped[a.voff_lm1 + G];
      if (p < nVl) {
        float tv = 0.f;
        for (int j = 0; j < dh; ++j) tv = fmaf(zr[j], a.a_dst[hh * dh + j], tv);
        a.t[(int64_t)(ownl + a.rank[a.voff_l + p]) * H + hh] = tv;
      }
    }
  }
}

// ---------------------------------------------------------------- online-softmax aggregation
struct AggArgs {
  int l, d, dout, heads, stride;
  float slope;
  int64_t eoff_li, rbase_li, pbase_l;
  const int32_t* rowbeg;
  const int32_t* rowend;
  const int32_t* lsrc;
  const int32_t* dperm;
  const int32_t* sendpos;
  const float* z;
  const float* s;
  const float* t;
  const float* t_recv;  // pair layout, stride H
  float* pre_e;         // [edge][head]
  float* loc_m;         // [row][head]
  float* loc_s;
  float* loc_U;         // [row][D]
  float* sendbuf;       // [U (D) | m (H) | s (H)]
  // one device (no holders to combine): the owner combine and alpha folded in
  int fuse, final_;
  float* md;     // [m (H) | den (H)] per owned row
  float* num;    // [row][D]
  float* h;      // [row][D]
  float* alpha;  // [edge][head]
};

// Team of RL = LPR*EG lanes per destination row; LPR lanes span D (VEC each),
// LH = LPR/H lanes per head; EG edge groups merged by a fixed xor tree.
template <int VEC, int LPR, int EG>
__global__ void __launch_bounds__(256) k_gat_agg(const SgMeta* __restrict__ meta, AggArgs a) {
  SG_PDL_ENTRY();
  using V = V4<VEC>;
  using T = typename V::T;
  constexpr int RL = LPR * EG;
  constexpr int RPW = 32 / RL;
  const int l = a.l, d = a.d, dout = a.dout, H = a.heads, LH = LPR / H;
  const int n_own = meta->n_own[l][d];
  const int R = n_own + meta->n_ref[l][d];
  const int own0 = meta->own_off[l][d], ref0 = meta->ref_off[l][d];
  const int prev0 = meta->own_off[l - 1][d];
  const int64_t rb = a.rbase_li + own0 + ref0;
  const int lane = threadIdx.x & 31;
  const int team = lane / RL, tl = lane % RL, eg = tl / LPR, lr = tl % LPR;
  const int hl = lr / LH;           // this lane's head
  const bool head_lead = (lr % LH) == 0;
  const unsigned tmask = (RL == 32) ? 0xffffffffu : (((1u << RL) - 1u) << (team * RL));
  const int col = lr * VEC;
  const bool colok = col < dout;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = gw * RPW + team; q < R; q += nw * RPW) {
    const bool own = q < n_own;
    const int slot = own ? 0 : a.sendpos[a.pbase_l + ref0 + (q - n_own)];
    const float tq = own ? a.t[(int64_t)(own0 + q) * H + hl] : a.t_recv[(int64_t)slot * H + hl];
    const int b = a.rowbeg[rb + q], e = a.rowend[rb + q];
    float m = -INFINITY, ssum = 0.f;
    T U = V::zero();
    // four edges' loads in flight per edge group, applied in edge order
    for (int j0 = b + eg; j0 < e; j0 += 4 * EG) {
      int64_t xs[4];
      int us[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int j = j0 + t * EG;
        xs[t] = j < e ? (a.dperm ? (int64_t)a.dperm[j] : a.eoff_li + j) : 0;
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) us[t] = j0 + t * EG < e ? prev0 + a.lsrc[xs[t]] : 0;
      float pres[4];
      T zs[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const bool ok = j0 + t * EG < e;
        pres[t] = ok ? a.s[(int64_t)us[t] * H + hl] + tq : 0.f;
        zs[t] = (ok && colok) ? V::ld(a.z + (int64_t)us[t] * dout + col) : V::zero();
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if (j0 + t * EG >= e) break;
        const float pre = pres[t];
        const float ev = leaky(pre, a.slope);
        if (head_lead && colok) a.pre_e[xs[t] * H + hl] = pre;
        const T zu = zs[t];
        if (ev > m) {
          const float sc = expf(m - ev);  // 0 on the first edge (m = -inf)
          ssum = fmaf(ssum, sc, 1.f);
          U = V::axpby(1.f, zu, sc, U);
          m = ev;
        } else {
          const float wv = expf(ev - m);
          ssum += wv;
          V::fma_(U, wv, zu);
        }
      }
    }
#pragma unroll
    for (int o = LPR; o < RL; o <<= 1) {
      const float m2 = __shfl_xor_sync(tmask, m, o, RL);
      const float s2 = __shfl_xor_sync(tmask, ssum, o, RL);
      const T U2 = V::shfl_xor(tmask, U, o, RL);
      const float mm = fmaxf(m, m2);
      const float f1 = (m == -INFINITY) ? 0.f : expf(m - mm);
      const float f2 = (m2 == -INFINITY) ? 0.f : expf(m2 - mm);
      ssum = ssum * f1 + s2 * f2;
      U = V::axpby(f1, U, f2, U2);
      m = mm;
    }
    if (a.fuse) {  // warp-uniform; every row is owned (g == 1)
      const int64_t G = own0 + q;
      if (eg == 0 && colok) {  // k_gat_combine with no senders: num = U / den
        const T nv = V::div(U, ssum);
        V::st(a.num + G * dout + col, nv);
        V::st(a.h + G * dout + col, a.final_ ? nv : V::relu(nv));
        if (head_lead) {
          a.md[G * 2 * H + hl] = m;
          a.md[G * 2 * H + H + hl] = ssum;
        }
      }
      // k_gat_alpha over this row's edges: each edge group re-reads the pre_e its
      // head lead wrote in the first pass (one hop instead of lsrc -> s)
      if (head_lead && colok)
        for (int j0 = b + eg; j0 < e; j0 += 4 * EG) {
          int64_t xs[4];
          float pr[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int j = j0 + t * EG;
            xs[t] = j < e ? (a.dperm ? (int64_t)a.dperm[j] : a.eoff_li + j) : 0;
          }
#pragma unroll
          for (int t = 0; t < 4; ++t) pr[t] = j0 + t * EG < e ? a.pre_e[xs[t] * H + hl] : 0.f;
#pragma unroll
          for (int t = 0; t < 4; ++t)
            if (j0 + t * EG < e) a.alpha[xs[t] * H + hl] = expf(leaky(pr[t], a.slope) - m) / ssum;
        }
      continue;
    }
    if (eg != 0) continue;
    if (own) {
      const int64_t G = own0 + q;
      if (colok) V::st(a.loc_U + G * dout + col, U);
      if (head_lead && colok) {
        a.loc_m[G * H + hl] = m;
        a.loc_s[G * H + hl] = ssum;
      }
    } else {
      float* out = a.sendbuf + (int64_t)slot * a.stride;
      if (colok) {
        if ((a.stride & 3) == 0 && VEC == 4) V::st(out + col, U); else V::st_any(out + col, U);
      }
      if (head_lead && colok) {
        out[dout + hl] = m;
        out[dout + H + hl] = ssum;
      }
    }
  }
}

// ---------------------------------------------------------------- owner combine
struct CombArgs {
  int l, d, dout, heads, g, stride, final_;
  int64_t voff_l;
  const int32_t* contrib;
  const float* loc_m;
  const float* loc_s;
  const float* loc_U;
  const float* recv;  // [U | m | s] rows, receive layout
  float* md;          // [m (H) | den (H)] per owned row
  float* num;
  float* h;
};

__global__ void k_gat_combine(const SgMeta* __restrict__ meta, CombArgs a) {
  SG_PDL_ENTRY();
  const int l = a.l, d = a.d, dout = a.dout, g = a.g, H = a.heads, dh = dout / H;
  const int n = meta->n_own[l][d];
  const int own0 = meta->own_off[l][d];
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)n * dout;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(idx / dout), j = (int)(idx - (int64_t)q * dout);
    const int hh = j / dh;
    const int64_t G = own0 + q;
    const int* cb = a.contrib + (int64_t)g * a.voff_l + G * g;
    const float m0 = a.loc_m[G * H + hh];
    float m = m0;
    for (int s = 0; g > 1 && s < g; ++s) {
      const int rs = cb[s];
      if (rs >= 0) m = fmaxf(m, a.recv[(int64_t)rs * a.stride + dout + hh]);
    }
    const float f = expf(m0 - m);
    float den = a.loc_s[G * H + hh] * f;
    float U = a.loc_U[G * dout + j] * f;
    for (int s = 0; g > 1 && s < g; ++s) {  // ascending sender order
      const int rs = cb[s];
      if (rs >= 0) {
        const float* r = a.recv + (int64_t)rs * a.stride;
        const float fs = expf(r[dout + hh] - m);
        den = fmaf(r[dout + H + hh], fs, den);
        U = fmaf(r[j], fs, U);
      }
    }
    const float nv = U / den;
    a.num[G * dout + j] = nv;
    a.h[G * dout + j] = a.final_ ? nv : sg_relu(nv);
    if (j - hh * dh == 0) {
      a.md[G * 2 * H + hh] = m;
      a.md[G * 2 * H + H + hh] = den;
    }
  }
}

// ---------------------------------------------------------------- alpha per edge and head
struct AlphaArgs {
  int l, d, heads;
  float slope;
  int64_t eoff_li, pbase_l;
  const int32_t* ldst;
  const int32_t* sendpos;
  const float* pre_e;
  const float* md;        // owned rows, stride 2H
  const float* md_recv;   // pair layout, stride 2H
  float* alpha;
};

__global__ void k_gat_alpha(const SgMeta* __restrict__ meta, AlphaArgs a) {
  SG_PDL_ENTRY();
  const int l = a.l, d = a.d, li = l - 1, H = a.heads;
  const int b = meta->edge_off[li][d], e = meta->edge_off[li][d + 1];
  const int n_own = meta->n_own[l][d];
  const int own0 = meta->own_off[l][d], ref0 = meta->ref_off[l][d];
  const int64_t tot = (int64_t)(e - b) * H;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < tot;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int i = b + (int)(k / H), hh = (int)(k % H);
    const int64_t x = a.eoff_li + i;
    const int q = a.ldst[x];
    const float* mdp = q < n_own ? a.md + 2 * (int64_t)H * (own0 + q)
                                 : a.md_recv + 2 * (int64_t)H * a.sendpos[a.pbase_l + ref0 + (q - n_own)];
    a.alpha[x * H + hh] = expf(leaky(a.pre_e[x * H + hh], a.slope) - mdp[hh]) / mdp[H + hh];
  }
}

// ---------------------------------------------------------------- backward
struct BRowsArgs {
  int l, d, dout, heads, final_;
  const float* d_h;
  const float* num;
  float* dnc;  // [d_num (D) | c (H)] per owned row (stride D+H)
};

__global__ void k_gat_bwd_rows(const SgMeta* __restrict__ meta, BRowsArgs a) {
  SG_PDL_ENTRY();
  const int l = a.l, d = a.d, dout = a.dout, H = a.heads, dh = dout / H, st = dout + H;
  const int n = meta->n_own[l][d];
  const int own0 = meta->own_off[l][d];
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < (int64_t)n * H;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(k / H), hh = (int)(k % H);
    const int64_t G = own0 + q;
    float c = 0.f;
    for (int j = hh * dh; j < (hh + 1) * dh; ++j) {
      const float nv = a.num[G * dout + j];
      float dn = a.d_h[G * dout + j];
      if (!a.final_ && !(nv > 0.f)) dn = 0.f;
      a.dnc[G * st + j] = dn;
      c = fmaf(dn, nv, c);
    }
    a.dnc[G * st + dout + hh] = c;
  }
}

// k_gat_bwd_rows with float4 lanes: LPH = d_head / 4 consecutive threads per
// head of a row (power of two, <= 32), c reduced by an xor tree inside the
// group; coalesced float4 loads of d_h / num (the scalar kernel walked d_head
// contiguous floats per thread: 16 us for C3 layer 1 -> a few us).
template <int LPH>
__global__ void k_gat_bwd_rows4(const SgMeta* __restrict__ meta, BRowsArgs a) {
  SG_PDL_ENTRY();
  const int l = a.l, d = a.d, dout = a.dout, H = a.heads, st = dout + H, q4 = dout / 4;
  const int n = meta->n_own[l][d];
  const int own0 = meta->own_off[l][d];
  const int64_t tot = (int64_t)n * q4;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k0 = t0 - (t0 % 32); k0 < tot; k0 += step) {  // warp-uniform trip count
    const int64_t k = k0 + (threadIdx.x & 31);
    const bool ok = k < tot;
    const int64_t q = ok ? k / q4 : 0;
    const int c4 = ok ? (int)(k - q * q4) : 0;
    const int64_t G = own0 + q;
    float4 nv = make_float4(0.f, 0.f, 0.f, 0.f), dn = nv;
    if (ok) {
      nv = *reinterpret_cast<const float4*>(a.num + G * dout + 4 * c4);
      dn = *reinterpret_cast<const float4*>(a.d_h + G * dout + 4 * c4);
      if (!a.final_) {
        if (!(nv.x > 0.f)) dn.x = 0.f;
        if (!(nv.y > 0.f)) dn.y = 0.f;
        if (!(nv.z > 0.f)) dn.z = 0.f;
        if (!(nv.w > 0.f)) dn.w = 0.f;
      }
      float* o = a.dnc + G * st + 4 * c4;  // stride D + H: not 16 B aligned
      o[0] = dn.x; o[1] = dn.y; o[2] = dn.z; o[3] = dn.w;
    }
    float c = fmaf(dn.x, nv.x, fmaf(dn.y, nv.y, fmaf(dn.z, nv.z, dn.w * nv.w)));
#pragma unroll
    for (int o2 = 1; o2 < LPH; o2 <<= 1) c += __shfl_xor_sync(0xffffffffu, c, o2);
    if (ok && c4 % LPH == 0) a.dnc[G * st + dout + c4 / LPH] = c;
  }
}

struct BDstArgs {
  int l, d, dout, heads, stride;
  float slope;
  int64_t eoff_li, rbase_li, pbase_l;
  const int32_t* rowbeg;
  const int32_t* rowend;
  const int32_t* lsrc;
  const int32_t* dperm;
  const int32_t* sendpos;
  const float* z;
  const float* alpha;
  const float* pre_e;
  const float* dnc;       // owned rows, stride D+H
  const float* dnc_recv;  // pair layout, stride `stride`
  float* d_pre;           // [edge][head]
  float* dt_loc;          // [row][head]
  float* sendbuf;         // dt per pair slot (stride H)
};

template <int VEC, int LPR, int EG>
__global__ void __launch_bounds__(256) k_gat_bwd_dst(const SgMeta* __restrict__ meta, BDstArgs a) {
  SG_PDL_ENTRY();
  using V = V4<VEC>;
  using T = typename V::T;
  constexpr int RL = LPR * EG;
  constexpr int RPW = 32 / RL;
  const int l = a.l, d = a.d, dout = a.dout, H = a.heads, LH = LPR / H;
  const int n_own = meta->n_own[l][d];
  const int R = n_own + meta->n_ref[l][d];
  const int own0 = meta->own_off[l][d], ref0 = meta->ref_off[l][d];
  const int prev0 = meta->own_off[l - 1][d];
  const int64_t rb = a.rbase_li + own0 + ref0;
  const int lane = threadIdx.x & 31;
  const int team = lane / RL, tl = lane % RL, eg = tl / LPR, lr = tl % LPR;
  const int hl = lr / LH;
  const bool head_lead = (lr % LH) == 0;
  const unsigned tmask = (RL == 32) ? 0xffffffffu : (((1u << RL) - 1u) << (team * RL));
  const int col = lr * VEC;
  const bool colok = col < dout;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = gw * RPW + team; q < R; q += nw * RPW) {
    const bool own = q < n_own;
    const int slot = own ? 0 : a.sendpos[a.pbase_l + ref0 + (q - n_own)];
    const float* dn_row = own ? a.dnc + (int64_t)(own0 + q) * (dout + H) : a.dnc_recv + (int64_t)slot * a.stride;
    const T dn = colok ? V::ld_any(dn_row + col) : V::zero();  // stride D+H: not 16B aligned
    const float c = dn_row[dout + hl];
    const int b = a.rowbeg[rb + q], e = a.rowend[rb + q];
    float dt = 0.f;
    const int rounds = (e - b + EG - 1) / EG;
    // four rounds' loads in flight (the index chain and the z / alpha / pre_e
    // reads of round k no longer wait for round k-1); rounds still applied in order
    for (int k0 = 0; k0 < rounds; k0 += 4) {
      int64_t xs[4];
      int us[4];
      bool oks[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int j = b + (k0 + t) * EG + eg;
        oks[t] = k0 + t < rounds && j < e;
        xs[t] = oks[t] ? (a.dperm ? (int64_t)a.dperm[j] : a.eoff_li + j) : 0;
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) us[t] = oks[t] ? prev0 + a.lsrc[xs[t]] : 0;
      T zs[4];
      float als[4], prs[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        zs[t] = (oks[t] && colok) ? V::ld(a.z + (int64_t)us[t] * dout + col) : V::zero();
        als[t] = oks[t] ? a.alpha[xs[t] * H + hl] : 0.f;
        prs[t] = oks[t] ? a.pre_e[xs[t] * H + hl] : 0.f;
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if (k0 + t >= rounds) break;  // team-uniform
        float part = (oks[t] && colok) ? V::dot(dn, zs[t]) : 0.f;
        // d_alpha = d_num . z_u per head: reduce over the LH lanes of the head
        for (int o = 1; o < LH; o <<= 1) part += __shfl_xor_sync(tmask, part, o, RL);
        if (oks[t]) {
          const float de = als[t] * (part - c);
          const float dp = de * (prs[t] > 0.f ? 1.f : a.slope);
          if (head_lead && colok) a.d_pre[xs[t] * H + hl] = dp;
          dt += dp;
        }
      }
    }
#pragma unroll
    for (int o = LPR; o < RL; o <<= 1) dt += __shfl_xor_sync(tmask, dt, o, RL);
    if (eg != 0 || !head_lead || !colok) continue;
    if (own) a.dt_loc[(int64_t)(own0 + q) * H + hl] = dt;
    else a.sendbuf[(int64_t)slot * H + hl] = dt;
  }
}

struct BSrcArgs {
  int l, d, dout, heads, g, stride;
  int64_t voff_lm1, voff_l, pbase_l, key_base;
  const int32_t* grouped;
  const int32_t* rank;
  const int32_t* contrib;
  const int32_t* ldst;
  const int32_t* sendpos;
  const int32_t* perm;  // edge slots sorted by source row
  const int32_t* srcbeg;
  const int32_t* srcend;
  const float* alpha;
  const float* d_pre;
  const float* dnc;
  const float* dnc_recv;
  int dnc_stride;
  const float* dt_loc;
  const float* dt_recv;  // receive layout, stride H
  const float* a_src;
  const float* a_dst;
  float* d_z;
  float* ds;      // [row][head]
  float* dt_tot;  // [row][head]
};

// warp per source row; NG = 32/LPR lane groups split the out-edges
template <int VEC, int LPR>
__global__ void __launch_bounds__(256) k_gat_bwd_src(const SgMeta* __restrict__ meta, BSrcArgs a) {
  SG_PDL_ENTRY();
  using V = V4<VEC>;
  using T = typename V::T;
  constexpr int NG = 32 / LPR;
  const int l = a.l, d = a.d, dout = a.dout, H = a.heads, LH = LPR / H;
  const int n_prev = meta->n_own[l - 1][d];
  const int prev0 = meta->own_off[l - 1][d];
  const int own0 = meta->own_off[l][d], n_own = meta->n_own[l][d], ref0 = meta->ref_off[l][d];
  const int64_t nVl = meta->nV[l];
  const int lane = threadIdx.x & 31;
  const int gi = lane / LPR, lr = lane % LPR;
  const int hl = lr / LH;
  const bool head_lead = (lr % LH) == 0;
  const int col = lr * VEC;
  const bool colok = col < dout;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // software-pipelined over this warp's rows: the next row's out-edge range is
  // fetched while the current row's edges land, and the self-row chain
  // (grouped -> rank -> dt) is issued before the edge loop so the two
  // dependent chains overlap
  int nb_ = 0, ne_ = 0;
  if (gw < n_prev) {
    nb_ = a.srcbeg[a.key_base + prev0 + gw];
    ne_ = a.srcend[a.key_base + prev0 + gw];
  }
  for (int64_t u = gw; u < n_prev; u += nw) {
    const int64_t U = prev0 + u;
    T acc = V::zero();
    float dsv = 0.f;
    const int b = nb_, e = ne_;
    if (u + nw < n_prev) {
      nb_ = a.srcbeg[a.key_base + U + nw];
      ne_ = a.srcend[a.key_base + U + nw];
    }
    const int p = a.grouped[a.voff_lm1 + U];
    int64_t vself = -1;
    float dt = 0.f;
    if (p < nVl) {  // self row of owned v: d_z += dt_v * a_dst (owner combines holders' dt)
      vself = own0 + a.rank[a.voff_l + p];
      dt = a.dt_loc[vself * H + hl];
      const int* cb = a.contrib + (int64_t)a.g * a.voff_l + vself * a.g;
      for (int s = 0; a.g > 1 && s < a.g; ++s) {
        const int rs = cb[s];
        if (rs >= 0) dt += a.dt_recv[(int64_t)rs * H + hl];
      }
    }
    for (int jb = b; jb < e; jb += 32) {
      const int j = jb + lane;
      const int my = j < e ? a.perm[j] : 0;
      const int cnt = min(32, e - jb);
      const int rounds = (cnt + NG - 1) / NG;
      // four rounds' edges in flight at once (hub rows have hundreds of
      // out-edges: one dependent load chain per round was their whole cost);
      // accumulation order unchanged (rounds ascending)
      for (int kk = 0; kk < rounds; kk += 4) {
        int xs[4];
        bool ok[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = (kk + u) * NG + gi;
          xs[u] = __shfl_sync(0xffffffffu, my, k < 32 ? k : 31);
          ok[u] = kk + u < rounds && k < cnt;
        }
        const float* rows[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          rows[u] = nullptr;
          if (ok[u]) {
            const int q = a.ldst[xs[u]];
            rows[u] = q < n_own ? a.dnc + (int64_t)(own0 + q) * (dout + H)
                                : a.dnc_recv + (int64_t)a.sendpos[a.pbase_l + ref0 + (q - n_own)] * a.dnc_stride;
          }
        }
        T vals[4];
        float al[4], dp[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const bool go = ok[u] && colok;
          vals[u] = go ? V::ld_any(rows[u] + col) : V::zero();
          al[u] = go ? a.alpha[(int64_t)xs[u] * H + hl] : 0.f;
          dp[u] = go ? a.d_pre[(int64_t)xs[u] * H + hl] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (ok[u] && colok) {
            V::fma_(acc, al[u], vals[u]);
            dsv += dp[u];
          }
      }
    }
#pragma unroll
    for (int o = LPR; o < 32; o <<= 1) {
      V::add(acc, V::shfl_xor(0xffffffffu, acc, o, 32));
      dsv += __shfl_xor_sync(0xffffffffu, dsv, o);
    }
    if (gi != 0) continue;
    if (colok) V::fma_(acc, dsv, V::ld_any(a.a_src + col));  // d_z += ds * a_src
    if (vself >= 0) {
      if (colok) V::fma_(acc, dt, V::ld_any(a.a_dst + col));
      if (head_lead && colok) a.dt_tot[vself * H + hl] = dt;
    }
    if (colok) V::st(a.d_z + U * dout + col, acc);  // dout % VEC == 0: aligned
    if (head_lead && colok) a.ds[U * H + hl] = dsv;
  }
}

// per-block partials of [dW | da_src | da_dst] over source rows; d_h_prev
constexpr int QTR = 32;
constexpr int QMAXQ = 8;  // scalar slots / 4 per thread: w*dout <= 8192

struct BParamArgs {
  int l, d, w, dout, heads;
  int64_t voff_lm1, voff_l;
  const float* h_prev;
  const int32_t* src_row;
  const int32_t* grouped;
  const int32_t* rank;
  const float* z;
  const float* d_z;
  const float* ds;
  const float* dt_tot;
  const float* W;
  float* partial;
  float* d_prev;
};

// T4 (w % 4 == 0 and dout % 4 == 0): thread slot (cg, jg) owns a 4x4 dW tile,
// per row 2 LDS.128 + 16 FFMA; otherwise one scalar slot per (c, j).
template <int MODE>  // 0 scalar FFMA, 1 4x4 FFMA tiles (dout == 64 runs k_gat_wgrad_mma)
__global__ void __launch_bounds__(256) k_gat_bwd_param(const SgMeta* __restrict__ meta, BParamArgs a) {
  SG_PDL_ENTRY();
  extern __shared__ __align__(16) float smem[];
  const int w = a.w, dout = a.dout, H = a.heads, dh = dout / H;
  constexpr bool T4 = MODE >= 1;
  const int wp = T4 ? w + 4 : w + 1;  // h row stride (float4-aligned for T4)
  const int dzp = dout;
  const int wt = w + 1;               // W^T row stride (d_prev: lanes run along c)
  float* dz_s = smem;               // [QTR][dzp]
  float* Wt_s = dz_s + QTR * dzp;   // [dout][w+1] = W^T (for d_prev)
  float* h_s = Wt_s + dout * wt;    // [QTR][wp]
  float* z_s = h_s + QTR * wp;      // [QTR][dout]
  float* ds_s = z_s + QTR * dout;   // [QTR][H]
  float* dt_s = ds_s + QTR * H;     // [QTR][H] (0 when not a self row)
  int* prow_s = (int*)(dt_s + QTR * H);
  if (a.d_prev)
    for (int i = threadIdx.x; i < w * dout; i += blockDim.x) {
      const int c = i / dout, j = i - c * dout;
      Wt_s[j * wt + c] = a.W[i];
    }
  const int l = a.l, d = a.d;
  const int n = meta->n_own[l - 1][d];
  const int own0 = meta->own_off[l - 1][d];
  const int ownl = meta->own_off[l][d];
  const int64_t nVl = meta->nV[l];
  const int nslots = T4 ? (w / 4) * (dout / 4) : w * dout;
  const int nq = dout / 4;
  float acc[QMAXQ * 4];
#pragma unroll
  for (int k = 0; k < QMAXQ * 4; ++k) acc[k] = 0.f;
  float as = 0.f, ad = 0.f;
  const int ntiles = (n + QTR - 1) / QTR;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    __syncthreads();
    const int nrow = min(QTR, n - tile * QTR);
    if (threadIdx.x < QTR) {
      const int rr = threadIdx.x;
      prow_s[rr] = -1;
      if (rr < nrow) {
        const int G = own0 + tile * QTR + rr;
        int r = G;
        if (a.src_row) r = a.src_row[r];
        prow_s[rr] = r;
      }
    }
    for (int idx = threadIdx.x; idx < QTR * H; idx += blockDim.x) {
      const int rr = idx / H, hh = idx - rr * H;
      float dsv = 0.f, dtv = 0.f;
      if (rr < nrow) {
        const int G = own0 + tile * QTR + rr;
        dsv = a.ds[(int64_t)G * H + hh];
        const int p = a.grouped[a.voff_lm1 + G];
        if (p < nVl) dtv = a.dt_tot[(int64_t)(ownl + a.rank[a.voff_l + p]) * H + hh];
      }
      ds_s[idx] = dsv;
      dt_s[idx] = dtv;
    }
    if (T4) {
      for (int idx = threadIdx.x; idx < QTR * nq; idx += blockDim.x) {
        const int rr = idx / nq, q = idx - rr * nq;
        float4 vz = make_float4(0.f, 0.f, 0.f, 0.f), vd = vz;
        if (rr < nrow) {
          const int64_t G = own0 + tile * QTR + rr;
          vd = *reinterpret_cast<const float4*>(a.d_z + G * dout + 4 * q);
          vz = *reinterpret_cast<const float4*>(a.z + G * dout + 4 * q);
        }
        *reinterpret_cast<float4*>(dz_s + rr * dzp + 4 * q) = vd;
        *reinterpret_cast<float4*>(z_s + rr * dout + 4 * q) = vz;
      }
    } else {
      for (int idx = threadIdx.x; idx < QTR * dout; idx += blockDim.x) {
        const int rr = idx / dout;
        const bool v = rr < nrow;
        const int64_t G = own0 + tile * QTR + rr;
        dz_s[idx] = v ? a.d_z[G * dout + (idx - rr * dout)] : 0.f;
        z_s[idx] = v ? a.z[G * dout + (idx - rr * dout)] : 0.f;
      }
    }
    __syncthreads();
    if (T4) {
      const int w4 = w / 4;
      for (int idx = threadIdx.x; idx < QTR * w4; idx += blockDim.x) {
        const int rr = idx / w4, q = idx - rr * w4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (prow_s[rr] >= 0) v = __ldg(reinterpret_cast<const float4*>(a.h_prev + (int64_t)prow_s[rr] * w) + q);
        *reinterpret_cast<float4*>(h_s + rr * wp + 4 * q) = v;
      }
    } else {
#pragma unroll 4
      for (int idx = threadIdx.x; idx < QTR * w; idx += blockDim.x) {
        const int rr = idx / w, c = idx - rr * w;
        h_s[rr * wp + c] = prow_s[rr] >= 0 ? __ldg(a.h_prev + (int64_t)prow_s[rr] * w + c) : 0.f;
      }
    }
    __syncthreads();
    if (T4) {
#pragma unroll
      for (int s2 = 0; s2 < QMAXQ / 4 * 2; ++s2) {  // up to 4 tiles of 16 per thread
        const int slot = threadIdx.x + 256 * s2;
        if (s2 < 2 && slot < nslots) {
          const int cg = slot / nq, jg = slot - cg * nq;
          float* t = acc + 16 * s2;
#pragma unroll 4
          for (int rr = 0; rr < QTR; ++rr) {
            const float4 a4 = *reinterpret_cast<const float4*>(h_s + rr * wp + 4 * cg);
            const float4 g4 = *reinterpret_cast<const float4*>(dz_s + rr * dzp + 4 * jg);
            const float av[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              t[4 * i + 0] = fmaf(av[i], g4.x, t[4 * i + 0]);
              t[4 * i + 1] = fmaf(av[i], g4.y, t[4 * i + 1]);
              t[4 * i + 2] = fmaf(av[i], g4.z, t[4 * i + 2]);
              t[4 * i + 3] = fmaf(av[i], g4.w, t[4 * i + 3]);
            }
          }
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < QMAXQ * 4; ++k) {
        const int idx = threadIdx.x + 256 * k;
        if (idx < nslots) {
          const int c = idx / dout, j = idx - c * dout;
          float sacc = acc[k];
#pragma unroll 8
          for (int rr = 0; rr < QTR; ++rr) sacc = fmaf(h_s[rr * wp + c], dz_s[rr * dout + j], sacc);
          acc[k] = sacc;
        }
      }
    }
    if (threadIdx.x < dout) {
      const int j = threadIdx.x, hh = j / dh;
      for (int rr = 0; rr < QTR; ++rr) {
        as = fmaf(z_s[rr * dout + j], ds_s[rr * H + hh], as);
        ad = fmaf(z_s[rr * dout + j], dt_s[rr * H + hh], ad);
      }
    }
    if (a.d_prev) {
      for (int idx = threadIdx.x; idx < nrow * w; idx += blockDim.x) {
        const int rr = idx / w, c = idx - rr * w;
        float sacc = 0.f;
        const float* dzr = dz_s + rr * dzp;
#pragma unroll 8
        for (int j = 0; j < dout; ++j) sacc = fmaf(dzr[j], Wt_s[j * wt + c], sacc);
        a.d_prev[(int64_t)(own0 + tile * QTR + rr) * w + c] = sacc;
      }
    }
  }
  const int64_t ntot = (int64_t)w * dout + 2 * dout;
  float* out = a.partial + (int64_t)blockIdx.x * ntot;
  if (T4) {
#pragma unroll
    for (int s2 = 0; s2 < 2; ++s2) {
      const int slot = threadIdx.x + 256 * s2;
      if (slot < nslots) {
        const int cg = slot / nq, jg = slot - cg * nq;
        const float* t = acc + 16 * s2;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          *reinterpret_cast<float4*>(out + (4 * cg + i) * dout + 4 * jg) =
              make_float4(t[4 * i + 0], t[4 * i + 1], t[4 * i + 2], t[4 * i + 3]);
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < QMAXQ * 4; ++k) {
      const int idx = threadIdx.x + 256 * k;
      if (idx < nslots) out[idx] = acc[k];
    }
  }
  if (threadIdx.x < dout) {
    out[(int64_t)w * dout + threadIdx.x] = as;
    out[(int64_t)w * dout + dout + threadIdx.x] = ad;
  }
}

// dout == 64 weight gradient on HMMA (3xTF32), cp.async double-buffered: the
// next tile's gathered h rows, d_z / z rows, ds and the self rows' dt land
// while this tile multiplies (the row indirections -- src_row for h, grouped
// -> rank for dt -- are resolved one tile further ahead). dW[c][j] += sum_r
// h[r][c] dz[r][j]: M = c (MB blocks of 16), N = j (warp = n-block of 8),
// K = the tile's 32 rows. Same partial layout as k_gat_bwd_param.
__device__ __forceinline__ void cp_async4g(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

template <int MB>
__global__ void __launch_bounds__(256, 2) k_gat_wgrad_mma(const SgMeta* __restrict__ meta, BParamArgs a) {
  // W^T staging and the K-padding zeros run before the PDL wait (parameters only)
  constexpr int D = 64, DZP = D + 8;
  constexpr int WP = ((16 * MB + 8 + 31) / 32 * 32 - 8) < 16 * MB ? (16 * MB + 8 + 31) / 32 * 32 + 24
                                                                   : (16 * MB + 8 + 31) / 32 * 32 - 8;
  extern __shared__ __align__(16) float smem[];
  const int w = a.w, H = a.heads, dh = D / H, w4 = w / 4;
  const int wt = w;  // W^T rows, float4-aligned (w % 4 == 0 on this path)
  const int stage_f = QTR * WP + QTR * DZP + QTR * D + 2 * QTR * H;
  float* Wt_s = smem;                                      // [D][w] (d_prev only)
  float* stg = Wt_s + (a.d_prev ? D * wt : 0);             // 2 x stage
  int* idx_s = reinterpret_cast<int*>(stg + 2 * stage_f);  // [2][2][QTR]: h row, dt row
  if (a.d_prev)
    for (int i = threadIdx.x; i < w * D; i += blockDim.x) {
      const int c = i / D, j = i - c * D;
      Wt_s[j * wt + c] = a.W[i];
    }
  for (int i = threadIdx.x; i < 2 * QTR * (WP - w); i += blockDim.x) {  // K padding columns stay zero
    const int r = i / (WP - w), c = w + (i - r * (WP - w));
    stg[(r / QTR) * stage_f + (r % QTR) * WP + c] = 0.f;
  }
  SG_PDL_ENTRY();
  const int l = a.l, d = a.d;
  const int n = meta->n_own[l - 1][d];
  const int own0 = meta->own_off[l - 1][d];
  const int ownl = meta->own_off[l][d];
  const int64_t nVl = meta->nV[l];
  const int ntiles = (n + QTR - 1) / QTR;
  const int G = gridDim.x;
  auto rows_of = [&](int tile, int& hr, int& tr) {  // thread < QTR: its tile row's h row and dt row
    hr = -1;
    tr = -1;
    const int r = tile * QTR + (int)threadIdx.x;
    if (tile >= ntiles || r >= n) return;
    const int g = own0 + r;
    hr = a.src_row ? a.src_row[g] : g;
    const int p = a.grouped[a.voff_lm1 + g];
    if (p < nVl) tr = ownl + a.rank[a.voff_l + p];
  };
  auto issue = [&](int tile, int b) {
    float* h_s = stg + b * stage_f;
    float* dz_s = h_s + QTR * WP;
    float* z_s = dz_s + QTR * DZP;
    float* ds_s = z_s + QTR * D;
    float* dt_s = ds_s + QTR * H;
    const int* hrow = idx_s + b * 2 * QTR;
    const int* trow = hrow + QTR;
    if (tile < ntiles) {
      const int r0 = tile * QTR;
      for (int i = threadIdx.x; i < QTR * w4; i += 256) {
        const int r = i / w4, q = i - r * w4;
        float* dst = h_s + r * WP + 4 * q;
        if (hrow[r] >= 0) cp_async16g(dst, a.h_prev + (int64_t)hrow[r] * w + 4 * q);
        else *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      for (int i = threadIdx.x; i < QTR * (D / 4); i += 256) {
        const int r = i / (D / 4), q = i - r * (D / 4);
        if (r0 + r < n) {
          const int64_t g = own0 + r0 + r;
          cp_async16g(dz_s + r * DZP + 4 * q, a.d_z + g * D + 4 * q);
          cp_async16g(z_s + r * D + 4 * q, a.z + g * D + 4 * q);
        } else {
          *reinterpret_cast<float4*>(dz_s + r * DZP + 4 * q) = make_float4(0.f, 0.f, 0.f, 0.f);
          *reinterpret_cast<float4*>(z_s + r * D + 4 * q) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      for (int i = threadIdx.x; i < QTR * H; i += 256) {
        const int r = i / H, hh = i - r * H;
        if (r0 + r < n) cp_async4g(ds_s + i, a.ds + (int64_t)(own0 + r0 + r) * H + hh);
        else ds_s[i] = 0.f;
        if (trow[r] >= 0) cp_async4g(dt_s + i, a.dt_tot + (int64_t)trow[r] * H + hh);
        else dt_s[i] = 0.f;
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  float acc[MB][4];
#pragma unroll
  for (int mb = 0; mb < MB; ++mb) acc[mb][0] = acc[mb][1] = acc[mb][2] = acc[mb][3] = 0.f;
  float as = 0.f, ad = 0.f;
  int hn = -1, tn = -1;
  if (threadIdx.x < QTR) {
    int h0, t0;
    rows_of(blockIdx.x, h0, t0);
    idx_s[threadIdx.x] = h0;
    idx_s[QTR + threadIdx.x] = t0;
    rows_of(blockIdx.x + G, hn, tn);
  }
  __syncthreads();
  issue(blockIdx.x, 0);
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, nb = threadIdx.x >> 5;
  for (int k = 0, tile = blockIdx.x; tile < ntiles; ++k, tile += G) {
    const int b = k & 1;
    if (threadIdx.x < QTR) {
      idx_s[(b ^ 1) * 2 * QTR + threadIdx.x] = hn;
      idx_s[(b ^ 1) * 2 * QTR + QTR + threadIdx.x] = tn;
    }
    __syncthreads();  // buffer b ^ 1 is free (tile k - 1 done) and its row indices visible
    issue(tile + G, b ^ 1);
    if (threadIdx.x < QTR) rows_of(tile + 2 * G, hn, tn);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();  // tile k landed
    const float* h_s = stg + b * stage_f;
    const float* dz_s = h_s + QTR * WP;
    const float* z_s = dz_s + QTR * DZP;
    const float* ds_s = z_s + QTR * D;
    const float* dt_s = ds_s + QTR * H;
#pragma unroll
    for (int k0 = 0; k0 < QTR; k0 += 8) {
      uint32_t bh0, bh1, bl0, bl1;
      split_tf32(dz_s[(k0 + t) * DZP + nb * 8 + g], bh0, bl0);
      split_tf32(dz_s[(k0 + t + 4) * DZP + nb * 8 + g], bh1, bl1);
#pragma unroll
      for (int mb = 0; mb < MB; ++mb) {
        const float* hr = h_s + mb * 16 + g;
        const float x[4] = {hr[(k0 + t) * WP], hr[(k0 + t) * WP + 8], hr[(k0 + t + 4) * WP],
                            hr[(k0 + t + 4) * WP + 8]};
        uint32_t ah[4], al[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) split_tf32(x[u], ah[u], al[u]);
        mma_tf32(acc[mb], al, bh0, bh1);
        mma_tf32(acc[mb], ah, bl0, bl1);
        mma_tf32(acc[mb], ah, bh0, bh1);
      }
    }
    if (threadIdx.x < D) {
      const int j = threadIdx.x, hh = j / dh;
#pragma unroll 8
      for (int rr = 0; rr < QTR; ++rr) {
        as = fmaf(z_s[rr * D + j], ds_s[rr * H + hh], as);
        ad = fmaf(z_s[rr * D + j], dt_s[rr * H + hh], ad);
      }
    }
    if (a.d_prev) {  // d_prev = d_z W^T: 4 columns per thread (one LDS.128 of W^T per j)
      const int nrow = min(QTR, n - tile * QTR);
      for (int i = threadIdx.x; i < nrow * w4; i += blockDim.x) {
        const int rr = i / w4, cg = i - rr * w4;
        float4 sacc = make_float4(0.f, 0.f, 0.f, 0.f);
        const float* dzr = dz_s + rr * DZP;
#pragma unroll 8
        for (int j = 0; j < D; ++j) {
          const float g = dzr[j];
          const float4 wv = *reinterpret_cast<const float4*>(Wt_s + j * wt + 4 * cg);
          sacc.x = fmaf(g, wv.x, sacc.x); sacc.y = fmaf(g, wv.y, sacc.y);
          sacc.z = fmaf(g, wv.z, sacc.z); sacc.w = fmaf(g, wv.w, sacc.w);
        }
        *reinterpret_cast<float4*>(a.d_prev + (int64_t)(own0 + tile * QTR + rr) * w + 4 * cg) = sacc;
      }
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  const int64_t ntot = (int64_t)w * D + 2 * D;
  float* out = a.partial + (int64_t)blockIdx.x * ntot;
#pragma unroll
  for (int mb = 0; mb < MB; ++mb) {
    const int m0 = mb * 16 + g, n0 = nb * 8 + 2 * t;
    if (m0 < w) {
      out[m0 * D + n0] = acc[mb][0];
      out[m0 * D + n0 + 1] = acc[mb][1];
    }
    if (m0 + 8 < w) {
      out[(m0 + 8) * D + n0] = acc[mb][2];
      out[(m0 + 8) * D + n0 + 1] = acc[mb][3];
    }
  }
  if (threadIdx.x < D) {
    out[(int64_t)w * D + threadIdx.x] = as;
    out[(int64_t)w * D + D + threadIdx.x] = ad;
  }
}

template <int MB>
int launch_wgrad_mma(const SgMeta* meta, const BParamArgs& a, int nblocks, cudaStream_t st) {
  constexpr int D = 64;
  constexpr int WP = ((16 * MB + 8 + 31) / 32 * 32 - 8) < 16 * MB ? (16 * MB + 8 + 31) / 32 * 32 + 24
                                                                   : (16 * MB + 8 + 31) / 32 * 32 - 8;
  const size_t stage_f = (size_t)QTR * WP + (size_t)QTR * (D + 8) + (size_t)QTR * D + 2 * (size_t)QTR * a.heads;
  const size_t smem = sizeof(float) * ((a.d_prev ? (size_t)D * a.w : 0) + 2 * stage_f) + sizeof(int) * 4 * QTR;
  if (smem > 227 * 1024) {
    set_error("gat_bwd_param: width too large for the MMA path");
    return SG_ERR_ARG;
  }
  SG_CUDA(allow_max_smem<k_gat_wgrad_mma<MB>>());
  ::sg::launch(k_gat_wgrad_mma<MB>, nblocks, 256, smem, st, meta, a);
  SG_CHECK_LAUNCH("k_gat_wgrad_mma");
  return SG_OK;
}

// ---------------------------------------------------------------- wide layers (dense.cu GEMMs)
// scores after a dense projection: s = z . a_src per head; t on self rows
__global__ void __launch_bounds__(256) k_gat_scores(const SgMeta* __restrict__ meta, ProjArgs a) {
  SG_PDL_ENTRY();
  const int H = a.heads, D = a.dout, dh = D / H;
  const int l = a.l, d = a.d;
  const int n = meta->n_own[l - 1][d];
  const int own0 = meta->own_off[l - 1][d], ownl = meta->own_off[l][d];
  const int64_t nVl = meta->nV[l];
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t item = gw; item < (int64_t)n * H; item += nw) {  // warp per (row, head)
    const int64_t r = item / H;
    const int hh = (int)(item - r * H);
    const int64_t G = own0 + r;
    const float* zr = a.z + G * D + hh * dh;
    float sv = 0.f, tv = 0.f;
    for (int j = lane; j < dh; j += 32) {
      sv = fmaf(zr[j], a.a_src[hh * dh + j], sv);
      tv = fmaf(zr[j], a.a_dst[hh * dh + j], tv);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      sv += __shfl_xor_sync(0xffffffffu, sv, o);
      tv += __shfl_xor_sync(0xffffffffu, tv, o);
    }
    if (lane == 0) {
      a.s[G * H + hh] = sv;
      const int p = a.grouped[a.voff_lm1 + G];
      if (p < nVl) a.t[(int64_t)(ownl + a.rank[a.voff_l + p]) * H + hh] = tv;
    }
  }
}

// per-split partials of da_src = sum_r z_r * ds_r(head), da_dst = sum_self z_r * dt(head)
// into partial[s][w*D .. w*D + 2D) (dW comes from dense_gemm_tn_partial)
__global__ void __launch_bounds__(256) k_gat_attn_partial(const SgMeta* __restrict__ meta, BParamArgs a,
                                                         int nsplit) {
  SG_PDL_ENTRY();
  const int D = a.dout, H = a.heads, dh = D / H, w = a.w;
  const int l = a.l, d = a.d;
  const int n = meta->n_own[l - 1][d];
  const int own0 = meta->own_off[l - 1][d], ownl = meta->own_off[l][d];
  const int64_t nVl = meta->nV[l];
  const int s = blockIdx.x;
  const int per = (n + nsplit - 1) / nsplit;
  const int rb = s * per, re = min(n, rb + per);
  float* out = a.partial + (int64_t)s * ((int64_t)w * D + 2 * D) + (int64_t)w * D;
  for (int j = threadIdx.x; j < D; j += blockDim.x) {
    const int hh = j / dh;
    float as = 0.f, ad = 0.f;
    for (int r = rb; r < re; ++r) {
      const int64_t G = own0 + r;
      const float zv = a.z[G * D + j];
      as = fmaf(zv, a.ds[G * H + hh], as);
      const int p = a.grouped[a.voff_lm1 + G];
      if (p < nVl) ad = fmaf(zv, a.dt_tot[(int64_t)(ownl + a.rank[a.voff_l + p]) * H + hh], ad);
    }
    out[j] = as;
    out[D + j] = ad;
  }
}

// ---------------------------------------------------------------- dispatch helpers
// Team shape from (D, H): LPR lanes span D (a power of two, multiple of H),
// EG edge groups fill the team to 8..32 lanes.
#define GAT_TEAM_DISPATCH(KERNEL, DOUT, HEADS, GRIDROWS, ST, ...)                          \
  do {                                                                                    \
    const int dd_ = (DOUT), hh_ = (HEADS);                                                \
    auto go_ = [&](auto vec_, auto lpr_, auto eg_) {                                      \
      constexpr int VEC_ = decltype(vec_)::value, LPR_ = decltype(lpr_)::value,           \
                    EG_ = decltype(eg_)::value;                                           \
      constexpr int RPB_ = 8 * (32 / (LPR_ * EG_));                                       \
      const int grid_ = clamp_grid(div_up((GRIDROWS), RPB_), kSMs * 8);                   \
      ::sg::launch(KERNEL<VEC_, LPR_, EG_>, grid_, 256, 0, ST, __VA_ARGS__);                        \
    };                                                                                    \
    using I1 = std::integral_constant<int, 1>;                                            \
    using I2 = std::integral_constant<int, 2>;                                            \
    using I4 = std::integral_constant<int, 4>;                                            \
    using I8 = std::integral_constant<int, 8>;                                            \
    using I16 = std::integral_constant<int, 16>;                                          \
    using I32 = std::integral_constant<int, 32>;                                          \
    const int q_ = dd_ / (4 * hh_);                                                       \
    const bool v4_ = dd_ % (4 * hh_) == 0 && (q_ & (q_ - 1)) == 0 && (hh_ & (hh_ - 1)) == 0; \
    if (v4_ && dd_ <= 4) go_(I4(), I1(), I8());                                           \
    else if (v4_ && dd_ <= 8) go_(I4(), I2(), I8());                                      \
    else if (v4_ && dd_ <= 16) go_(I4(), I4(), I4());                                     \
    else if (v4_ && dd_ <= 32) go_(I4(), I8(), I2());                                     \
    else if (v4_ && dd_ <= 64) go_(I4(), I16(), I2());                                    \
    else if (v4_ && dd_ <= 128) go_(I4(), I32(), I1());                                   \
    else if (hh_ == 1 && dd_ <= 4) go_(I1(), I4(), I4());                                 \
    else if (hh_ == 1 && dd_ <= 8) go_(I1(), I8(), I2());                                 \
    else if (hh_ == 1 && dd_ <= 16) go_(I1(), I16(), I2());                               \
    else if (hh_ == 1 && dd_ <= 32) go_(I1(), I32(), I1());                               \
    else {                                                                                \
      set_error("gat: unsupported width/heads (multi-head needs power-of-two heads and "  \
                "d_head/4, D <= 128; one head: D <= 128)");                               \
      return SG_ERR_ARG;                                                                  \
    }                                                                                     \
  } while (0)

// ---------------------------------------------------------------- layer-1 weight gradient, destination-centric
// At layer 1 nothing needs d(loss)/d(h0), only dW, da_src, da_dst. Per source
// row u the reference gradient is (engine.py:480-552)
//   dz_u = sum_{e=(u->v)} alpha_e (.) dn_v + ds_u a_src + [u = self(v)] dt_v a_dst,
//   ds_u = sum_e dpre_e,   dW = sum_u h_u^T dz_u,
//   da_src = sum_u ds_u z_u,   da_dst = sum_v dt_v z_self(v),   z = h W.
// All of it is linear in the edges, so it regroups by DESTINATION:
//   dW^(h) = sum_v A_v^(h)T dn_v^(h) + SB^(h) (x) a_src^(h) + SC^(h) (x) a_dst^(h),
//   A_v^(h) = sum_{u in N(v)} alpha_uv^(h) h_u,   SB^(h) = sum_v sum_u dpre_uv^(h) h_u,
//   SC^(h) = sum_v dt_v^(h) h_self(v),   da_src^(h) = SB^(h) W^(h),  da_dst^(h) = SC^(h) W^(h).
// One pass over each destination's in-edges (the forward's CSR-by-destination,
// no sort by source), h rows gathered once per edge, no d_z / ds / dt_tot
// round trip through HBM; replaces k_gat_bwd_src + the weight-gradient kernel
// at layer 1. Warp per destination row (lanes own 4 columns of h), TM = 8 rows
// per tile; per tile the A / B / h_self / dt / dn rows go to shared memory,
// then dW (shared, 4x4 register blocks) += A^T dn and SB / SC += column sums.
// Per-CTA partials in the k_gat_bwd_param layout [dW | da_src | da_dst].
struct WdArgs {
  int d, w, heads, stride, g;
  int64_t eoff_li, rbase_li, pbase_l, voff_l;
  const int32_t* rowbeg;
  const int32_t* rowend;
  const int32_t* lsrc;
  const int32_t* dperm;
  const int32_t* sendpos;
  const int32_t* selfrow;
  const int32_t* contrib;
  const int32_t* src_row;
  const float* h0;        // feature table [rows][w]
  const float* alpha;     // [edge][head]
  const float* d_pre;     // [edge][head]
  const float* dnc;       // owned rows, stride D + H
  const float* dnc_recv;  // pair layout, stride `stride`
  const float* dt_loc;    // [row][head]
  const float* dt_recv;   // receive layout, stride H
  const float* W;         // [w][D]
  const float* a_src;     // [D]
  const float* a_dst;
  float* partial;
};

constexpr int WD_D = 64;
constexpr int WD_RPW = 2;          // destination rows per warp per tile (measured: 4 -> 0.479 vs 0.456 ms C3)
constexpr int WD_TM = 8 * WD_RPW;  // rows per tile: 16 (65 KB shared, 3 CTAs / SM)

template <int H>
__global__ void __launch_bounds__(256, 3) k_gat_wgrad_dst(const SgMeta* __restrict__ meta, WdArgs a) {
  // (the shared accumulators are zeroed before the PDL wait)
  constexpr int D = WD_D, DH = D / H, TM = WD_TM, RPW = WD_RPW;
  extern __shared__ __align__(16) float sm[];
  const int w = a.w, d = a.d;
  const int HW = H * w;
  float* dW_s = sm;                    // [w][D]
  float* SB_s = dW_s + w * D;          // [H][w]
  float* SC_s = SB_s + HW;             // [H][w]
  float* A_s = SC_s + HW;              // [TM][H][w]
  float* hs_s = A_s + TM * HW;         // [TM][w]
  float* dn_s = hs_s + TM * w;         // [TM][D]
  float* dt_s = dn_s + TM * D;         // [TM][H]
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int i = tid; i < w * D + 2 * HW; i += 256) sm[i] = 0.f;
  SG_PDL_ENTRY();
  const int l = 1;
  const int n_own = meta->n_own[l][d];
  const int R = n_own + meta->n_ref[l][d];
  const int own0 = meta->own_off[l][d], ref0 = meta->ref_off[l][d];
  const int prev0 = meta->own_off[l - 1][d];
  const int64_t rb = a.rbase_li + own0 + ref0;
  const int col = 4 * lane;
  const bool colok = col < w;
  const int nslots = (w / 4) * (D / 4);
  const int ntiles = (R + TM - 1) / TM;
  auto edge_x = [&](int j) -> int64_t { return a.dperm ? (int64_t)a.dperm[j] : a.eoff_li + j; };
  auto ld_h = [&](int r) -> float4 {
    return colok ? __ldg(reinterpret_cast<const float4*>(a.h0 + (int64_t)r * w + col))
                 : make_float4(0.f, 0.f, 0.f, 0.f);
  };
  auto ld_e = [&](const float* base, int64_t x) -> float4 {  // the edge's H values (warp-uniform address)
    if (H == 4) return __ldg(reinterpret_cast<const float4*>(base + x * 4));
    float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
    t.x = base[x * H];
    if (H > 1) t.y = base[x * H + 1];
    return t;
  };
  // B = sum_e dpre_e h_u only enters through its total SB: this lane's running part
  float4 B[H];
#pragma unroll
  for (int h = 0; h < H; ++h) B[h] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int q0 = tile * TM + wid * RPW;
    // row bounds of this warp's RPW rows; the first row's index chain
    int be = 0;
    if (lane < 2 * RPW && q0 + (lane >> 1) < R)
      be = (lane & 1) ? a.rowend[rb + q0 + (lane >> 1)] : a.rowbeg[rb + q0 + (lane >> 1)];
    int b = __shfl_sync(0xffffffffu, be, 0), e = __shfl_sync(0xffffffffu, be, 1);
    int xn = 0, hn = 0, un = 0;
    if (q0 < R && lane < e - b) {
      xn = (int)edge_x(b + lane);
      un = prev0 + a.lsrc[xn];
      hn = a.src_row ? a.src_row[un] : un;
    }
    __syncthreads();  // the previous tile's pass is done with the tile buffers
    for (int i = 0; i < RPW; ++i) {
      const int q = q0 + i;
      const int rr = wid * RPW + i;  // tile row
      float4 A[H];
#pragma unroll
      for (int h = 0; h < H; ++h) A[h] = make_float4(0.f, 0.f, 0.f, 0.f);
      float4 hs = make_float4(0.f, 0.f, 0.f, 0.f);
      float dn_v = 0.f, dn_v2 = 0.f, dt_v = 0.f;
      if (q < R) {  // warp-uniform
        const int xc = xn, hc = hn, bc = b, ec = e;
        // next row's bounds + first index hop, issued before this row's loads
        int nb = 0, ne = 0;
        const bool more = i + 1 < RPW && q + 1 < R;
        if (more) {
          nb = __shfl_sync(0xffffffffu, be, 2 * (i + 1));
          ne = __shfl_sync(0xffffffffu, be, 2 * (i + 1) + 1);
          if (lane < ne - nb) {
            xn = (int)edge_x(nb + lane);
            un = prev0 + a.lsrc[xn];
          }
        }
        const bool own = q < n_own;
        const float* dn_row = own ? a.dnc + (int64_t)(own0 + q) * (D + H)
                                  : a.dnc_recv + (int64_t)a.sendpos[a.pbase_l + ref0 + (q - n_own)] * a.stride;
        dn_v = dn_row[lane];
        dn_v2 = dn_row[lane + 32];
        if (own) {
          const int64_t G = own0 + q;
          int rs = prev0 + a.selfrow[a.voff_l + G];
          if (a.src_row) rs = a.src_row[rs];
          hs = ld_h(rs);
          if (lane < H) {
            dt_v = a.dt_loc[G * H + lane];
            if (a.g > 1) {
              const int* cb = a.contrib + (int64_t)a.g * a.voff_l + G * a.g;
              for (int s2 = 0; s2 < a.g; ++s2) {
                const int r2 = cb[s2];
                if (r2 >= 0) dt_v += a.dt_recv[(int64_t)r2 * H + lane];
              }
            }
          }
        }
        // one edge: A += alpha h_u, B += dpre h_u
        // alpha / d_pre of the row's first 32 edges, one edge per lane (coalesced),
        // handed to every lane by shuffles as the edges are applied
        const float4 al_l = lane < ec - bc ? ld_e(a.alpha, xc) : make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 dp_l = lane < ec - bc ? ld_e(a.d_pre, xc) : make_float4(0.f, 0.f, 0.f, 0.f);
        auto edge_k = [&](const float4& v, int k) {  // edge k < 32 of the row (k warp-uniform)
          float alh[4], dph[4];
          alh[0] = __shfl_sync(0xffffffffu, al_l.x, k); dph[0] = __shfl_sync(0xffffffffu, dp_l.x, k);
          if (H > 1) { alh[1] = __shfl_sync(0xffffffffu, al_l.y, k); dph[1] = __shfl_sync(0xffffffffu, dp_l.y, k); }
          if (H > 2) {
            alh[2] = __shfl_sync(0xffffffffu, al_l.z, k); dph[2] = __shfl_sync(0xffffffffu, dp_l.z, k);
            alh[3] = __shfl_sync(0xffffffffu, al_l.w, k); dph[3] = __shfl_sync(0xffffffffu, dp_l.w, k);
          }
#pragma unroll
          for (int h = 0; h < H; ++h) {
            A[h].x = fmaf(alh[h], v.x, A[h].x); A[h].y = fmaf(alh[h], v.y, A[h].y);
            A[h].z = fmaf(alh[h], v.z, A[h].z); A[h].w = fmaf(alh[h], v.w, A[h].w);
            B[h].x = fmaf(dph[h], v.x, B[h].x); B[h].y = fmaf(dph[h], v.y, B[h].y);
            B[h].z = fmaf(dph[h], v.z, B[h].z); B[h].w = fmaf(dph[h], v.w, B[h].w);
          }
        };
        auto edge = [&](const float4& v, int64_t x) {
          const float4 al = ld_e(a.alpha, x), dp = ld_e(a.d_pre, x);
          const float alh[4] = {al.x, al.y, al.z, al.w}, dph[4] = {dp.x, dp.y, dp.z, dp.w};
#pragma unroll
          for (int h = 0; h < H; ++h) {
            A[h].x = fmaf(alh[h], v.x, A[h].x); A[h].y = fmaf(alh[h], v.y, A[h].y);
            A[h].z = fmaf(alh[h], v.z, A[h].z); A[h].w = fmaf(alh[h], v.w, A[h].w);
            B[h].x = fmaf(dph[h], v.x, B[h].x); B[h].y = fmaf(dph[h], v.y, B[h].y);
            B[h].z = fmaf(dph[h], v.z, B[h].z); B[h].w = fmaf(dph[h], v.w, B[h].w);
          }
        };
        const int cnt0 = min(32, ec - bc);
        for (int k0 = 0; k0 < cnt0; k0 += 4) {  // warp-uniform trip count
          float4 v[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int k = min(k0 + t, 31);
            const int r = __shfl_sync(0xffffffffu, hc, k);
            v[t] = (k0 + t < cnt0) ? ld_h(r) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int t = 0; t < 4; ++t)
            if (k0 + t < cnt0) edge_k(v[t], k0 + t);
        }
        // rows with more than 32 in-edges: the remaining edges, one at a time (rare)
        for (int j = bc + 32; j < ec; ++j) {
          const int64_t x = edge_x(j);
          const int u = prev0 + a.lsrc[x];
          edge(ld_h(a.src_row ? a.src_row[u] : u), x);
        }
        // second index hop of the next row, overlapping this row's tail
        if (more) {
          hn = (lane < ne - nb) ? (a.src_row ? a.src_row[un] : un) : 0;
          b = nb;
          e = ne;
        }
      }
      if (colok) {
#pragma unroll
        for (int h = 0; h < H; ++h) *reinterpret_cast<float4*>(A_s + (rr * H + h) * w + col) = A[h];
        *reinterpret_cast<float4*>(hs_s + rr * w + col) = hs;
      }
      dn_s[rr * D + lane] = dn_v;
      dn_s[rr * D + lane + 32] = dn_v2;
      if (lane < H) dt_s[rr * H + lane] = dt_v;
    }
    __syncthreads();
    // dW += A^T dn (4x4 blocks: c-group cg of w, j-group jg of D; head of jg)
    for (int s2 = tid; s2 < nslots; s2 += 256) {
      const int cg = s2 / (D / 4), jg = s2 - cg * (D / 4);
      const int hh = (4 * jg) / DH;
      float acc[16];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float4 t4 = *reinterpret_cast<const float4*>(dW_s + (4 * cg + i) * D + 4 * jg);
        acc[4 * i] = t4.x; acc[4 * i + 1] = t4.y; acc[4 * i + 2] = t4.z; acc[4 * i + 3] = t4.w;
      }
#pragma unroll
      for (int r = 0; r < TM; ++r) {
        const float4 a4 = *reinterpret_cast<const float4*>(A_s + (r * H + hh) * w + 4 * cg);
        const float4 g4 = *reinterpret_cast<const float4*>(dn_s + r * D + 4 * jg);
        const float av[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          acc[4 * i + 0] = fmaf(av[i], g4.x, acc[4 * i + 0]);
          acc[4 * i + 1] = fmaf(av[i], g4.y, acc[4 * i + 1]);
          acc[4 * i + 2] = fmaf(av[i], g4.z, acc[4 * i + 2]);
          acc[4 * i + 3] = fmaf(av[i], g4.w, acc[4 * i + 3]);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
        *reinterpret_cast<float4*>(dW_s + (4 * cg + i) * D + 4 * jg) =
            make_float4(acc[4 * i], acc[4 * i + 1], acc[4 * i + 2], acc[4 * i + 3]);
    }
    // SC += dt-weighted column sums of h_self
    for (int idx = tid; idx < HW; idx += 256) {
      const int hh = idx / w, c = idx - hh * w;
      float sc = SC_s[idx];
#pragma unroll
      for (int r = 0; r < TM; ++r) sc = fmaf(dt_s[r * H + hh], hs_s[r * w + c], sc);
      SC_s[idx] = sc;
    }
  }
  // SB = the warps' running B parts, summed in warp order (A_s is free now)
  __syncthreads();
  if (colok) {
#pragma unroll
    for (int h = 0; h < H; ++h) *reinterpret_cast<float4*>(A_s + (wid * H + h) * w + col) = B[h];
  }
  __syncthreads();
  for (int idx = tid; idx < HW; idx += 256) {
    float sb = 0.f;
#pragma unroll
    for (int ww = 0; ww < 8; ++ww) sb += A_s[ww * HW + idx];
    SB_s[idx] = sb;
  }
  __syncthreads();
  // dW^(h) += SB^(h) (x) a_src^(h) + SC^(h) (x) a_dst^(h); da = S W (per head)
  float* out = a.partial + (int64_t)blockIdx.x * ((int64_t)w * D + 2 * D);
  for (int idx = tid; idx < w * D; idx += 256) {
    const int c = idx / D, j = idx - c * D, hh = j / DH;
    out[idx] = dW_s[idx] + SB_s[hh * w + c] * a.a_src[j] + SC_s[hh * w + c] * a.a_dst[j];
  }
  if (tid < 2 * D) {
    const int j = tid & (D - 1), hh = j / DH;
    const float* S = (tid < D ? SB_s : SC_s) + hh * w;
    float v = 0.f;
    for (int c = 0; c < w; ++c) v = fmaf(S[c], a.W[c * D + j], v);
    out[(int64_t)w * D + tid] = v;
  }
}

}  // namespace

#define SPLIT_PTRS                                                     \
  const char* base = (const char*)split_ws;                           \
  const SgSplitLayout& y = *lay;                                       \
  const SgMeta* meta = (const SgMeta*)(base + y.o_meta);               \
  auto I32p = [&](int64_t o) { return (const int32_t*)(base + o); };

#define GAT_HEADS_CHECK(dout, heads)                                              \
  SG_REQUIRE((heads) >= 1 && (dout) % (heads) == 0, "gat: dout must be a multiple of heads")

extern "C" int sg_gat_project(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                              const float* h_prev, const int32_t* src_row, int32_t w, int32_t dout,
                              int32_t heads, const float* W, const float* a_src, const float* a_dst,
                              float* z, float* s, float* t, int64_t max_rows, void* stream) {
  SG_REQUIRE(split_ws && lay, "gat_project: null workspace");
  SPLIT_PTRS
  SG_REQUIRE(l >= 1 && l <= y.L && d >= 0 && d < y.g, "gat_project: bad layer/device");
  GAT_HEADS_CHECK(dout, heads);
  if (max_rows <= 0) return SG_OK;
  ProjArgs a;
  memset(&a, 0, sizeof(a));
  a.l = l; a.d = d; a.w = w; a.dout = dout; a.heads = heads;
  a.voff_lm1 = y.voff[l - 1];
  a.voff_l = y.voff[l];
  a.h_prev = h_prev; a.src_row = src_row;
  a.grouped = I32p(y.o_grouped);
  a.rank = I32p(y.o_rank);
  a.W = W; a.a_src = a_src; a.a_dst = a_dst;
  a.z = z; a.s = s; a.t = t;
  const size_t smem = sizeof(float) * ((size_t)w * dout + (size_t)PTR * (w + 1) + (size_t)PTR * (dout + 1) + PTR);
  cudaStream_t st = (cudaStream_t)stream;
  const int nq = dout / 4;
  static const bool use_mma = !getenv("SG_NO_MMA");
  static const bool use_tc5 = !getenv("SG_NO_TC05");
  const int dh = dout / heads;
  if (use_mma && use_tc5 && dout == tc5::N && w % 4 == 0 && w > 32 && w <= tc5::KMAX &&
      (dh == 8 || dh == 16 || dh == 32)) {
    // tcgen05 (TMEM accumulator) 3xTF32 projection, one CTA per SM
    const int grid = clamp_grid(div_up(max_rows, tc5::M), kSMs);
    switch (dh) {
#define TC_CASE(DD)                                                             \
  case DD:                                                                      \
    SG_CUDA(allow_max_smem<k_gat_project_tc<DD>>());                            \
    ::sg::launch(k_gat_project_tc<DD>, grid, 256, tc5::SMEM, st, meta, a);      \
    break;
      TC_CASE(8) TC_CASE(16) TC_CASE(32)
#undef TC_CASE
    }
    SG_CHECK_LAUNCH("k_gat_project_tc");
    return SG_OK;
  }
  if (use_mma && w % 4 == 0 && w > 32 && w <= 256 && (dout == 32 || dout == 64 || dout == 128)) {
    // tensor-core path (3xTF32 HMMA) for the wide layer-1 projection
    const int KPAD = (w + 7) & ~7;
    const size_t smem_m = sizeof(float) * ((size_t)KPAD * (dout + 8) + 2 * 32 * (size_t)(KPAD + 4) +
                                           32 * (size_t)dout) + 2 * 32 * 4;
    if (smem_m <= 227 * 1024) {
      const int per_sm = std::max<int>(1, std::min<int>(4, (int)((228 * 1024) / (smem_m + 1024))));
      const int grid_m = clamp_grid(div_up(max_rows, 32), kSMs * per_sm);
      cudaError_t attr = cudaSuccess;
      switch (dout) {
#define GM_CASE(DD, NT)                                              \
  case DD:                                                           \
    attr = allow_max_smem<k_gat_project_mma<NT>>();                  \
    SG_CUDA(attr);                                                   \
    ::sg::launch(k_gat_project_mma<NT>, grid_m, 256, smem_m, st, meta, a); \
    break;
        GM_CASE(32, 1) GM_CASE(64, 2) GM_CASE(128, 4)
#undef GM_CASE
      }
      SG_CHECK_LAUNCH("k_gat_project_mma");
      return SG_OK;
    }
  }
  if (w % 4 == 0 && w <= 128 && dout % 4 == 0 && nq <= 32 && (nq & (nq - 1)) == 0) {
    // register-tiled path: 4x4 tiles, K split over slices (TM = 32 rows per tile)
    const int NS = 256 / (8 * nq);
    const size_t smem_t = sizeof(float) * ((size_t)w * dout + (size_t)w * 36 + (size_t)NS * 32 * dout) + 32 * 4;
    const int grid_t = clamp_grid(div_up(max_rows, 32), kSMs * 8);
    cudaError_t attr = cudaSuccess;
    switch (nq) {
#define GP_CASE(Q)                                                   \
  case Q:                                                            \
    attr = allow_max_smem<k_gat_project_tiled<Q>>();                 \
    SG_CUDA(attr);                                                   \
    ::sg::launch(k_gat_project_tiled<Q>, grid_t, 256, smem_t, st, meta, a);    \
    break;
      GP_CASE(1) GP_CASE(2) GP_CASE(4) GP_CASE(8) GP_CASE(16) GP_CASE(32)
#undef GP_CASE
    }
    SG_CHECK_LAUNCH("k_gat_project_tiled");
    return SG_OK;
  }
  if (smem > 227 * 1024) {
    // wide layer: z = h_prev[rows] W as a dense GEMM, then the per-head scores
    GemmArgs g;
    memset(&g, 0, sizeof(g));
    g.R_dev = &meta->n_own[l - 1][d];
    g.K = w; g.N = dout; g.A = h_prev; g.lda = w;
    g.ar.mode = src_row ? 1 : 0; g.ar.map = src_row; g.ar.base_dev = &meta->own_off[l - 1][d];
    g.B = W; g.ldb = dout; g.C = z; g.ldc = dout; g.c_base_dev = &meta->own_off[l - 1][d];
    int rc = dense_gemm_rows(g, max_rows, st);
    if (rc) return rc;
    ::sg::launch(k_gat_scores, clamp_grid(div_up(max_rows * heads, 8), kSMs * 8), 256, 0, st, meta, a);
    SG_CHECK_LAUNCH("k_gat_scores");
    return SG_OK;
  }
  const int grid = clamp_grid(div_up(max_rows, PTR), kSMs * 4);
  if (dout % 4 == 0) {
    SG_CUDA(allow_max_smem<k_gat_project<true>>());
    ::sg::launch(k_gat_project<true>, grid, 256, smem, st, meta, a);
  } else {
    SG_CUDA(allow_max_smem<k_gat_project<false>>());
    ::sg::launch(k_gat_project<false>, grid, 256, smem, st, meta, a);
  }
  SG_CHECK_LAUNCH("k_gat_project");
  return SG_OK;
}

extern "C" int sg_gat_agg(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                          int32_t dout, int32_t heads, float slope, const float* z, const float* s,
                          const float* t, const float* t_recv, const int32_t* dperm, float* pre_e,
                          float* loc_m, float* loc_s, float* loc_U, float* sendbuf,
                          int32_t send_stride, int64_t max_rows, void* stream) {
  SG_REQUIRE(split_ws && lay, "gat_agg: null workspace");
  SPLIT_PTRS
  SG_REQUIRE(l >= 1 && l <= y.L && d >= 0 && d < y.g, "gat_agg: bad layer/device");
  GAT_HEADS_CHECK(dout, heads);
  SG_REQUIRE(send_stride >= dout + 2 * heads || y.g == 1, "gat_agg: send stride < D+2H");
  if (max_rows <= 0) return SG_OK;
  AggArgs a;
  memset(&a, 0, sizeof(a));
  a.l = l; a.d = d; a.dout = dout; a.heads = heads; a.stride = send_stride; a.slope = slope;
  a.eoff_li = y.eoff[l - 1]; a.rbase_li = y.rbase[l - 1]; a.pbase_l = y.pbase[l];
  a.rowbeg = I32p(y.o_rowbeg); a.rowend = I32p(y.o_rowend); a.lsrc = I32p(y.o_lsrc);
  a.dperm = dperm; a.sendpos = I32p(y.o_sendpos);
  a.z = z; a.s = s; a.t = t; a.t_recv = t_recv;
  a.pre_e = pre_e; a.loc_m = loc_m; a.loc_s = loc_s; a.loc_U = loc_U; a.sendbuf = sendbuf;
  cudaStream_t st = (cudaStream_t)stream;
  GAT_TEAM_DISPATCH(k_gat_agg, dout, heads, max_rows, st, meta, a);
  SG_CHECK_LAUNCH("k_gat_agg");
  return SG_OK;
}

// sg_gat_agg with the owner combine and alpha folded in (one device: every
// row is owned, no holder partials): writes md, num, h and alpha directly.
extern "C" int sg_gat_agg_fused(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t dout,
                                int32_t heads, float slope, const float* z, const float* s, const float* t,
                                const int32_t* dperm, float* pre_e, int32_t final_layer, float* md, float* num,
                                float* h, float* alpha, int64_t max_rows, void* stream) {
  SG_REQUIRE(split_ws && lay && z && s && t && pre_e && md && num && h && alpha, "gat_agg_fused: null argument");
  SPLIT_PTRS
  SG_REQUIRE(y.g == 1 && l >= 1 && l <= y.L, "gat_agg_fused: one device only (no holders to combine)");
  GAT_HEADS_CHECK(dout, heads);
  if (max_rows <= 0) return SG_OK;
  AggArgs a;
  memset(&a, 0, sizeof(a));
  a.l = l; a.d = 0; a.dout = dout; a.heads = heads; a.stride = 0; a.slope = slope;
  a.eoff_li = y.eoff[l - 1]; a.rbase_li = y.rbase[l - 1]; a.pbase_l = y.pbase[l];
  a.rowbeg = I32p(y.o_rowbeg); a.rowend = I32p(y.o_rowend); a.lsrc = I32p(y.o_lsrc);
  a.dperm = dperm; a.sendpos = I32p(y.o_sendpos);
  a.z = z; a.s = s; a.t = t; a.pre_e = pre_e;
  a.fuse = 1; a.final_ = final_layer; a.md = md; a.num = num; a.h = h; a.alpha = alpha;
  cudaStream_t st = (cudaStream_t)stream;
  GAT_TEAM_DISPATCH(k_gat_agg, dout, heads, max_rows, st, meta, a);
  SG_CHECK_LAUNCH("k_gat_agg(fused)");
  return SG_OK;
}

extern "C" int sg_gat_combine(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                              int32_t dout, int32_t heads, const float* loc_m, const float* loc_s,
                              const float* loc_U, const float* recv, int32_t recv_stride,
                              int32_t final_layer, float* md, float* num, float* h,
                              int64_t max_rows, void* stream) {
  SG_REQUIRE(split_ws && lay, "gat_combine: null workspace");
  SPLIT_PTRS
  SG_REQUIRE(l >= 1 && l <= y.L && d >= 0 && d < y.g, "gat_combine: bad layer/device");
  GAT_HEADS_CHECK(dout, heads);
  if (max_rows <= 0) return SG_OK;
  CombArgs a;
  memset(&a, 0, sizeof(a));
  a.l = l; a.d = d; a.dout = dout; a.heads = heads; a.g = y.g; a.stride = recv_stride;
  a.final_ = final_layer;
  a.voff_l = y.voff[l]; a.contrib = I32p(y.o_contrib);
  a.loc_m = loc_m; a.loc_s = loc_s; a.loc_U = loc_U; a.recv = recv; a.md = md; a.num = num; a.h = h;
  ::sg::launch(k_gat_combine, clamp_grid(div_up(max_rows * dout, 256), kSMs * 8), 256, 0, (cudaStream_t)stream, meta, a);
  SG_CHECK_LAUNCH("k_gat_combine");
  return SG_OK;
}

extern "C" int sg_gat_alpha(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                            int32_t heads, float slope, const float* pre_e, const float* md,
                            const float* md_recv, float* alpha, int64_t max_edges, void* stream) {
  SG_REQUIRE(split_ws && lay, "gat_alpha: null workspace");
  SPLIT_PTRS
  SG_REQUIRE(l >= 1 && l <= y.L && d >= 0 && d < y.g, "gat_alpha: bad layer/device");
  if (max_edges <= 0) return SG_OK;
  AlphaArgs a;
  memset(&a, 0, sizeof(a));
  a.l = l; a.d = d; a.heads = heads; a.slope = slope; a.eoff_li = y.eoff[l - 1]; a.pbase_l = y.pbase[l];
  a.ldst = I32p(y.o_ldst); a.sendpos = I32p(y.o_sendpos);
  a.pre_e = pre_e; a.md = md; a.md_recv = md_recv; a.alpha = alpha;
  ::sg::launch(k_gat_alpha, clamp_grid(div_up(max_edges * heads, 256), kSMs * 8), 256, 0, (cudaStream_t)stream, meta, a);
  SG_CHECK_LAUNCH("k_gat_alpha");
  return SG_OK;
}

extern "C" int sg_gat_bwd_rows(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                               int32_t dout, int32_t heads, const float* d_h, const float* num,
                               int32_t final_layer, float* dnc, int64_t max_rows, void* stream) {
  SG_REQUIRE(split_ws && lay, "gat_bwd_rows: null workspace");
  SPLIT_PTRS
  GAT_HEADS_CHECK(dout, heads);
  if (max_rows <= 0) return SG_OK;
  BRowsArgs a{l, d, dout, heads, final_layer, d_h, num, dnc};
  const int dh = dout / heads;
  if (dh % 4 == 0 && dh <= 128 && ((dh / 4) & (dh / 4 - 1)) == 0) {
    const int grid = clamp_grid(div_up(max_rows * (dout / 4), 256), kSMs * 8);
    cudaStream_t st = (cudaStream_t)stream;
    switch (dh / 4) {
      case 1: ::sg::launch(k_gat_bwd_rows4<1>, grid, 256, 0, st, meta, a); break;
      case 2: ::sg::launch(k_gat_bwd_rows4<2>, grid, 256, 0, st, meta, a); break;
      case 4: ::sg::launch(k_gat_bwd_rows4<4>, grid, 256, 0, st, meta, a); break;
      case 8: ::sg::launch(k_gat_bwd_rows4<8>, grid, 256, 0, st, meta, a); break;
      case 16: ::sg::launch(k_gat_bwd_rows4<16>, grid, 256, 0, st, meta, a); break;
      default: ::sg::launch(k_gat_bwd_rows4<32>, grid, 256, 0, st, meta, a); break;
    }
    SG_CHECK_LAUNCH("k_gat_bwd_rows4");
    return SG_OK;
  }
  ::sg::launch(k_gat_bwd_rows, clamp_grid(div_up(max_rows * heads, 256), kSMs * 4), 256, 0, (cudaStream_t)stream, meta, a);
  SG_CHECK_LAUNCH("k_gat_bwd_rows");
  return SG_OK;
}

extern "C" int sg_gat_bwd_dst(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                              int32_t dout, int32_t heads, float slope, const float* z,
                              const float* alpha, const float* pre_e, const float* dnc,
                              const float* dnc_recv, int32_t recv_stride, const int32_t* dperm,
                              float* d_pre, float* dt_loc, float* sendbuf, int64_t max_rows,
                              void* stream) {
  SG_REQUIRE(split_ws && lay, "gat_bwd_dst: null workspace");
  SPLIT_PTRS
  GAT_HEADS_CHECK(dout, heads);
  if (max_rows <= 0) return SG_OK;
  BDstArgs a;
  memset(&a, 0, sizeof(a));
  a.l = l; a.d = d; a.dout = dout; a.heads = heads; a.stride = recv_stride; a.slope = slope;
  a.eoff_li = y.eoff[l - 1]; a.rbase_li = y.rbase[l - 1]; a.pbase_l = y.pbase[l];
  a.rowbeg = I32p(y.o_rowbeg); a.rowend = I32p(y.o_rowend); a.lsrc = I32p(y.o_lsrc);
  a.dperm = dperm; a.sendpos = I32p(y.o_sendpos);
  a.z = z; a.alpha = alpha; a.pre_e = pre_e; a.dnc = dnc; a.dnc_recv = dnc_recv;
  a.d_pre = d_pre; a.dt_loc = dt_loc; a.sendbuf = sendbuf;
  cudaStream_t st = (cudaStream_t)stream;
  GAT_TEAM_DISPATCH(k_gat_bwd_dst, dout, heads, max_rows, st, meta, a);
  SG_CHECK_LAUNCH("k_gat_bwd_dst");
  return SG_OK;
}

extern "C" int sg_gat_bwd_src(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                              int32_t dout, int32_t heads, const int32_t* perm, const int32_t* srcbeg,
                              const int32_t* srcend, int64_t key_base, const float* alpha,
                              const float* d_pre, const float* dnc, const float* dnc_recv,
                              int32_t dnc_stride, const float* dt_loc, const float* dt_recv,
                              const float* a_src, const float* a_dst, float* d_z, float* ds,
                              float* dt_tot, int64_t max_rows, void* stream) {
  SG_REQUIRE(split_ws && lay, "gat_bwd_src: null workspace");
  SPLIT_PTRS
  GAT_HEADS_CHECK(dout, heads);
  if (max_rows <= 0) return SG_OK;
  BSrcArgs a;
  memset(&a, 0, sizeof(a));
  a.l = l; a.d = d; a.dout = dout; a.heads = heads; a.g = y.g;
  a.voff_lm1 = y.voff[l - 1]; a.voff_l = y.voff[l]; a.pbase_l = y.pbase[l]; a.key_base = key_base;
  a.grouped = I32p(y.o_grouped); a.rank = I32p(y.o_rank); a.contrib = I32p(y.o_contrib);
  a.ldst = I32p(y.o_ldst); a.sendpos = I32p(y.o_sendpos);
  a.perm = perm; a.srcbeg = srcbeg; a.srcend = srcend;
  a.alpha = alpha; a.d_pre = d_pre; a.dnc = dnc; a.dnc_recv = dnc_recv; a.dnc_stride = dnc_stride;
  a.dt_loc = dt_loc; a.dt_recv = dt_recv; a.a_src = a_src; a.a_dst = a_dst;
  a.d_z = d_z; a.ds = ds; a.dt_tot = dt_tot;
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = clamp_grid(div_up(max_rows, 8), kSMs * 8);
  const int q = dout / (4 * heads);
  const bool v4 = dout % (4 * heads) == 0 && (q & (q - 1)) == 0 && (heads & (heads - 1)) == 0;
  if (v4 && dout <= 16) ::sg::launch(k_gat_bwd_src<4, 4>, grid, 256, 0, st, meta, a);
  else if (v4 && dout <= 32) ::sg::launch(k_gat_bwd_src<4, 8>, grid, 256, 0, st, meta, a);
  else if (v4 && dout <= 64) ::sg::launch(k_gat_bwd_src<4, 16>, grid, 256, 0, st, meta, a);
  else if (v4 && dout <= 128) ::sg::launch(k_gat_bwd_src<4, 32>, grid, 256, 0, st, meta, a);
  else if (heads == 1 && dout <= 8) ::sg::launch(k_gat_bwd_src<1, 8>, grid, 256, 0, st, meta, a);
  else if (heads == 1 && dout <= 32) ::sg::launch(k_gat_bwd_src<1, 32>, grid, 256, 0, st, meta, a);
  else {
    set_error("gat_bwd_src: unsupported width/heads");
    return SG_ERR_ARG;
  }
  SG_CHECK_LAUNCH("k_gat_bwd_src");
  return SG_OK;
}

// CTAs the weight-gradient launch wants (the partial buffer holds one slice per CTA)
extern "C" int32_t sg_gat_bwd_param_blocks(int32_t w, int32_t dout, int32_t heads, int64_t rows) {
  (void)heads;
  const int64_t tiles = std::max<int64_t>(1, (rows + QTR - 1) / QTR);
  const bool mma = !getenv("SG_NO_MMA") && dout == 64 && w % 4 == 0 && w > 32 && w <= 128;
  const int64_t cap = mma ? 2 * kSMs : 6 * kSMs;  // pipelined MMA tiles: 2 CTAs per SM; else latency-bound
  return (int32_t)std::min(tiles, cap);
}

extern "C" int sg_gat_bwd_param(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t d,
                                const float* h_prev, const int32_t* src_row, int32_t w, int32_t dout,
                                int32_t heads, const float* z, const float* d_z, const float* ds,
                                const float* dt_tot, const float* W, float* partial, int32_t nblocks,
                                float* d_prev, int64_t max_rows, void* stream) {
  SG_REQUIRE(split_ws && lay, "gat_bwd_param: null workspace");
  SPLIT_PTRS
  GAT_HEADS_CHECK(dout, heads);
  SG_REQUIRE(nblocks >= 1, "gat_bwd_param: nblocks >= 1");
  BParamArgs a;
  memset(&a, 0, sizeof(a));
  a.l = l; a.d = d; a.w = w; a.dout = dout; a.heads = heads;
  a.voff_lm1 = y.voff[l - 1]; a.voff_l = y.voff[l];
  a.h_prev = h_prev; a.src_row = src_row; a.grouped = I32p(y.o_grouped); a.rank = I32p(y.o_rank);
  a.z = z; a.d_z = d_z; a.ds = ds; a.dt_tot = dt_tot; a.W = W; a.partial = partial; a.d_prev = d_prev;
  // T4 tiles: (w/4)*(dout/4) <= 512 slots (2 tiles of 16 per thread)
  const bool t4 = w % 4 == 0 && dout % 4 == 0 && (w / 4) * (dout / 4) <= 512;
  const size_t smem = sizeof(float) * (2 * (size_t)QTR * dout + (size_t)dout * (w + 1) +
                                       (size_t)QTR * (w + 4) + 2 * (size_t)QTR * heads + QTR);
  cudaStream_t st = (cudaStream_t)stream;
  if ((int64_t)w * dout > 256 * QMAXQ * 4 || smem > 227 * 1024) {
    // wide layer: dW partials as a dense GEMM, attention-vector partials, d_prev = d_z W^T
    TnArgs t;
    memset(&t, 0, sizeof(t));
    t.R_dev = &meta->n_own[l - 1][d];
    t.K = w; t.N = dout; t.A = h_prev; t.lda = w;
    t.ar.mode = src_row ? 1 : 0; t.ar.map = src_row; t.ar.base_dev = &meta->own_off[l - 1][d];
    t.G = d_z; t.ldg = dout; t.g_base_dev = &meta->own_off[l - 1][d];
    t.P = partial; t.pstride = (int64_t)w * dout + 2 * dout; t.p_off = 0; t.nsplit = nblocks;
    int rc = dense_gemm_tn_partial(t, st);
    if (rc) return rc;
    ::sg::launch(k_gat_attn_partial, nblocks, 256, 0, st, meta, a, nblocks);
    SG_CHECK_LAUNCH("k_gat_attn_partial");
    if (d_prev) {
      GemmArgs g;
      memset(&g, 0, sizeof(g));
      g.R_dev = &meta->n_own[l - 1][d];
      g.K = dout; g.N = w; g.A = d_z; g.lda = dout; g.ar.mode = 0;
      g.ar.base_dev = &meta->own_off[l - 1][d];
      g.B = W; g.ldb = dout; g.bt = 1; g.C = d_prev; g.ldc = w; g.c_base_dev = &meta->own_off[l - 1][d];
      rc = dense_gemm_rows(g, max_rows, st);
      if (rc) return rc;
    }
    return SG_OK;
  }
  static const bool use_mma = !getenv("SG_NO_MMA");
  if (use_mma && dout == 64 && w % 4 == 0 && w > 32 && w <= 128) {
    switch ((w + 15) / 16) {
      case 3: return launch_wgrad_mma<3>(meta, a, nblocks, st);
      case 4: return launch_wgrad_mma<4>(meta, a, nblocks, st);
      case 5: return launch_wgrad_mma<5>(meta, a, nblocks, st);
      case 6: return launch_wgrad_mma<6>(meta, a, nblocks, st);
      case 7: return launch_wgrad_mma<7>(meta, a, nblocks, st);
      default: return launch_wgrad_mma<8>(meta, a, nblocks, st);
    }
  } else if (t4) {
    SG_CUDA(allow_max_smem<k_gat_bwd_param<1>>());
    ::sg::launch(k_gat_bwd_param<1>, nblocks, 256, smem, st, meta, a);
  } else {
    SG_CUDA(allow_max_smem<k_gat_bwd_param<0>>());
    ::sg::launch(k_gat_bwd_param<0>, nblocks, 256, smem, st, meta, a);
  }
  SG_CHECK_LAUNCH("k_gat_bwd_param");
  return SG_OK;
}


// Layer-1 weight gradient of GAT in one destination-centric pass (see
// k_gat_wgrad_dst): replaces sg_gat_bwd_src + sg_gat_bwd_param at layer 1
// (engine.py:480-552, nothing needs d(loss)/d(features)). D = 64, heads in
// {1, 2, 4}, w % 4 == 0 and w <= 128; partial holds nblocks slices of
// w*64 + 128 floats ([dW | da_src | da_dst], the k_gat_bwd_param layout).
extern "C" int32_t sg_gat_wgrad_dst_blocks(int64_t rows) {
  return (int32_t)std::max<int64_t>(1, std::min<int64_t>((rows + WD_TM - 1) / WD_TM, 3 * kSMs));  // 3 CTAs / SM
}

extern "C" int sg_gat_wgrad_dst(const void* split_ws, const SgSplitLayout* lay, int32_t d, int32_t w, int32_t heads,
                                const float* h0, const int32_t* src_row, const int32_t* dperm, const float* alpha,
                                const float* d_pre, const float* dnc, const float* dnc_recv, int32_t recv_stride,
                                const float* dt_loc, const float* dt_recv, const float* W, const float* a_src,
                                const float* a_dst, float* partial, int32_t nblocks, void* stream) {
  SG_REQUIRE(split_ws && lay && h0 && alpha && d_pre && dnc && dt_loc && W && a_src && a_dst && partial,
             "gat_wgrad_dst: null argument");
  SPLIT_PTRS
  SG_REQUIRE(d >= 0 && d < y.g && y.L >= 1, "gat_wgrad_dst: bad device");
  SG_REQUIRE(w % 4 == 0 && w >= 4 && w <= 128 && (heads == 1 || heads == 2 || heads == 4),
             "gat_wgrad_dst: needs w % 4 == 0, w <= 128, heads in {1, 2, 4}, D = 64");
  SG_REQUIRE(nblocks >= 1, "gat_wgrad_dst: nblocks >= 1");
  WdArgs a;
  memset(&a, 0, sizeof(a));
  a.d = d; a.w = w; a.heads = heads; a.stride = recv_stride; a.g = y.g;
  a.eoff_li = y.eoff[0]; a.rbase_li = y.rbase[0]; a.pbase_l = y.pbase[1]; a.voff_l = y.voff[1];
  a.rowbeg = I32p(y.o_rowbeg); a.rowend = I32p(y.o_rowend); a.lsrc = I32p(y.o_lsrc); a.dperm = dperm;
  a.sendpos = I32p(y.o_sendpos); a.selfrow = I32p(y.o_selfrow); a.contrib = I32p(y.o_contrib);
  a.src_row = src_row; a.h0 = h0; a.alpha = alpha; a.d_pre = d_pre; a.dnc = dnc; a.dnc_recv = dnc_recv;
  a.dt_loc = dt_loc; a.dt_recv = dt_recv; a.W = W; a.a_src = a_src; a.a_dst = a_dst; a.partial = partial;
  const int HW = heads * w;
  const size_t smem = sizeof(float) * ((size_t)w * WD_D + 2 * HW + (size_t)WD_TM * (HW + w + WD_D + heads));
  SG_REQUIRE(smem <= 227 * 1024, "gat_wgrad_dst: shared memory");
  cudaStream_t st = (cudaStream_t)stream;
switch (heads) {
    case 1: { const cudaError_t e1 = allow_max_smem<k_gat_wgrad_dst<1>>(); SG_CUDA(e1);
              ::sg::launch(k_gat_wgrad_dst<1>, nblocks, 256, smem, st, meta, a); break; }
    case 2: { const cudaError_t e2 = allow_max_smem<k_gat_wgrad_dst<2>>(); SG_CUDA(e2);
              ::sg::launch(k_gat_wgrad_dst<2>, nblocks, 256, smem, st, meta, a); break; }
    default: { const cudaError_t e4 = allow_max_smem<k_gat_wgrad_dst<4>>(); SG_CUDA(e4);
               ::sg::launch(k_gat_wgrad_dst<4>, nblocks, 256, smem, st, meta, a); break; }
  }
  SG_CHECK_LAUNCH("k_gat_wgrad_dst");
  return SG_OK;
}

}  // namespace sg
