// Stable LSD radix sort of (uint32 key, int32 value) pairs and the CSR builders
// that use it. The reference's segment_sum sorts by key with a stable argsort
// (models.py:155-159); the transpose SpMM of the backward pass
// (engine.py:263-273) needs the local edges grouped by SOURCE row, in sample
// order within a row, which is exactly a stable sort by source row.
//
// One pass per 8 key bits: per-tile digit histogram -> single-block scan of the
// digit-major table -> stable scatter (warp __match_any_sync ranks, warps in
// order), so equal keys keep their input order and the result is deterministic.
#include <cstring>
#include <utility>

#include "common.cuh"

namespace sg {
namespace {

constexpr int RS_THREADS = 256;
constexpr int RS_ROUNDS = 4;
constexpr int RS_T = RS_THREADS * RS_ROUNDS;  // 4096 elements per tile
constexpr int RADIX = 256;

__global__ void __launch_bounds__(RS_THREADS) rs_hist(const uint32_t* __restrict__ keys,
                                                      const int32_t* __restrict__ n_dev, int shift,
                                                      int ntiles, int32_t* __restrict__ hist) {
  SG_PDL_ENTRY();
  __shared__ int cnt[RADIX];
  const int t = blockIdx.x;
  const int n = *n_dev;
  cnt[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)t * RS_T;
  for (int64_t i = base + threadIdx.x; i < min(base + (int64_t)RS_T, (int64_t)n); i += RS_THREADS)
    atomicAdd(&cnt[(keys[i] >> shift) & 0xff], 1);
  __syncthreads();
  hist[threadIdx.x * ntiles + t] = cnt[threadIdx.x];
}

// One block per digit: exclusive scan of that digit's tile counts (in place)
// and the digit total. The scatter kernel scans the 256 totals itself.
__global__ void __launch_bounds__(256) rs_scan(int32_t* __restrict__ hist, int ntiles,
                                               int32_t* __restrict__ dtot) {
  SG_PDL_ENTRY();
  __shared__ int wsum[8];
  __shared__ int carry;
  const int dg = blockIdx.x;
  int32_t* h = hist + (int64_t)dg * ntiles;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < ntiles; b0 += 256) {
    const int i = b0 + threadIdx.x;
    const int v = i < ntiles ? h[i] : 0;
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    int wp = 0;
    for (int w = 0; w < warp; ++w) wp += wsum[w];
    const int base = carry;
    if (i < ntiles) h[i] = base + wp + inc - v;
    __syncthreads();
    if (threadIdx.x == 255) carry = base + wp + inc;
    __syncthreads();
  }
  if (threadIdx.x == 0) dtot[dg] = carry;
}

__global__ void __launch_bounds__(RS_THREADS) rs_scatter(const uint32_t* __restrict__ kin,
                                                         const int32_t* __restrict__ vin,
                                                         const int32_t* __restrict__ n_dev,
                                                         int shift, int ntiles,
                                                         const int32_t* __restrict__ hist,
                                                         const int32_t* __restrict__ dtot,
                                                         uint32_t* __restrict__ kout,
                                                         int32_t* __restrict__ vout) {
  SG_PDL_ENTRY();
  __shared__ int wcnt[RS_THREADS / 32][RADIX];
  __shared__ int dsum[8];
  const int t = blockIdx.x;
  const int n = *n_dev;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = lane; k < RADIX; k += 32) wcnt[warp][k] = 0;
  __syncwarp();
  const int64_t base = (int64_t)t * RS_T + warp * (32 * RS_ROUNDS);
  const unsigned lt = lanemask_lt();
  uint32_t key[RS_ROUNDS];
  int rnk[RS_ROUNDS];
  (void)ntiles;
#pragma unroll
  for (int j = 0; j < RS_ROUNDS; ++j) {
    const int64_t i = base + j * 32 + lane;
    const bool valid = i < n;
    key[j] = valid ? kin[i] : 0u;
    const int dg = valid ? (int)((key[j] >> shift) & 0xff) : RADIX;
    const unsigned peers = __match_any_sync(0xffffffffu, dg);
    const int r = __popc(peers & lt);
    const int prior = valid ? wcnt[warp][dg] : 0;
    __syncwarp();
    if (valid && r == 0) wcnt[warp][dg] = prior + __popc(peers);
    __syncwarp();
    rnk[j] = prior + r;
  }
  __syncthreads();
  // digit base = exclusive scan of the 256 digit totals (thread = digit),
  // plus this tile's prefix inside the digit, plus the warps before
  {
    const int dg = threadIdx.x;
    const int v = dtot[dg];
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) dsum[warp] = inc;
    __syncthreads();
    int wp = 0;
    for (int w = 0; w < warp; ++w) wp += dsum[w];
    int run = wp + inc - v + hist[dg * ntiles + t];
#pragma unroll
    for (int w = 0; w < RS_THREADS / 32; ++w) {
      int v = wcnt[w][dg];
      wcnt[w][dg] = run;
      run += v;
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < RS_ROUNDS; ++j) {
    const int64_t i = base + j * 32 + lane;
    if (i < n) {
      const int dg = (key[j] >> shift) & 0xff;
      const int pos = wcnt[warp][dg] + rnk[j];
      kout[pos] = key[j];
      vout[pos] = vin[i];
    }
  }
}

__global__ void k_copy_pairs(const uint32_t* __restrict__ ks, const int32_t* __restrict__ vs,
                             const int32_t* __restrict__ n_dev, uint32_t* __restrict__ kd,
                             int32_t* __restrict__ vd) {
  SG_PDL_ENTRY();
  const int n = *n_dev;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    kd[i] = ks[i];
    vd[i] = vs[i];
  }
}

struct KeyBase {
  int64_t v[SG_MAXL];
  int64_t pbase[SG_MAXL + 2];
};

// Edges of device d, layers [lmin, L], as (row key, edge slot). mode 0: key =
// global source row at l-1 (+ per-layer base); mode 1: key = destination row
// in the split's per-layer row space (owned rows then reference rows).
// val_mode 0: value = global edge slot; 1: value = encoded destination row of
// the backward gradient (>= 0: owned row own_off+q, < 0: -(1 + pair slot)).
__global__ void k_edge_row_keys(const SgMeta* __restrict__ meta, const int32_t* __restrict__ lidx,
                                const int32_t* __restrict__ ldst, const int32_t* __restrict__ sendpos,
                                int d, int lmin, int mode, int val_mode, KeyBase kb,
                                uint32_t* __restrict__ keys, int32_t* __restrict__ vals,
                                int32_t* __restrict__ n_dev) {
  SG_PDL_ENTRY();
  const int L = meta->L;
  const int64_t e0 = meta->eoff[lmin - 1], e1 = meta->eoff[L];
  int flat0[SG_MAXL];
  int acc = 0;
  for (int li = lmin - 1; li < L; ++li) {
    flat0[li] = acc;
    acc += meta->n_edge[li][d];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *n_dev = acc;
  for (int64_t x = e0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < e1;
       x += (int64_t)gridDim.x * blockDim.x) {
    int li = lmin - 1;
    while (li + 1 < L && meta->eoff[li + 1] <= x) ++li;
    const int i = (int)(x - meta->eoff[li]);
    const int b = meta->edge_off[li][d], e = meta->edge_off[li][d + 1];
    if (i < b || i >= e) continue;
    const int f = flat0[li] + (i - b);
    const int64_t row = mode == 0
        ? meta->own_off[li][d]
        : (int64_t)meta->own_off[li + 1][d] + meta->ref_off[li + 1][d];
    keys[f] = (uint32_t)(kb.v[li] + row + lidx[x]);
    if (val_mode == 0) {
      vals[f] = (int32_t)x;
    } else {
      const int l = li + 1;
      const int q = ldst[x];
      const int no = meta->n_own[l][d];
      vals[f] = q < no ? meta->own_off[l][d] + q
                       : -1 - sendpos[kb.pbase[l] + meta->ref_off[l][d] + (q - no)];
    }
  }
}

// Run boundaries of a sorted key array -> [beg, end) per key.
__global__ void k_runs(const uint32_t* __restrict__ keys, const int32_t* __restrict__ n_dev,
                       int32_t* __restrict__ beg, int32_t* __restrict__ end) {
  SG_PDL_ENTRY();
  const int n = *n_dev;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t k = keys[i];
    if (i == 0 || keys[i - 1] != k) beg[k] = i;
    if (i == n - 1 || keys[i + 1] != k) end[k] = i + 1;
  }
}

}  // namespace

static int64_t a256(int64_t x) { return (x + 255) & ~int64_t(255); }

extern "C" int64_t sg_sort_ws_bytes(int64_t n_max) {
  const int64_t ntiles = (n_max + RS_T - 1) / RS_T;
  return a256(4 * n_max) * 2 + a256(4 * RADIX * (ntiles > 0 ? ntiles : 1)) + a256(4 * RADIX);
}

extern "C" int sg_sort_pairs(void* ws, int64_t n_max, const int32_t* n_dev, uint32_t* keys,
                             int32_t* vals, int32_t key_bits, void* stream) {
  SG_REQUIRE(ws && n_dev && keys && vals, "sort: null pointer");
  SG_REQUIRE(key_bits >= 0 && key_bits <= 32, "sort: key_bits out of range");
  if (n_max <= 0) return SG_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int ntiles = (int)((n_max + RS_T - 1) / RS_T);
  char* b = (char*)ws;
  uint32_t* k2 = (uint32_t*)b;
  int32_t* v2 = (int32_t*)(b + a256(4 * n_max));
  int32_t* hist = (int32_t*)(b + 2 * a256(4 * n_max));
  int32_t* dtot = (int32_t*)(b + 2 * a256(4 * n_max) + a256(4 * RADIX * ntiles));
  const int passes = (key_bits + 7) / 8;
  uint32_t* ka = keys;
  int32_t* va = vals;
  uint32_t* kb = k2;
  int32_t* vb = v2;
  for (int p = 0; p < passes; ++p) {
    const int shift = 8 * p;
    ::sg::launch(rs_hist, ntiles, RS_THREADS, 0, st, ka, n_dev, shift, ntiles, hist);
    SG_CHECK_LAUNCH("rs_hist");
    ::sg::launch(rs_scan, RADIX, 256, 0, st, hist, ntiles, dtot);
    SG_CHECK_LAUNCH("rs_scan");
    ::sg::launch(rs_scatter, ntiles, RS_THREADS, 0, st, ka, va, n_dev, shift, ntiles, hist, dtot, kb, vb);
    SG_CHECK_LAUNCH("rs_scatter");
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  if (ka != keys) {
    ::sg::launch(k_copy_pairs, clamp_grid(div_up(n_max, 256), kSMs * 4), 256, 0, st, ka, va, n_dev, keys,
                                                                          vals);
    SG_CHECK_LAUNCH("k_copy_pairs");
  }
  return SG_OK;
}

extern "C" int sg_src_csr(const void* split_ws, const SgSplitLayout* lay, int32_t d,
                          int32_t lmin, int32_t val_mode, void* sort_ws, int64_t n_max,
                          int32_t* n_dev, uint32_t* keys, int32_t* perm, int32_t* srcbeg,
                          int32_t* srcend, int64_t n_rows_total, void* stream) {
  SG_REQUIRE(split_ws && lay, "src_csr: null workspace");
  const SgSplitLayout& y = *lay;
  SG_REQUIRE(lmin >= 1 && lmin <= y.L, "src_csr: lmin out of range");
  SG_REQUIRE(d >= 0 && d < y.g, "src_csr: device out of range");
  cudaStream_t st = (cudaStream_t)stream;
  const char* base = (const char*)split_ws;
  const SgMeta* meta = (const SgMeta*)(base + y.o_meta);
  KeyBase kb;
  memset(&kb, 0, sizeof(kb));
  int64_t acc = 0;
  for (int l = lmin; l <= y.L; ++l) {
    kb.v[l - 1] = acc;
    acc += y.nV[l - 1];
  }
  SG_REQUIRE(acc <= n_rows_total, "src_csr: row table too small");
  int bits = 0;
  while ((int64_t(1) << bits) < acc) ++bits;
  SG_CUDA(cudaMemsetAsync(srcbeg, 0, 4 * acc, st));
  SG_CUDA(cudaMemsetAsync(srcend, 0, 4 * acc, st));
  const int64_t e_span = y.eoff[y.L] - y.eoff[lmin - 1];
  for (int l = 0; l <= y.L + 1; ++l) kb.pbase[l] = y.pbase[l];
  ::sg::launch(k_edge_row_keys, clamp_grid(div_up(e_span, 256), kSMs * 8), 256, 0, st, meta, (const int32_t*)(base + y.o_lsrc), (const int32_t*)(base + y.o_ldst),
      (const int32_t*)(base + y.o_sendpos), d, lmin, 0, val_mode, kb, keys, perm, n_dev);
  SG_CHECK_LAUNCH("k_edge_row_keys(src)");
  int rc = sg_sort_pairs(sort_ws, n_max, n_dev, keys, perm, bits, stream);
  if (rc) return rc;
  ::sg::launch(k_runs, clamp_grid(div_up(n_max, 256), kSMs * 8), 256, 0, st, keys, n_dev, srcbeg, srcend);
  SG_CHECK_LAUNCH("k_runs(src)");
  return SG_OK;
}

extern "C" int sg_dst_csr(void* split_ws, const SgSplitLayout* lay, int32_t d, void* sort_ws,
                          int64_t n_max, int32_t* n_dev, uint32_t* keys, int32_t* perm,
                          void* stream) {
  SG_REQUIRE(split_ws && lay, "dst_csr: null workspace");
  const SgSplitLayout& y = *lay;
  SG_REQUIRE(d >= 0 && d < y.g, "dst_csr: device out of range");
  cudaStream_t st = (cudaStream_t)stream;
  char* base = (char*)split_ws;
  const SgMeta* meta = (const SgMeta*)(base + y.o_meta);
  KeyBase kb;
  memset(&kb, 0, sizeof(kb));
  for (int l = 1; l <= y.L; ++l) kb.v[l - 1] = y.rbase[l - 1];
  int bits = 0;
  while ((int64_t(1) << bits) < y.rbase[y.L]) ++bits;
  ::sg::launch(k_edge_row_keys, clamp_grid(div_up(y.nEtot, 256), kSMs * 8), 256, 0, st, meta, (const int32_t*)(base + y.o_ldst), nullptr, nullptr, d, 1, 1, 0, kb, keys, perm, n_dev);
  SG_CHECK_LAUNCH("k_edge_row_keys(dst)");
  int rc = sg_sort_pairs(sort_ws, n_max, n_dev, keys, perm, bits, stream);
  if (rc) return rc;
  ::sg::launch(k_runs, clamp_grid(div_up(n_max, 256), kSMs * 8), 256, 0, st, keys, n_dev, (int32_t*)(base + y.o_rowbeg), (int32_t*)(base + y.o_rowend));
  SG_CHECK_LAUNCH("k_runs(dst)");
  return SG_OK;
}

}  // namespace sg
