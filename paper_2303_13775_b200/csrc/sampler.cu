// k-hop neighbourhood sampler on the GPU: sample_minibatch (sampling.py:118-177)
// from a device-resident in-CSR, bit-identical to the native host sampler
// (host.cpp, same counter-based RNG), so a sample never crosses PCIe.
//
// Per layer l = L..1, with cur = V^l (device sizes, no host round trip):
//   k_smp_mark    stamp[cur[i]] = gen, pos[cur[i]] = i   (membership of V^l)
//   k_smp_pick    one thread per destination: self loop and parallel edges
//                 dropped, partial Fisher-Yates with a sparse swap map when
//                 the degree exceeds the fanout (hash(seed, l<<40 ^ i, j))
//   scan          edge offsets: eoff[i] = i + sum_{i'<i} picks(i')
//   k_smp_first   first occurrence of every picked vertex outside V^l:
//                 64-bit atomicMin of (generation, edge position)
//   k_smp_isfirst flag the first-occurrence positions; scan -> the new
//                 vertices' indices in first-seen order (the reference's
//                 dict insertion order) without a sort
//   k_smp_assign  V^{l-1} = V^l ++ new vertices; pos / stamp of the new ones
//   k_smp_edges   (src, dst) per edge: self edge first, then the picks
// Generations make the n-sized stamp / first arrays reusable without
// clearing (a newer generation always wins the 64-bit min).
#include <algorithm>
#include <cstring>

#include "common.cuh"
#include "rng.h"

namespace sg {
namespace {

constexpr int SMP_FMAX = 64;  // max fanout (sparse swap map: 2 * fanout entries per thread)

struct SmpLayer {
  int l, f;
  uint32_t gen;
  uint64_t seed;
  int64_t cur_off, prev_off;  // capacity offsets of V^l and V^{l-1} in the packed V
  int64_t e_off;              // capacity offset of E^l in the packed edge arrays
  int size_cur, size_prev;    // indices into sizes[]: nV[l], nV[l-1]; edges at size_e
  int size_e;
  int64_t cap_prev, cap_e;    // capacities of V^{l-1} and E^l (overflow sets err)
  int* err;
};

__device__ __forceinline__ int nv_of(const int64_t* sizes, int idx) { return (int)sizes[idx]; }

__global__ void k_smp_targets(const int64_t* __restrict__ targets, int64_t nt, int64_t n, int32_t* __restrict__ V,
                              int64_t off, int64_t* __restrict__ sizes, int size_idx, int* __restrict__ err) {
  SG_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nt; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = targets[i];
    if (t < 0 || t >= n) atomicOr(err, 1);
    V[off + i] = (int32_t)t;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) sizes[size_idx] = nt;
}

__global__ void k_smp_mark(const int32_t* __restrict__ V, const int64_t* __restrict__ sizes, SmpLayer s,
                           uint32_t* __restrict__ stamp, int32_t* __restrict__ pos) {
  SG_PDL_ENTRY();
  const int nc = nv_of(sizes, s.size_cur);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nc; i += gridDim.x * blockDim.x) {
    const int32_t v = V[s.cur_off + i];
    stamp[v] = s.gen;
    pos[v] = i;
  }
}

__global__ void k_smp_pick(const int32_t* __restrict__ V, const int64_t* __restrict__ sizes, SmpLayer s,
                           const int64_t* __restrict__ ro, const int32_t* __restrict__ ci,
                           int32_t* __restrict__ picks, int32_t* __restrict__ npk) {
  SG_PDL_ENTRY();
  const int nc = nv_of(sizes, s.size_cur);
  const int f = s.f;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nc; i += gridDim.x * blockDim.x) {
    const int32_t v = V[s.cur_off + i];
    const int64_t s0 = ro[v], m = ro[v + 1] - s0;
    const int64_t k = m < f ? m : f;
    int cnt = 0;
    int32_t* out = picks + (int64_t)i * f;
    auto accept = [&](int32_t u) {
      if (u == v) return;  // the input's own self-loop
      for (int t = 0; t < cnt; ++t)
        if (out[t] == u) return;  // parallel edge
      out[cnt++] = u;
    };
    if (k > 0) {
      if (k >= m) {
        for (int64_t j = 0; j < m; ++j) accept(ci[s0 + j]);
      } else {
        int64_t mk[2 * SMP_FMAX];
        int64_t mv[2 * SMP_FMAX];
        int nm = 0;
        auto get = [&](int64_t x) -> int64_t {
          for (int t = 0; t < nm; ++t)
            if (mk[t] == x) return mv[t];
          return ci[s0 + x];
        };
        auto set = [&](int64_t x, int64_t val) {
          for (int t = 0; t < nm; ++t)
            if (mk[t] == x) {
              mv[t] = val;
              return;
            }
          mk[nm] = x;
          mv[nm] = val;
          ++nm;
        };
        for (int64_t j = 0; j < k; ++j) {
          const uint64_t h = sg_hash3(s.seed, ((uint64_t)s.l << 40) ^ (uint64_t)i, (uint64_t)j);
          const int64_t r = j + (int64_t)sg_bounded(h, (uint64_t)(m - j));
          const int64_t vj = get(j), vr = get(r);
          set(r, vj);
          set(j, vr);
          accept((int32_t)vr);
        }
      }
    }
    npk[i] = 1 + cnt;  // the self edge plus the picks
  }
}

// Exclusive scan of int32 counts (n from sizes[size_idx] or a fixed n):
// per-block sums, a one-block scan of the block sums, then the local scan.
constexpr int SCAN_B = 1024;  // elements per block (256 threads x 4)

__global__ void __launch_bounds__(256) k_scan_blocks(const int32_t* __restrict__ in, const int64_t* __restrict__ sizes,
                                                     int size_idx, int64_t nfix, int32_t* __restrict__ bsum) {
  SG_PDL_ENTRY();
  const int64_t n = size_idx >= 0 ? sizes[size_idx] : nfix;
  __shared__ int red[8];
  const int64_t b0 = (int64_t)blockIdx.x * SCAN_B;
  int v = 0;
  for (int k = 0; k < 4; ++k) {
    const int64_t i = b0 + threadIdx.x * 4 + k;
    if (i < n) v += in[i];
  }
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < 8; ++w) t += red[w];
    bsum[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(1024) k_scan_top(int32_t* __restrict__ bsum, int nb, int64_t* __restrict__ total_out) {
  SG_PDL_ENTRY();
  __shared__ int wsum[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nb; base += 1024) {
    const int i = base + threadIdx.x;
    const int v = i < nb ? bsum[i] : 0;
    int x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if ((threadIdx.x & 31) >= o) x += y;
    }
    if ((threadIdx.x & 31) == 31) wsum[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      int ws = wsum[threadIdx.x];
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, ws, o);
        if (threadIdx.x >= o) ws += y;
      }
      wsum[threadIdx.x] = ws;
    }
    __syncthreads();
    const int excl = carry + x - v + ((threadIdx.x >> 5) ? wsum[(threadIdx.x >> 5) - 1] : 0);
    if (i < nb) bsum[i] = excl;
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total_out) *total_out = carry;
}

__global__ void __launch_bounds__(256) k_scan_local(const int32_t* __restrict__ in, const int64_t* __restrict__ sizes,
                                                    int size_idx, int64_t nfix, const int32_t* __restrict__ bsum,
                                                    int32_t* __restrict__ out) {
  SG_PDL_ENTRY();
  const int64_t n = size_idx >= 0 ? sizes[size_idx] : nfix;
  __shared__ int wsum[8];
  const int64_t b0 = (int64_t)blockIdx.x * SCAN_B;
  int v[4], t = 0;
  for (int k = 0; k < 4; ++k) {
    const int64_t i = b0 + threadIdx.x * 4 + k;
    v[k] = i < n ? in[i] : 0;
    t += v[k];
  }
  int x = t;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) >= o) x += y;
  }
  if ((threadIdx.x & 31) == 31) wsum[threadIdx.x >> 5] = x;
  __syncthreads();
  int wpre = 0;
  for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) wpre += wsum[w];
  int run = bsum[blockIdx.x] + wpre + x - t;
  for (int k = 0; k < 4; ++k) {
    const int64_t i = b0 + threadIdx.x * 4 + k;
    if (i < n) out[i] = run;
    run += v[k];
  }
}

__global__ void k_smp_first(const int64_t* __restrict__ sizes, SmpLayer s, const int32_t* __restrict__ picks,
                            const int32_t* __restrict__ npk, const int32_t* __restrict__ eoff,
                            const uint32_t* __restrict__ stamp, unsigned long long* __restrict__ first) {
  SG_PDL_ENTRY();
  const int nc = nv_of(sizes, s.size_cur);
  const unsigned long long hi = (unsigned long long)(0xFFFFFFFFu - s.gen) << 32;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nc; i += gridDim.x * blockDim.x) {
    const int c = npk[i] - 1;
    for (int t = 0; t < c; ++t) {
      const int32_t u = picks[(int64_t)i * s.f + t];
      if (stamp[u] != s.gen) atomicMin(&first[u], hi | (unsigned)(eoff[i] + 1 + t));
    }
  }
}

__global__ void k_smp_isfirst(const int64_t* __restrict__ sizes, SmpLayer s, const int32_t* __restrict__ picks,
                              const int32_t* __restrict__ npk, const int32_t* __restrict__ eoff,
                              const uint32_t* __restrict__ stamp, const unsigned long long* __restrict__ first,
                              int32_t* __restrict__ isfirst) {
  SG_PDL_ENTRY();
  const int nc = nv_of(sizes, s.size_cur);
  const unsigned long long hi = (unsigned long long)(0xFFFFFFFFu - s.gen) << 32;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nc; i += gridDim.x * blockDim.x) {
    const int e0 = eoff[i];
    const int c = npk[i] - 1;
    if (e0 + c >= s.cap_e) {  // E^l over capacity
      atomicOr(s.err, 2);
      continue;
    }
    isfirst[e0] = 0;
    for (int t = 0; t < c; ++t) {
      const int32_t u = picks[(int64_t)i * s.f + t];
      const unsigned p = (unsigned)(e0 + 1 + t);
      isfirst[e0 + 1 + t] = (stamp[u] != s.gen && first[u] == (hi | p)) ? 1 : 0;
    }
  }
}

__global__ void k_smp_assign(int32_t* __restrict__ V, int64_t* __restrict__ sizes, SmpLayer s,
                             const int32_t* __restrict__ picks, const int32_t* __restrict__ npk,
                             const int32_t* __restrict__ eoff, const int32_t* __restrict__ isfirst,
                             const int32_t* __restrict__ newidx, const int64_t* __restrict__ totals,
                             uint32_t* __restrict__ stamp, int32_t* __restrict__ pos) {
  SG_PDL_ENTRY();
  const int nc = nv_of(sizes, s.size_cur);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nc; i += gridDim.x * blockDim.x) {
    V[s.prev_off + i] = V[s.cur_off + i];  // V^l is a prefix of V^{l-1}
    const int e0 = eoff[i];
    const int c = npk[i] - 1;
    for (int t = 0; t < c; ++t) {
      const int p = e0 + 1 + t;
      if (!isfirst[p]) continue;
      const int32_t u = picks[(int64_t)i * s.f + t];
      const int j = nc + newidx[p];
      if (j >= s.cap_prev) {  // V^{l-1} over capacity
        atomicOr(s.err, 4);
        continue;
      }
      V[s.prev_off + j] = u;
      pos[u] = j;
      stamp[u] = s.gen;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    sizes[s.size_prev] = nc + totals[1];  // new vertices
    sizes[s.size_e] = totals[0];          // edges of E^l
  }
}

__global__ void k_smp_edges(const int64_t* __restrict__ sizes, SmpLayer s, const int32_t* __restrict__ picks,
                            const int32_t* __restrict__ npk, const int32_t* __restrict__ eoff,
                            const int32_t* __restrict__ pos, int32_t* __restrict__ esrc, int32_t* __restrict__ edst) {
  SG_PDL_ENTRY();
  const int nc = nv_of(sizes, s.size_cur);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nc; i += gridDim.x * blockDim.x) {
    const int c = npk[i] - 1;
    if (eoff[i] + c >= s.cap_e) continue;
    const int64_t e0 = s.e_off + eoff[i];
    esrc[e0] = i;
    edst[e0] = i;
    for (int t = 0; t < c; ++t) {
      esrc[e0 + 1 + t] = pos[picks[(int64_t)i * s.f + t]];
      edst[e0 + 1 + t] = i;
    }
  }
}

}  // namespace
}  // namespace sg

using namespace sg;

// One-time scratch initialisation: generation stamps 0, first-occurrence keys
// all-ones (any current generation's key is smaller).
extern "C" int sg_gpu_sampler_ws_init(void* ws, int64_t n, void* stream) {
  SG_REQUIRE(ws && n > 0, "gpu_sampler_ws_init: bad argument");
  cudaStream_t st = (cudaStream_t)stream;
  SG_CUDA(cudaMemsetAsync(ws, 0, 8 * (size_t)n, st));
  SG_CUDA(cudaMemsetAsync((char*)ws + 8 * n, 0xFF, 8 * (size_t)n, st));
  return SG_OK;
}

// Scratch bytes for sg_gpu_sample: n-sized stamp / pos / first arrays plus
// per-layer pick buffers for capacities cap_nV / cap_nE and fanout fmax.
extern "C" int64_t sg_gpu_sampler_ws_bytes(int64_t n, int64_t max_dst, int64_t max_edges, int32_t fmax) {
  const int64_t nb = (max_edges + SCAN_B - 1) / SCAN_B + 1;
  return 4 * n + 4 * n + 8 * n + 4 * max_dst * (int64_t)fmax + 4 * max_dst * 3 + 4 * max_edges * 2 + 4 * nb + 64;
}

// sample_minibatch on the device. targets: device int64[nt]. Output at the
// capacity offsets of a packed sample: V^l at voff[l], E^l at eoff[l-1]
// (esrc/edst), sizes = [nV_0..nV_L, nE_1..nE_L] (device int64). ws: the
// scratch above, zero-filled once before the first call (generation stamps);
// gen0: a per-call base generation, advanced by L + 1 per call by the caller.
extern "C" int sg_gpu_sample(const int64_t* row_offsets, const int32_t* col_indices, int64_t n,
                             const int64_t* targets, int64_t nt, const int32_t* fanouts, int32_t L,
                             uint64_t seed, uint32_t gen0, const int64_t* voff, const int64_t* eoff_cap,
                             int64_t max_dst, int64_t max_edges, int32_t* V, int32_t* esrc, int32_t* edst,
                             int64_t* sizes, void* ws, int32_t* err, void* stream) {
  SG_REQUIRE(row_offsets && col_indices && targets && fanouts && V && esrc && edst && sizes && ws && err,
             "gpu_sample: null argument");
  SG_REQUIRE(L >= 1 && L <= SG_MAXL, "gpu_sample: 1 <= layers <= SG_MAXL");
  SG_REQUIRE(nt >= 1 && nt <= max_dst, "gpu_sample: target count out of range");
  int fmax = 1;
  for (int l = 0; l < L; ++l) {
    SG_REQUIRE(fanouts[l] >= 0 && fanouts[l] <= SMP_FMAX, "gpu_sample: fanout must be in [0, 64]");
    fmax = std::max(fmax, (int)fanouts[l]);
  }
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)ws;
  uint32_t* stamp = (uint32_t*)w; w += 4 * n;
  int32_t* pos = (int32_t*)w; w += 4 * n;
  unsigned long long* first = (unsigned long long*)w; w += 8 * n;
  int32_t* picks = (int32_t*)w; w += 4 * max_dst * (int64_t)fmax;
  int32_t* npk = (int32_t*)w; w += 4 * max_dst;
  int32_t* eoffs = (int32_t*)w; w += 4 * max_dst;
  w += 4 * max_dst;
  int32_t* isfirst = (int32_t*)w; w += 4 * max_edges;
  int32_t* newidx = (int32_t*)w; w += 4 * max_edges;
  const int64_t nbmax = (max_edges + SCAN_B - 1) / SCAN_B + 1;
  int32_t* bsum = (int32_t*)w; w += 4 * nbmax;
  int64_t* totals = (int64_t*)(((uintptr_t)w + 7) & ~(uintptr_t)7);  // [edges, new vertices]
  SG_CUDA(cudaMemsetAsync(err, 0, sizeof(int32_t), st));
  const int gd = clamp_grid(div_up(max_dst, 256), kSMs * 8);
  ::sg::launch(k_smp_targets, clamp_grid(div_up(nt, 256), kSMs), 256, 0, st, targets, nt, n, V, voff[L], sizes, L, err);
  SG_CHECK_LAUNCH("k_smp_targets");
  for (int l = L; l >= 1; --l) {
    SmpLayer s;
    s.l = l;
    s.f = std::max(1, (int)fanouts[l - 1]);
    s.gen = gen0 + (uint32_t)(L - l) + 1;
    s.seed = seed;
    s.cur_off = voff[l];
    s.prev_off = voff[l - 1];
    s.e_off = eoff_cap[l - 1];
    s.size_cur = l;
    s.size_prev = l - 1;
    s.size_e = L + 1 + (l - 1);
    s.cap_prev = voff[l] - voff[l - 1];
    s.cap_e = eoff_cap[l] - eoff_cap[l - 1];
    s.err = err;
    ::sg::launch(k_smp_mark, gd, 256, 0, st, (const int32_t*)V, (const int64_t*)sizes, s, stamp, pos);
    SG_CHECK_LAUNCH("k_smp_mark");
    if (fanouts[l - 1] > 0) {
      ::sg::launch(k_smp_pick, gd, 256, 0, st, (const int32_t*)V, (const int64_t*)sizes, s, row_offsets,
                   col_indices, picks, npk);
    } else {
      SmpLayer s1 = s;
      s1.f = 0;
      ::sg::launch(k_smp_pick, gd, 256, 0, st, (const int32_t*)V, (const int64_t*)sizes, s1, row_offsets,
                   col_indices, picks, npk);
    }
    SG_CHECK_LAUNCH("k_smp_pick");
    // eoff = exclusive scan of (1 + picks) over the destinations; total = |E^l|
    const int nbd = (int)((max_dst + SCAN_B - 1) / SCAN_B);
    ::sg::launch(k_scan_blocks, nbd, 256, 0, st, (const int32_t*)npk, (const int64_t*)sizes, l, (int64_t)0, bsum);
    ::sg::launch(k_scan_top, 1, 1024, 0, st, bsum, nbd, totals + 0);
    ::sg::launch(k_scan_local, nbd, 256, 0, st, (const int32_t*)npk, (const int64_t*)sizes, l, (int64_t)0,
                 (const int32_t*)bsum, eoffs);
    SG_CHECK_LAUNCH("sampler scan (edges)");
    ::sg::launch(k_smp_first, gd, 256, 0, st, (const int64_t*)sizes, s, (const int32_t*)picks, (const int32_t*)npk,
                 (const int32_t*)eoffs, (const uint32_t*)stamp, first);
    ::sg::launch(k_smp_isfirst, gd, 256, 0, st, (const int64_t*)sizes, s, (const int32_t*)picks,
                 (const int32_t*)npk, (const int32_t*)eoffs, (const uint32_t*)stamp,
                 (const unsigned long long*)first, isfirst);
    SG_CHECK_LAUNCH("k_smp_first/isfirst");
    // new-vertex indices: exclusive scan of the first-occurrence flags over E^l
    const int nbe = (int)((max_edges + SCAN_B - 1) / SCAN_B);
    ::sg::launch(k_scan_blocks, nbe, 256, 0, st, (const int32_t*)isfirst, (const int64_t*)totals, 0, (int64_t)0, bsum);
    ::sg::launch(k_scan_top, 1, 1024, 0, st, bsum, nbe, totals + 1);
    ::sg::launch(k_scan_local, nbe, 256, 0, st, (const int32_t*)isfirst, (const int64_t*)totals, 0, (int64_t)0,
                 (const int32_t*)bsum, newidx);
    SG_CHECK_LAUNCH("sampler scan (new vertices)");
    ::sg::launch(k_smp_assign, gd, 256, 0, st, V, sizes, s, (const int32_t*)picks, (const int32_t*)npk,
                 (const int32_t*)eoffs, (const int32_t*)isfirst, (const int32_t*)newidx, (const int64_t*)totals,
                 stamp, pos);
    ::sg::launch(k_smp_edges, gd, 256, 0, st, (const int64_t*)sizes, s, (const int32_t*)picks, (const int32_t*)npk,
                 (const int32_t*)eoffs, (const int32_t*)pos, esrc, edst);
    SG_CHECK_LAUNCH("k_smp_assign/edges");
  }
  return SG_OK;
}
