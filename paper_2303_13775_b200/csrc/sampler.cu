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

constexpr int SMP_FMAX = 64;  // max fanout (swap map <= 128 entries: 4 register slots per lane)

struct SmpLayer {
  int l, f;
  uint32_t gen_off;           // this layer's generation = *gen_dev + gen_off
  const uint32_t* gen_dev;    // per-call base generation (device: graph replays advance it)
  uint64_t seed;
  const uint64_t* seed_dev;   // if set, the seed is read from device memory (per replay)
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
  const uint32_t gen = *s.gen_dev + s.gen_off;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nc; i += gridDim.x * blockDim.x) {
    const int32_t v = V[s.cur_off + i];
    stamp[v] = gen;
    pos[v] = i;
  }
}

// One WARP per destination. The partial Fisher-Yates' sparse swap map
// (<= 2k entries) and the accepted list (<= k) live in registers spread over
// the lanes (4 map slots, 2 output slots per lane) and are searched with
// ballots; every random position r_j depends only on (seed, l, i, j, m), so
// all of them -- and the column entries at positions j and r_j -- are loaded
// in two parallel rounds before the (inherently sequential) swaps run.
// Semantically the same as the host sampler's per-thread loop (same order,
// same hash, same accept rules), so the output is identical.
__global__ void __launch_bounds__(256) k_smp_pick(const int32_t* __restrict__ V, const int64_t* __restrict__ sizes,
                                                  SmpLayer s, const int64_t* __restrict__ ro,
                                                  const int32_t* __restrict__ ci, int32_t* __restrict__ picks,
                                                  int32_t* __restrict__ npk) {
  SG_PDL_ENTRY();
  const int nc = nv_of(sizes, s.size_cur);
  const int f = s.f;
  const uint64_t seed = s.seed_dev ? *s.seed_dev : s.seed;
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = gw; i < nc; i += nw) {
    const int32_t v = V[s.cur_off + i];
    const int64_t s0 = ro[v];
    const int m = (int)(ro[v + 1] - s0);
    const int k = m < f ? m : f;
    int32_t outv0 = 0, outv1 = 0;
    int cnt = 0;
    auto accept = [&](int32_t u) {
      if (u == v) return;  // the input's own self-loop
      const unsigned b = __ballot_sync(0xffffffffu, (lane < cnt && outv0 == u) || (32 + lane < cnt && outv1 == u));
      if (b) return;  // parallel edge
      if (lane == (cnt & 31)) {
        if (cnt < 32) outv0 = u; else outv1 = u;
      }
      ++cnt;
    };
    if (k > 0 && k <= 32 && (k < m || m <= 32)) {
      // ---- all k steps at once (k <= 32, one lane per step). Step t swaps
      // positions t and r_t (r_t >= t); position t is never touched after
      // step t, so the pick of step j is the value at r_j before step j:
      // the value W(t) that the LAST earlier step t with r_t == r_j moved
      // there, else the column entry itself. W(t) (position t's value before
      // step t) is likewise the W of the last earlier step that targeted t,
      // else ci[t]: a chain resolved by pointer jumping. Duplicates / self
      // loops are then dropped keeping first occurrences (match_any), which
      // is exactly the sequential accept loop.
      __shared__ int lw_s[8][32];
      int* lw = lw_s[threadIdx.x >> 5];
      const bool act = lane < k;
      const int32_t pj = (lane < m && act) ? ci[s0 + lane] : 0;
      int r = -1 - lane;  // unique dummy for idle lanes
      int32_t pr = 0;
      if (k < m && act) {
        r = lane + (int)sg_bounded(sg_hash3(seed, ((uint64_t)s.l << 40) ^ (uint64_t)i, (uint64_t)lane),
                                   (uint64_t)(m - lane));
        pr = ci[s0 + r];
      }
      int32_t picked = pj;
      if (k < m) {
        const unsigned grp = __match_any_sync(0xffffffffu, r);
        const unsigned below = grp & lanemask_lt();
        const int prev = below ? 31 - __clz(below) : -1;
        lw[lane] = -1;
        __syncwarp();
        if (act && r < k && r != lane) atomicMax(&lw[r], lane);
        __syncwarp();
        int nxt = (act && lw[lane] >= 0) ? lw[lane] : lane;
#pragma unroll
        for (int it = 0; it < 5; ++it) nxt = __shfl_sync(0xffffffffu, nxt, nxt);
        const int32_t W = __shfl_sync(0xffffffffu, pj, nxt);
        const int32_t fromW = __shfl_sync(0xffffffffu, W, prev >= 0 ? prev : lane);
        picked = prev >= 0 ? fromW : pr;
      }
      const bool valid = act && picked != v;
      const unsigned g2 = __match_any_sync(0xffffffffu, valid ? picked : (int32_t)(-1 - lane));
      const bool first = valid && lane == __ffs(g2) - 1;
      const unsigned acc = __ballot_sync(0xffffffffu, first);
      if (first) picks[i * f + __popc(acc & lanemask_lt())] = picked;
      if (lane == 0) npk[i] = 1 + __popc(acc);
      continue;
    }
    if (k > 0) {
      // column entries at positions 0..63 (all that the take-all case and the
      // j positions of the partial shuffle need)
      const int32_t pj0 = lane < m ? ci[s0 + lane] : 0;
      const int32_t pj1 = 32 + lane < m ? ci[s0 + 32 + lane] : 0;
      if (k >= m) {
        for (int j = 0; j < m; ++j) accept(__shfl_sync(0xffffffffu, j < 32 ? pj0 : pj1, j & 31));
      } else {
        // r_j for j = lane, lane + 32 and the column entries there
        int r0 = 0, r1 = 0;
        if (lane < k)
          r0 = lane + (int)sg_bounded(sg_hash3(seed, ((uint64_t)s.l << 40) ^ (uint64_t)i, (uint64_t)lane),
                                      (uint64_t)(m - lane));
        if (32 + lane < k)
          r1 = 32 + lane + (int)sg_bounded(sg_hash3(seed, ((uint64_t)s.l << 40) ^ (uint64_t)i, (uint64_t)(32 + lane)),
                                           (uint64_t)(m - 32 - lane));
        const int32_t pr0 = lane < k ? ci[s0 + r0] : 0;
        const int32_t pr1 = 32 + lane < k ? ci[s0 + r1] : 0;
        int keys[4], vals[4];
        int nm = 0;
        auto find = [&](int x, int& slot) -> int {  // lane holding key x, or -1
          // only the occupied slots (one ballot while the map has <= 32 entries)
          unsigned b = __ballot_sync(0xffffffffu, lane < nm && keys[0] == x);
          if (b) {
            slot = 0;
            return __ffs(b) - 1;
          }
#pragma unroll
          for (int t = 1; t < 4; ++t) {
            if (t * 32 >= nm) break;
            b = __ballot_sync(0xffffffffu, t * 32 + lane < nm && keys[t] == x);
            if (b) {
              slot = t;
              return __ffs(b) - 1;
            }
          }
          return -1;
        };
        auto value_at = [&](int slot, int src) -> int {
          int mine = vals[0];
#pragma unroll
          for (int t = 1; t < 4; ++t)
            if (slot == t) mine = vals[t];
          return __shfl_sync(0xffffffffu, mine, src);
        };
        auto set = [&](int x, int val) {
          int slot = 0;
          const int at = find(x, slot);
          if (at >= 0) {
            if (lane == at) {
#pragma unroll
              for (int t = 0; t < 4; ++t)
                if (slot == t) vals[t] = val;
            }
            return;
          }
          if (lane == (nm & 31)) {
#pragma unroll
            for (int t = 0; t < 4; ++t)
              if ((nm >> 5) == t) {
                keys[t] = x;
                vals[t] = val;
              }
          }
          ++nm;
        };
        for (int j = 0; j < k; ++j) {
          const int r = __shfl_sync(0xffffffffu, j < 32 ? r0 : r1, j & 31);
          int slot = 0;
          int at = find(j, slot);
          const int vj = at >= 0 ? value_at(slot, at) : __shfl_sync(0xffffffffu, j < 32 ? pj0 : pj1, j & 31);
          at = find(r, slot);
          const int vr = at >= 0 ? value_at(slot, at) : __shfl_sync(0xffffffffu, j < 32 ? pr0 : pr1, j & 31);
          set(r, vj);
          set(j, vr);
          accept(vr);
        }
      }
    }
    int32_t* out = picks + i * f;
    if (lane < cnt) out[lane] = outv0;
    if (32 + lane < cnt) out[32 + lane] = outv1;
    if (lane == 0) npk[i] = 1 + cnt;  // the self edge plus the picks
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

// The per-pick kernels run one thread per (destination, pick slot): slot
// t < f is pick t of destination i (edge position eoff[i] + 1 + t), slot f is
// the destination's self edge (position eoff[i]).
__global__ void k_smp_first(const int64_t* __restrict__ sizes, SmpLayer s, const int32_t* __restrict__ picks,
                            const int32_t* __restrict__ npk, const int32_t* __restrict__ eoff,
                            const uint32_t* __restrict__ stamp, unsigned long long* __restrict__ first) {
  SG_PDL_ENTRY();
  const int nc = nv_of(sizes, s.size_cur);
  const int f = s.f;
  const uint32_t gen = *s.gen_dev + s.gen_off;
  const unsigned long long hi = (unsigned long long)(0xFFFFFFFFu - gen) << 32;
  const int64_t tot = (int64_t)nc * f;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < tot; x += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(x / f), t = (int)(x - (int64_t)i * f);
    if (t >= npk[i] - 1) continue;
    const int32_t u = picks[x];
    if (stamp[u] != gen) atomicMin(&first[u], hi | (unsigned)(eoff[i] + 1 + t));
  }
}

__global__ void k_smp_isfirst(const int64_t* __restrict__ sizes, SmpLayer s, const int32_t* __restrict__ picks,
                              const int32_t* __restrict__ npk, const int32_t* __restrict__ eoff,
                              const uint32_t* __restrict__ stamp, const unsigned long long* __restrict__ first,
                              int32_t* __restrict__ isfirst) {
  SG_PDL_ENTRY();
  const int nc = nv_of(sizes, s.size_cur);
  const int f = s.f, f1 = f + 1;
  const uint32_t gen = *s.gen_dev + s.gen_off;
  const unsigned long long hi = (unsigned long long)(0xFFFFFFFFu - gen) << 32;
  const int64_t tot = (int64_t)nc * f1;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < tot; x += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(x / f1), t = (int)(x - (int64_t)i * f1);
    const int c = npk[i] - 1, e0 = eoff[i];
    if (e0 + c >= s.cap_e) {  // E^l over capacity
      if (t == f) atomicOr(s.err, 2);
      continue;
    }
    if (t == f) {
      isfirst[e0] = 0;
    } else if (t < c) {
      const int32_t u = picks[(int64_t)i * f + t];
      const unsigned p = (unsigned)(e0 + 1 + t);
      isfirst[p] = (stamp[u] != gen && first[u] == (hi | p)) ? 1 : 0;
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
  const int f = s.f, f1 = f + 1;
  const uint32_t gen = *s.gen_dev + s.gen_off;
  const int64_t tot = (int64_t)nc * f1;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < tot; x += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(x / f1), t = (int)(x - (int64_t)i * f1);
    if (t == f) {
      V[s.prev_off + i] = V[s.cur_off + i];  // V^l is a prefix of V^{l-1}
      continue;
    }
    const int c = npk[i] - 1, e0 = eoff[i];
    if (t >= c || e0 + c >= s.cap_e) continue;
    const int p = e0 + 1 + t;
    if (!isfirst[p]) continue;
    const int32_t u = picks[(int64_t)i * f + t];
    const int j = nc + newidx[p];
    if (j >= s.cap_prev) {  // V^{l-1} over capacity
      atomicOr(s.err, 4);
      continue;
    }
    V[s.prev_off + j] = u;
    pos[u] = j;
    stamp[u] = gen;
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
  const int f = s.f, f1 = f + 1;
  const int64_t tot = (int64_t)nc * f1;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < tot; x += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(x / f1), t = (int)(x - (int64_t)i * f1);
    const int c = npk[i] - 1;
    if (eoff[i] + c >= s.cap_e) continue;
    const int64_t e0 = s.e_off + eoff[i];
    if (t == f) {
      esrc[e0] = i;
      edst[e0] = i;
    } else if (t < c) {
      esrc[e0 + 1 + t] = pos[picks[(int64_t)i * f + t]];
      edst[e0 + 1 + t] = i;
    }
  }
}

__global__ void k_smp_advance(uint32_t* gen_dev, uint32_t by) {
  SG_PDL_ENTRY();
  if (threadIdx.x == 0 && blockIdx.x == 0) *gen_dev += by;
}

}  // namespace
}  // namespace sg

using namespace sg;

// The per-call generation counter lives in its own 16-byte word at the end of
// the scratch (zeroed by sg_gpu_sampler_ws_init with the scratch size).
static uint32_t* gen_word(void* ws, int64_t ws_bytes) {
  return (uint32_t*)((char*)ws + ((ws_bytes - 16) & ~(int64_t)15));
}

// One-time scratch initialisation: generation stamps 0, first-occurrence keys
// all-ones (any current generation's key is smaller).
extern "C" int sg_gpu_sampler_ws_init(void* ws, int64_t n, int64_t ws_bytes, void* stream) {
  SG_REQUIRE(ws && n > 0 && ws_bytes >= 16 * n + 16, "gpu_sampler_ws_init: bad argument");
  cudaStream_t st = (cudaStream_t)stream;
  SG_CUDA(cudaMemsetAsync(ws, 0, 8 * (size_t)n, st));
  SG_CUDA(cudaMemsetAsync((char*)ws + 8 * n, 0xFF, 8 * (size_t)n, st));
  SG_CUDA(cudaMemsetAsync(gen_word(ws, ws_bytes), 0, 16, st));
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
                             uint64_t seed, const uint64_t* seed_dev, int64_t ws_bytes, const int64_t* voff,
                             const int64_t* eoff_cap,
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
    s.gen_off = (uint32_t)(L - l) + 1;
    s.gen_dev = gen_word(ws, ws_bytes);
    s.seed = seed;
    s.seed_dev = seed_dev;
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
    const int gw = clamp_grid(div_up(max_dst, 8), kSMs * 16);  // a warp per destination
    if (fanouts[l - 1] > 0) {
      ::sg::launch(k_smp_pick, gw, 256, 0, st, (const int32_t*)V, (const int64_t*)sizes, s, row_offsets,
                   col_indices, picks, npk);
    } else {
      SmpLayer s1 = s;
      s1.f = 0;
      ::sg::launch(k_smp_pick, gw, 256, 0, st, (const int32_t*)V, (const int64_t*)sizes, s1, row_offsets,
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
    const int gs = clamp_grid(div_up(max_dst * (int64_t)(s.f + 1), 256), kSMs * 8);  // per pick slot
    ::sg::launch(k_smp_first, gs, 256, 0, st, (const int64_t*)sizes, s, (const int32_t*)picks, (const int32_t*)npk,
                 (const int32_t*)eoffs, (const uint32_t*)stamp, first);
    ::sg::launch(k_smp_isfirst, gs, 256, 0, st, (const int64_t*)sizes, s, (const int32_t*)picks,
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
    ::sg::launch(k_smp_assign, gs, 256, 0, st, V, sizes, s, (const int32_t*)picks, (const int32_t*)npk,
                 (const int32_t*)eoffs, (const int32_t*)isfirst, (const int32_t*)newidx, (const int64_t*)totals,
                 stamp, pos);
    ::sg::launch(k_smp_edges, gs, 256, 0, st, (const int64_t*)sizes, s, (const int32_t*)picks, (const int32_t*)npk,
                 (const int32_t*)eoffs, (const int32_t*)pos, esrc, edst);
    SG_CHECK_LAUNCH("k_smp_assign/edges");
  }
  ::sg::launch(k_smp_advance, 1, 32, 0, st, gen_word(ws, ws_bytes), (uint32_t)(L + 1));
  SG_CHECK_LAUNCH("k_smp_advance");
  return SG_OK;
}
