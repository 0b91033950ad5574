// Balanced k-way partitioning on the GPU (the contract of reference
// partition.py:236-349, restated for the device as a parallel multilevel
// scheme; the host driver is partition.py, the coarsest level csrc/host.cpp).
//
// Every level is a symmetric weighted CSR (off, nbr, wt) with vertex weights
// vw: level 0 is the input graph symmetrised (weight(u,v) = arcs u->v + arcs
// v->u, self loops dropped, partition.py:123-136); coarser levels come from
// contracting a matching.
//
// * Matching (k_hem_pick / k_hem_commit): every unmatched vertex picks its
//   heaviest unmatched neighbour whose merged weight stays under the cap
//   (ties by a hash that is SYMMETRIC in the pair, so both ends rank an edge
//   the same); an edge picked from both ends (a locally dominant edge) is
//   matched. A few rounds match most vertices without sequential order.
// * Refinement round (k_pw_propose / k_pw_threshold / k_pw_apply): a seeded
//   half of the vertices (so two neighbours rarely move together) computes
//   its connection to every part (one warp per vertex, lanes accumulate the
//   edge weights in shared memory), proposes the part with the largest
//   strictly positive gain (lowest part id on ties, as partition.py:257-259);
//   proposals are admitted per target part in descending gain while the part
//   weight stays within the balance cap (weighted gain histogram -> per-part
//   threshold). The host measures the cut after the round and undoes a round
//   that raised it, so the cut history never increases (partition.py:273-295).
// Integer atomics only: every result is a deterministic function of the seed.
#include <cstring>

#include "common.cuh"
#include "rng.h"

namespace sg {
namespace {

constexpr int PG_MAX = 16;    // parts
constexpr int PG_GAINS = 64;  // gain bins: 1..31 exact, then one bin per power of two

__device__ __forceinline__ int gain_bin(long long gain) {
  if (gain < 32) return (int)gain;
  const int lg = 63 - __clzll(gain);  // >= 5
  return min(PG_GAINS - 1, 27 + lg);
}

__global__ void __launch_bounds__(256) k_pw_propose(int64_t n, const int64_t* __restrict__ off,
                                                    const int32_t* __restrict__ nbr, const int32_t* __restrict__ wt,
                                                    const int32_t* __restrict__ vw, int g,
                                                    const int32_t* __restrict__ part, uint64_t seed, int round,
                                                    int32_t* __restrict__ prop, int32_t* __restrict__ binv,
                                                    unsigned long long* __restrict__ hist) {
  SG_PDL_ENTRY();
  __shared__ long long conn_s[8][PG_MAX];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  long long* conn = conn_s[wl];
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = gw; v < n; v += nw) {
    const bool eligible = (sg_hash3(seed, (uint64_t)v, (uint64_t)round) & 1) == 0;
    if (!eligible) {
      if (lane == 0) prop[v] = -1;
      continue;
    }
    if (lane < PG_MAX) conn[lane] = 0;
    __syncwarp();
    for (int64_t j = off[v] + lane; j < off[v + 1]; j += 32)
      atomicAdd((unsigned long long*)&conn[part[nbr[j]]], (unsigned long long)wt[j]);
    __syncwarp();
    const int a = part[v];
    const long long ca = conn[a];
    // key = gain * 32 + (31 - p): max key -> largest gain, lowest part on ties
    long long key = -1;
    if (lane < g && lane != a) {
      const long long gain = conn[lane] - ca;
      if (gain > 0) key = gain * 32 + (31 - lane);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) key = max(key, (long long)__shfl_xor_sync(0xffffffffu, key, o));
    if (lane == 0) {
      if (key >= 0) {
        const int p = 31 - (int)(key & 31);
        const int b = gain_bin(key >> 5);
        prop[v] = p;
        binv[v] = b;
        atomicAdd(&hist[p * PG_GAINS + b], (unsigned long long)vw[v]);
      } else {
        prop[v] = -1;
      }
    }
    __syncwarp();
  }
}

// per target part: the lowest gain bin whose admitted moves (by weight) fit the room
__global__ void k_pw_threshold(const unsigned long long* __restrict__ hist, const int64_t* __restrict__ sizes,
                               int g, int64_t cap, int* __restrict__ thr) {
  SG_PDL_ENTRY();
  const int p = threadIdx.x;
  if (p >= g) return;
  const int64_t room = cap - sizes[p];
  int64_t acc = 0;
  int t = PG_GAINS;  // admit nothing by default
  for (int b = PG_GAINS - 1; b >= 1; --b) {
    acc += (int64_t)hist[p * PG_GAINS + b];
    if (acc > room) break;
    t = b;
  }
  thr[p] = t;
}

__global__ void k_pw_apply(int64_t n, const int32_t* __restrict__ prop, const int32_t* __restrict__ binv,
                           const int* __restrict__ thr, int32_t* __restrict__ part,
                           unsigned long long* __restrict__ moved) {
  SG_PDL_ENTRY();
  unsigned cnt = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int p = prop[v];
    if (p >= 0 && binv[v] >= thr[p]) {
      part[v] = p;
      ++cnt;
    }
  }
  if (cnt) atomicAdd(moved, (unsigned long long)cnt);
}

__global__ void k_pw_sizes(int64_t n, const int32_t* __restrict__ part, const int32_t* __restrict__ vw, int g,
                           int64_t* __restrict__ sizes) {
  SG_PDL_ENTRY();
  __shared__ unsigned long long loc[PG_MAX];
  if (threadIdx.x < PG_MAX) loc[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&loc[part[v]], (unsigned long long)(vw ? vw[v] : 1));
  __syncthreads();
  if (threadIdx.x < g && loc[threadIdx.x]) atomicAdd((unsigned long long*)&sizes[threadIdx.x], loc[threadIdx.x]);
}

// sum of wt over CSR entries whose endpoints lie in different parts; a warp per vertex
__global__ void k_pw_cut(int64_t n, const int64_t* __restrict__ off, const int32_t* __restrict__ nbr,
                         const int32_t* __restrict__ wt, const int32_t* __restrict__ part,
                         unsigned long long* __restrict__ cut) {
  SG_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long c = 0;
  for (int64_t v = gw; v < n; v += nw) {
    const int pv = part[v];
    for (int64_t j = off[v] + lane; j < off[v + 1]; j += 32)
      if (part[nbr[j]] != pv) c += wt ? (unsigned long long)wt[j] : 1ull;
  }
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0 && c) atomicAdd(cut, c);
}

// ---- heavy-edge matching
__global__ void __launch_bounds__(256) k_hem_pick(int64_t n, const int64_t* __restrict__ off,
                                                  const int32_t* __restrict__ nbr, const int32_t* __restrict__ wt,
                                                  const int32_t* __restrict__ vw, const int32_t* __restrict__ match,
                                                  int64_t wcap, uint64_t seed, int round,
                                                  int32_t* __restrict__ pick) {
  SG_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = gw; u < n; u += nw) {
    if (match[u] >= 0) {
      if (lane == 0) pick[u] = -1;
      continue;
    }
    const int64_t wu = vw[u];
    // key: weight in the high 32 bits, a pair-symmetric hash below; -1 = none
    long long best = -1;
    int bv = -1;
    for (int64_t j = off[u] + lane; j < off[u + 1]; j += 32) {
      const int32_t v = nbr[j];
      if (v == u || match[v] >= 0 || wu + vw[v] > wcap) continue;
      const uint64_t lo = (uint64_t)min((int64_t)v, u), hi = (uint64_t)max((int64_t)v, u);
      const long long key = ((long long)wt[j] << 31) | (long long)(sg_hash3(seed ^ (uint64_t)round, lo, hi) >> 33);
      if (key > best) {
        best = key;
        bv = v;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const long long ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int ov = __shfl_xor_sync(0xffffffffu, bv, o);
      if (ob > best || (ob == best && ov < bv)) {
        best = ob;
        bv = ov;
      }
    }
    if (lane == 0) pick[u] = bv;
  }
}

__global__ void k_hem_commit(int64_t n, const int32_t* __restrict__ pick, int32_t* __restrict__ match,
                             unsigned long long* __restrict__ matched) {
  SG_PDL_ENTRY();
  unsigned cnt = 0;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
    const int v = pick[u];
    if (v >= 0 && pick[v] == u) {
      match[u] = v;
      ++cnt;
    }
  }
  if (cnt) atomicAdd(matched, (unsigned long long)cnt);
}

}  // namespace
}  // namespace sg

using namespace sg;

// Cut (directed arcs across parts) of `part` on the device in-CSR.
extern "C" int sg_partition_cut(const int64_t* row_offsets, const int32_t* col_indices, int64_t n,
                                const int32_t* part, unsigned long long* cut_out, void* stream) {
  SG_REQUIRE(row_offsets && col_indices && part && cut_out && n >= 0, "partition_cut: null argument");
  cudaStream_t st = (cudaStream_t)stream;
  SG_CUDA(cudaMemsetAsync(cut_out, 0, sizeof(unsigned long long), st));
  if (n == 0) return SG_OK;
  ::sg::launch(k_pw_cut, clamp_grid(div_up(n, 8), kSMs * 16), 256, 0, st, n, row_offsets, col_indices,
               (const int32_t*)nullptr, part, cut_out);
  SG_CHECK_LAUNCH("k_pw_cut");
  return SG_OK;
}

// Weighted cut of a symmetric level graph: sum of wt over entries across parts
// (= 2 x the directed cut at level 0, where wt counts arcs).
extern "C" int sg_partition_cut_w(const int64_t* off, const int32_t* nbr, const int32_t* wt, int64_t n,
                                  const int32_t* part, unsigned long long* cut_out, void* stream) {
  SG_REQUIRE(off && nbr && wt && part && cut_out && n >= 0, "partition_cut_w: null argument");
  cudaStream_t st = (cudaStream_t)stream;
  SG_CUDA(cudaMemsetAsync(cut_out, 0, sizeof(unsigned long long), st));
  if (n == 0) return SG_OK;
  ::sg::launch(k_pw_cut, clamp_grid(div_up(n, 8), kSMs * 16), 256, 0, st, n, off, nbr, wt, part, cut_out);
  SG_CHECK_LAUNCH("k_pw_cut");
  return SG_OK;
}

// Part weights (int64[g]) of `part` under vertex weights vw (nullable: 1 each).
extern "C" int sg_partition_sizes(const int32_t* part, const int32_t* vw, int64_t n, int32_t g, int64_t* sizes,
                                  void* stream) {
  SG_REQUIRE(part && sizes && n >= 0, "partition_sizes: null argument");
  SG_REQUIRE(g >= 1 && g <= PG_MAX, "partition_sizes: 1 <= parts <= 16");
  cudaStream_t st = (cudaStream_t)stream;
  SG_CUDA(cudaMemsetAsync(sizes, 0, sizeof(int64_t) * g, st));
  if (n == 0) return SG_OK;
  ::sg::launch(k_pw_sizes, clamp_grid(div_up(n, 256), kSMs * 4), 256, 0, st, n, part, vw, (int)g, sizes);
  SG_CHECK_LAUNCH("k_pw_sizes");
  return SG_OK;
}

// One refinement round on a symmetric weighted level graph (see the file
// comment). part is updated in place; sizes (int64[g], part weights) is
// recomputed; ws >= 8 * n + 8 * 16 * 64 + 64 bytes; *moved_out = moved vertices.
extern "C" int sg_partition_round(const int64_t* off, const int32_t* nbr, const int32_t* wt, const int32_t* vw,
                                  int64_t n, int32_t g, int64_t cap, uint64_t seed, int32_t round, int32_t* part,
                                  int64_t* sizes, void* ws, unsigned long long* moved_out, void* stream) {
  SG_REQUIRE(off && nbr && wt && vw && part && sizes && ws && moved_out, "partition_round: null argument");
  SG_REQUIRE(g >= 1 && g <= PG_MAX, "partition_round: 1 <= parts <= 16");
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)ws;
  unsigned long long* hist = (unsigned long long*)w; w += 8 * PG_MAX * PG_GAINS;
  int* thr = (int*)w; w += 64;
  int32_t* prop = (int32_t*)w; w += 4 * n;
  int32_t* binv = (int32_t*)w;
  SG_CUDA(cudaMemsetAsync(hist, 0, 8 * PG_MAX * PG_GAINS, st));
  SG_CUDA(cudaMemsetAsync(moved_out, 0, sizeof(unsigned long long), st));
  if (n == 0) return SG_OK;
  ::sg::launch(k_pw_propose, clamp_grid(div_up(n, 8), kSMs * 16), 256, 0, st, n, off, nbr, wt, vw, (int)g,
               (const int32_t*)part, seed, (int)round, prop, binv, hist);
  SG_CHECK_LAUNCH("k_pw_propose");
  ::sg::launch(k_pw_threshold, 1, 32, 0, st, (const unsigned long long*)hist, (const int64_t*)sizes, (int)g, cap,
               thr);
  SG_CHECK_LAUNCH("k_pw_threshold");
  ::sg::launch(k_pw_apply, clamp_grid(div_up(n, 256), kSMs * 8), 256, 0, st, n, (const int32_t*)prop,
               (const int32_t*)binv, (const int*)thr, part, moved_out);
  SG_CHECK_LAUNCH("k_pw_apply");
  return sg_partition_sizes(part, vw, n, g, sizes, stream);
}

// One heavy-edge matching round: unmatched vertices (match < 0) pick their
// heaviest unmatched neighbour with vw[u] + vw[v] <= wcap; mutual picks are
// matched (match[u] = v, match[v] = u). ws >= 4 * n bytes; *matched_out =
// vertices matched in this round (device, accumulated: zero it first).
extern "C" int sg_partition_match_round(const int64_t* off, const int32_t* nbr, const int32_t* wt,
                                        const int32_t* vw, int64_t n, int64_t wcap, uint64_t seed, int32_t round,
                                        int32_t* match, void* ws, unsigned long long* matched_out, void* stream) {
  SG_REQUIRE(off && nbr && wt && vw && match && ws && matched_out, "partition_match_round: null argument");
  cudaStream_t st = (cudaStream_t)stream;
  if (n == 0) return SG_OK;
  int32_t* pick = (int32_t*)ws;
  ::sg::launch(k_hem_pick, clamp_grid(div_up(n, 8), kSMs * 16), 256, 0, st, n, off, nbr, wt, vw,
               (const int32_t*)match, wcap, seed, (int)round, pick);
  SG_CHECK_LAUNCH("k_hem_pick");
  ::sg::launch(k_hem_commit, clamp_grid(div_up(n, 256), kSMs * 8), 256, 0, st, n, (const int32_t*)pick, match,
               matched_out);
  SG_CHECK_LAUNCH("k_hem_commit");
  return SG_OK;
}
