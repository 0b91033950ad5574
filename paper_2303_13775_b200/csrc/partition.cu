// Balanced k-way partitioning on the GPU (partition.py:236-349 restated for
// the device): parallel label refinement on the symmetrised graph
// (weight(u,v) = arcs u->v + arcs v->u, self loops dropped, partition.py:123-136).
//
// A round: every eligible vertex (half of them, by a seeded hash, so two
// neighbours rarely move together) computes its connection to every part
// (one warp per vertex; lanes walk the in- and out-neighbours and count into
// shared memory), proposes the part with the largest strictly positive gain
// (lowest part id on ties, as partition.py:257-259), and the proposals are
// admitted per target part in descending gain while the part stays within
// the balance cap (gain histogram -> per-part threshold). The cut is measured
// after the round; a round that raised it is undone, so the cut history never
// increases (the reference's refinement guarantee, partition.py:273-295).
// Integer atomics only: the result is a deterministic function of the seed.
#include <cstring>

#include "common.cuh"
#include "rng.h"

namespace sg {
namespace {

constexpr int PG_MAX = 16;    // parts
constexpr int PG_GAINS = 64;  // gain histogram bins (gains >= 63 share the top bin)

__global__ void __launch_bounds__(256) k_part_propose(int64_t n, const int64_t* __restrict__ ro,
                                                      const int32_t* __restrict__ ci,
                                                      const int64_t* __restrict__ oro,
                                                      const int32_t* __restrict__ oci, int g,
                                                      const int32_t* __restrict__ part, uint64_t seed, int round,
                                                      int32_t* __restrict__ prop, int32_t* __restrict__ gainv,
                                                      unsigned* __restrict__ hist) {
  SG_PDL_ENTRY();
  __shared__ int conn_s[8][PG_MAX];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  int* conn = conn_s[wl];
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
    for (int64_t j = ro[v] + lane; j < ro[v + 1]; j += 32) {
      const int32_t u = ci[j];
      if (u != v) atomicAdd(&conn[part[u]], 1);
    }
    for (int64_t j = oro[v] + lane; j < oro[v + 1]; j += 32) {
      const int32_t u = oci[j];
      if (u != v) atomicAdd(&conn[part[u]], 1);
    }
    __syncwarp();
    const int a = part[v];
    const int ca = conn[a];
    // key = gain * 32 + (31 - p): max key -> largest gain, lowest part on ties
    int key = -1;
    if (lane < g && lane != a) {
      const int gain = conn[lane] - ca;
      if (gain > 0) key = gain * 32 + (31 - lane);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) key = max(key, __shfl_xor_sync(0xffffffffu, key, o));
    if (lane == 0) {
      if (key >= 0) {
        const int p = 31 - (key & 31), gain = key >> 5;
        prop[v] = p;
        gainv[v] = gain;
        atomicAdd(&hist[p * PG_GAINS + min(gain, PG_GAINS - 1)], 1u);
      } else {
        prop[v] = -1;
      }
    }
    __syncwarp();
  }
}

// per target part: the lowest gain threshold whose admitted moves fit the room
__global__ void k_part_threshold(const unsigned* __restrict__ hist, const int64_t* __restrict__ sizes, int g,
                                 int64_t cap, int* __restrict__ thr) {
  SG_PDL_ENTRY();
  const int p = threadIdx.x;
  if (p >= g) return;
  const int64_t room = cap - sizes[p];
  int64_t acc = 0;
  int t = PG_GAINS;  // admit nothing by default
  for (int b = PG_GAINS - 1; b >= 1; --b) {
    acc += hist[p * PG_GAINS + b];
    if (acc > room) break;
    t = b;
  }
  thr[p] = t;
}

__global__ void k_part_apply(int64_t n, const int32_t* __restrict__ prop, const int32_t* __restrict__ gainv,
                             const int* __restrict__ thr, int32_t* __restrict__ part,
                             unsigned long long* __restrict__ moved) {
  SG_PDL_ENTRY();
  unsigned cnt = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int p = prop[v];
    if (p >= 0 && min(gainv[v], PG_GAINS - 1) >= thr[p]) {
      part[v] = p;
      ++cnt;
    }
  }
  if (cnt) atomicAdd(moved, (unsigned long long)cnt);
}

__global__ void k_part_sizes(int64_t n, const int32_t* __restrict__ part, int g, int64_t* __restrict__ sizes) {
  SG_PDL_ENTRY();
  __shared__ unsigned loc[PG_MAX];
  if (threadIdx.x < PG_MAX) loc[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&loc[part[v]], 1u);
  __syncthreads();
  if (threadIdx.x < g && loc[threadIdx.x])
    atomicAdd((unsigned long long*)&sizes[threadIdx.x], (unsigned long long)loc[threadIdx.x]);
}

// directed arcs u -> v with part[u] != part[v] (== the symmetrised cut); a warp per vertex
__global__ void k_part_cut(int64_t n, const int64_t* __restrict__ ro, const int32_t* __restrict__ ci,
                           const int32_t* __restrict__ part, unsigned long long* __restrict__ cut) {
  SG_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long c = 0;
  for (int64_t v = gw; v < n; v += nw) {
    const int pv = part[v];
    for (int64_t j = ro[v] + lane; j < ro[v + 1]; j += 32) c += part[ci[j]] != pv;
  }
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0 && c) atomicAdd(cut, c);
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
  ::sg::launch(k_part_cut, clamp_grid(div_up(n, 8), kSMs * 16), 256, 0, st, n, row_offsets, col_indices, part, cut_out);
  SG_CHECK_LAUNCH("k_part_cut");
  return SG_OK;
}

// One refinement round (see the file comment). part is updated in place;
// sizes (int64[g]) is recomputed; ws >= 8 * n + 4 * (g * 64 + 64) bytes;
// moved_out receives the number of moved vertices (device).
extern "C" int sg_partition_round(const int64_t* row_offsets, const int32_t* col_indices,
                                  const int64_t* out_offsets, const int32_t* out_indices, int64_t n, int32_t g,
                                  int64_t cap, uint64_t seed, int32_t round, int32_t* part, int64_t* sizes,
                                  void* ws, unsigned long long* moved_out, void* stream) {
  SG_REQUIRE(row_offsets && col_indices && out_offsets && out_indices && part && sizes && ws && moved_out,
             "partition_round: null argument");
  SG_REQUIRE(g >= 1 && g <= PG_MAX, "partition_round: 1 <= parts <= 16");
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)ws;
  int32_t* prop = (int32_t*)w; w += 4 * n;
  int32_t* gainv = (int32_t*)w; w += 4 * n;
  unsigned* hist = (unsigned*)w; w += 4 * PG_MAX * PG_GAINS;
  int* thr = (int*)w;
  SG_CUDA(cudaMemsetAsync(hist, 0, 4 * PG_MAX * PG_GAINS, st));
  SG_CUDA(cudaMemsetAsync(moved_out, 0, sizeof(unsigned long long), st));
  if (n == 0) return SG_OK;
  ::sg::launch(k_part_propose, clamp_grid(div_up(n, 8), kSMs * 16), 256, 0, st, n, row_offsets, col_indices,
               out_offsets, out_indices, (int)g, (const int32_t*)part, seed, (int)round, prop, gainv, hist);
  SG_CHECK_LAUNCH("k_part_propose");
  ::sg::launch(k_part_threshold, 1, 32, 0, st, (const unsigned*)hist, (const int64_t*)sizes, (int)g, cap, thr);
  SG_CHECK_LAUNCH("k_part_threshold");
  ::sg::launch(k_part_apply, clamp_grid(div_up(n, 256), kSMs * 8), 256, 0, st, n, (const int32_t*)prop,
               (const int32_t*)gainv, (const int*)thr, part, moved_out);
  SG_CHECK_LAUNCH("k_part_apply");
  SG_CUDA(cudaMemsetAsync(sizes, 0, sizeof(int64_t) * g, st));
  ::sg::launch(k_part_sizes, clamp_grid(div_up(n, 256), kSMs * 4), 256, 0, st, n, (const int32_t*)part, (int)g, sizes);
  SG_CHECK_LAUNCH("k_part_sizes");
  return SG_OK;
}
