// split_cost (scheduler.py:257-309): per-layer communication cost C[v^l]
// (number of foreign devices holding a source of v's in-edges),
// per-device edge counts, local-edge counts.
//
//   k_cost_edges  one thread per sampled edge: devices of its source and
//                 destination through the uint8 partition map; per-CTA shared
//                 histograms of source devices and local edges, flushed with
//                 one integer atomic per bin; a foreign source sets bit
//                 sdev of the destination's 16-bit device mask (atomicOr).
//   k_cost_rows   one thread per destination: C[v] = popcount(mask), per-CTA
//                 sums -> one atomic per layer.
// Integer atomics only: results are exact and schedule-independent.
#include <algorithm>
#include <cstring>

#include "common.cuh"

namespace sg {
namespace {

struct CostGeom {
  int L, g;
  int64_t voff[SG_MAXL + 2];
  int64_t eoff[SG_MAXL + 1];
  int64_t moff[SG_MAXL + 1];  // destination-mask offset of layer l (1..L) at [l-1]
};

__global__ void __launch_bounds__(256) k_cost_edges(const int32_t* __restrict__ V,
                                                    const int32_t* __restrict__ esrc,
                                                    const int32_t* __restrict__ edst,
                                                    const uint8_t* __restrict__ asn, int64_t n_asn,
                                                    CostGeom cg, uint32_t* __restrict__ mask,
                                                    unsigned long long* __restrict__ counts,
                                                    unsigned long long* __restrict__ local,
                                                    int* __restrict__ err) {
  SG_PDL_ENTRY();
  __shared__ unsigned int hist[SG_MAXL * SG_MAXG];
  __shared__ unsigned int loc[SG_MAXL];
  const int L = cg.L, g = cg.g;
  for (int i = threadIdx.x; i < L * g; i += blockDim.x) hist[i] = 0;
  if (threadIdx.x < L) loc[threadIdx.x] = 0;
  __syncthreads();
  const int64_t nE = cg.eoff[L];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nE; e += (int64_t)gridDim.x * blockDim.x) {
    int l = 1;
    while (l < L && e >= cg.eoff[l]) ++l;  // edge e belongs to E^l (eoff[l-1] <= e < eoff[l])
    const int64_t gs = V[cg.voff[l - 1] + esrc[e]];
    const int64_t gd = V[cg.voff[l] + edst[e]];
    if (gs < 0 || gs >= n_asn || gd < 0 || gd >= n_asn) {
      atomicOr(err, 1);
      continue;
    }
    const int sd = asn[gs], dd = asn[gd];
    atomicAdd(&hist[(l - 1) * g + sd], 1u);
    if (sd == dd) {
      atomicAdd(&loc[l - 1], 1u);
    } else {
      atomicOr(&mask[cg.moff[l - 1] + edst[e]], 1u << sd);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < L * g; i += blockDim.x)
    if (hist[i]) atomicAdd(&counts[i], (unsigned long long)hist[i]);
  if (threadIdx.x < L && loc[threadIdx.x]) atomicAdd(&local[threadIdx.x], (unsigned long long)loc[threadIdx.x]);
}

__global__ void __launch_bounds__(256) k_cost_rows(const uint32_t* __restrict__ mask, CostGeom cg,
                                                   int32_t* __restrict__ cost_rows,
                                                   unsigned long long* __restrict__ cost) {
  SG_PDL_ENTRY();
  __shared__ unsigned int tot[SG_MAXL];
  const int L = cg.L;
  if (threadIdx.x < L) tot[threadIdx.x] = 0;
  __syncthreads();
  const int64_t n = cg.moff[L];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int l = 1;
    while (l < L && i >= cg.moff[l]) ++l;
    const int c = __popc(mask[i]);
    cost_rows[i] = c;
    if (c) atomicAdd(&tot[l - 1], (unsigned int)c);
  }
  __syncthreads();
  if (threadIdx.x < L && tot[threadIdx.x]) atomicAdd(&cost[threadIdx.x], (unsigned long long)tot[threadIdx.x]);
}

}  // namespace
}  // namespace sg

using namespace sg;

extern "C" int sg_split_cost(const int32_t* V, const int32_t* esrc, const int32_t* edst, const int64_t* nV,
                             const int64_t* nE, int32_t L, const uint8_t* assignment, int64_t n_vertices,
                             int32_t g, uint32_t* mask_ws, int32_t* cost_rows, int64_t* counts,
                             int64_t* local, int64_t* cost, int32_t* err, void* stream) {
  SG_REQUIRE(L >= 1 && L <= SG_MAXL, "split_cost: 1 <= layers <= SG_MAXL");
  SG_REQUIRE(g >= 1 && g <= SG_MAXG, "split_cost: 1 <= devices <= SG_MAXG");
  SG_REQUIRE(V && esrc && edst && nV && nE && assignment && mask_ws && cost_rows && counts && local && cost && err,
             "split_cost: null argument");
  CostGeom cg;
  memset(&cg, 0, sizeof(cg));
  cg.L = L;
  cg.g = g;
  for (int l = 0; l <= L; ++l) cg.voff[l + 1] = cg.voff[l] + nV[l];
  for (int l = 0; l < L; ++l) cg.eoff[l + 1] = cg.eoff[l] + nE[l];
  for (int l = 1; l <= L; ++l) cg.moff[l] = cg.moff[l - 1] + nV[l];
  cudaStream_t st = (cudaStream_t)stream;
  SG_CUDA(cudaMemsetAsync(mask_ws, 0, sizeof(uint32_t) * (size_t)std::max<int64_t>(cg.moff[L], 1), st));
  SG_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * (size_t)L * g, st));
  SG_CUDA(cudaMemsetAsync(local, 0, sizeof(int64_t) * (size_t)L, st));
  SG_CUDA(cudaMemsetAsync(cost, 0, sizeof(int64_t) * (size_t)L, st));
  SG_CUDA(cudaMemsetAsync(err, 0, sizeof(int32_t), st));
  if (cg.eoff[L] > 0) {
    ::sg::launch(k_cost_edges, clamp_grid(div_up(cg.eoff[L], 256), kSMs * 4), 256, 0, st, V, esrc, edst, assignment,
                 n_vertices, cg, mask_ws, (unsigned long long*)counts, (unsigned long long*)local, err);
    SG_CHECK_LAUNCH("k_cost_edges");
  }
  if (cg.moff[L] > 0) {
    ::sg::launch(k_cost_rows, clamp_grid(div_up(cg.moff[L], 256), kSMs * 4), 256, 0, st, (const uint32_t*)mask_ws,
                 cg, cost_rows, (unsigned long long*)cost);
    SG_CHECK_LAUNCH("k_cost_rows");
  }
  return SG_OK;
}
