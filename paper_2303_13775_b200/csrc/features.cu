// GPU-resident partitioned feature cache (replaces _load_inputs,
// engine.py:160-167, and the host loads of transfer_manifest,
// scheduler.py:324-347).
//
// Each device's cache shard holds its own partition's rows (CacheState keeps
// cached vertices inside the owner partition, partition.py:85-91), so every
// layer-0 row a device aggregates is a local hit or one of its own misses.
// Instead of materialising h0 = features[owned_gids[0]], layer 1 reads the
// shard through a row-index indirection (src_row0), fused into the
// aggregation's loads.
#include "common.cuh"
#include "rng.h"

namespace sg {
namespace {

__global__ void k_layer0_rows(const SgMeta* __restrict__ meta, int d,
                              const int32_t* __restrict__ grouped, const int32_t* __restrict__ rank,
                              const int32_t* __restrict__ V, const int32_t* __restrict__ cache_slot,
                              int32_t miss_base, int64_t nVtot, int miss_global,
                              int32_t* __restrict__ src_row0) {
  SG_PDL_ENTRY();
  const int n = meta->n_own[0][d];
  const int own0 = meta->own_off[0][d];
  const int lbase = miss_global ? meta->load_off[d] : 0;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    const int p = grouped[own0 + q];
    const int32_t gid = V[p];
    int32_t slot = cache_slot ? cache_slot[gid] : gid;
    if (slot < 0) slot = miss_base + lbase + rank[nVtot + p];
    src_row0[own0 + q] = slot;
  }
}

__global__ void k_gather_rows(const float* __restrict__ table, const int32_t* __restrict__ rows,
                              int64_t n, int w, float* __restrict__ out) {
  SG_PDL_ENTRY();
  const int64_t total = n * w;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / w;
    const int c = (int)(i - r * w);
    out[i] = table[(int64_t)rows[r] * w + c];
  }
}

__global__ void k_fill_uniform(float* __restrict__ out, int64_t rows, int w, uint64_t seed,
                               int64_t row0) {
  SG_PDL_ENTRY();
  const int64_t total = rows * w;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / w;
    const int c = (int)(i - r * w);
    out[i] = sg_uniform24(seed, (uint64_t)(row0 + r), (uint64_t)c);
  }
}

// Cache misses (the reference's load_gids, scheduler.py:193-203, loaded from
// the host by _load_inputs, engine.py:160-167): one warp per missed layer-0
// row of devices [d0, d1) reads the row straight from host feature memory
// mapped into the device address space (zero-copy over PCIe / C2C, 16 B per
// lane, a whole row in flight per warp) into the staging row n_cached + q, q
// the global load index -- the numbering k_layer0_rows assigns. Sizes come
// from the device SgMeta, so the staging is part of a captured step.
template <int VEC>
__global__ void __launch_bounds__(256) k_stage_misses(const SgMeta* __restrict__ meta, int d0, int d1,
                                                      const int32_t* __restrict__ grouped,
                                                      const int32_t* __restrict__ V, int64_t nVtot,
                                                      const float* __restrict__ host, int F,
                                                      float* __restrict__ table, int stride, int n_cached) {
  SG_PDL_ENTRY();
  const int q0 = meta->load_off[d0], q1 = meta->load_off[d1];
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int nv = F / VEC;
  for (int q = q0 + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5); q < q1; q += nw) {
    const int64_t gid = V[grouped[nVtot + q]];
    float* dst = table + (int64_t)(n_cached + q) * stride;
    const float* src = host + gid * F;
    if (VEC == 4) {
      for (int c = lane; c < nv; c += 32)
        reinterpret_cast<float4*>(dst)[c] = reinterpret_cast<const float4*>(src)[c];
    } else {
      for (int c = lane; c < F; c += 32) dst[c] = src[c];
    }
  }
}

}  // namespace

extern "C" int sg_layer0_rows(const void* split_ws, const SgSplitLayout* lay, int32_t d,
                              const int32_t* V, const int32_t* cache_slot, int32_t miss_base,
                              int32_t* src_row0, void* stream) {
  SG_REQUIRE(split_ws && lay, "layer0_rows: null workspace");
  const char* base = (const char*)split_ws;
  const SgSplitLayout& y = *lay;
  SG_REQUIRE(d >= 0 && d < y.g, "layer0_rows: bad device");
  if (y.nV[0] <= 0) return SG_OK;
  // miss_base < 0 encodes "per-device staging" (dist mode): staging index is
  // the rank inside this device's load list; otherwise the global load index.
  const int miss_global = miss_base >= 0 ? 1 : 0;
  const int32_t mb = miss_base >= 0 ? miss_base : -miss_base - 1;
  ::sg::launch(k_layer0_rows, clamp_grid(div_up(y.nV[0], 256), kSMs * 8), 256, 0, (cudaStream_t)stream, (const SgMeta*)(base + y.o_meta), d, (const int32_t*)(base + y.o_grouped),
      (const int32_t*)(base + y.o_rank), V, cache_slot, mb, y.nVtot, miss_global, src_row0);
  SG_CHECK_LAUNCH("k_layer0_rows");
  return SG_OK;
}

extern "C" int sg_stage_misses(const void* split_ws, const SgSplitLayout* lay, int32_t d0, int32_t d1,
                               const int32_t* V, const float* host_feats, int32_t feat_dim,
                               float* table, int32_t row_stride, int32_t n_cached,
                               int64_t staging_rows, void* stream) {
  SG_REQUIRE(split_ws && lay && V && host_feats && table, "stage_misses: null argument");
  const SgSplitLayout& y = *lay;
  SG_REQUIRE(d0 >= 0 && d0 <= d1 && d1 <= y.g, "stage_misses: bad device range");
  SG_REQUIRE(feat_dim > 0 && row_stride >= feat_dim, "stage_misses: bad row width");
  // every load-list entry is a distinct layer-0 position: nV[0] rows always suffice
  SG_REQUIRE(staging_rows >= y.nV[0], "stage_misses: staging area smaller than the layer-0 capacity");
  if (y.nV[0] <= 0 || d0 == d1) return SG_OK;
  const char* base = (const char*)split_ws;
  const bool vec = (feat_dim % 4 == 0) && (row_stride % 4 == 0) &&
                   ((uintptr_t)host_feats % 16 == 0) && ((uintptr_t)table % 16 == 0);
  const int grid = (int)clamp_grid(div_up(y.nV[0], 8), kSMs * 8);
  if (vec)
    ::sg::launch(k_stage_misses<4>, grid, 256, 0, (cudaStream_t)stream, (const SgMeta*)(base + y.o_meta), d0, d1,
                 (const int32_t*)(base + y.o_grouped), V, y.nVtot, host_feats, (int)feat_dim, table,
                 (int)row_stride, (int)n_cached);
  else
    ::sg::launch(k_stage_misses<1>, grid, 256, 0, (cudaStream_t)stream, (const SgMeta*)(base + y.o_meta), d0, d1,
                 (const int32_t*)(base + y.o_grouped), V, y.nVtot, host_feats, (int)feat_dim, table,
                 (int)row_stride, (int)n_cached);
  SG_CHECK_LAUNCH("k_stage_misses");
  return SG_OK;
}

// Host feature memory mapped for the zero-copy miss gather: page-locks a
// caller-owned host range (cudaHostRegisterMapped, read-only) and returns the
// device address of its first byte.
extern "C" int sg_host_map(void* host_ptr, int64_t bytes, void** dev_ptr) {
  SG_REQUIRE(host_ptr && bytes > 0 && dev_ptr, "host_map: bad argument");
  cudaError_t e = cudaHostRegister(host_ptr, (size_t)bytes,
                                   cudaHostRegisterMapped | cudaHostRegisterPortable | cudaHostRegisterReadOnly);
  if (e == cudaErrorHostMemoryAlreadyRegistered) {
    (void)cudaGetLastError();
  } else if (e != cudaSuccess) {
    (void)cudaGetLastError();
    // some platforms reject the read-only hint: retry without it
    e = cudaHostRegister(host_ptr, (size_t)bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      set_error(std::string("host_map: cudaHostRegister failed: ") + cudaGetErrorString(e));
      return SG_ERR_CUDA;
    }
  }
  e = cudaHostGetDevicePointer(dev_ptr, host_ptr, 0);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    set_error(std::string("host_map: cudaHostGetDevicePointer failed: ") + cudaGetErrorString(e));
    return SG_ERR_CUDA;
  }
  return SG_OK;
}

extern "C" int sg_host_unmap(void* host_ptr) {
  if (!host_ptr) return SG_OK;
  cudaError_t e = cudaHostUnregister(host_ptr);
  if (e != cudaSuccess) (void)cudaGetLastError();
  return SG_OK;
}

extern "C" int sg_gather_rows(const float* table, const int32_t* rows, int64_t n_rows,
                              int32_t width, float* out, void* stream) {
  if (n_rows <= 0 || width <= 0) return SG_OK;
  ::sg::launch(k_gather_rows, clamp_grid(div_up(n_rows * width, 256), kSMs * 8), 256, 0,
                  (cudaStream_t)stream, table, rows, n_rows, width, out);
  SG_CHECK_LAUNCH("k_gather_rows");
  return SG_OK;
}

extern "C" int sg_fill_uniform(float* out, int64_t rows, int32_t width, uint64_t seed,
                               int64_t row0, void* stream) {
  if (rows <= 0 || width <= 0) return SG_OK;
  ::sg::launch(k_fill_uniform, clamp_grid(div_up(rows * width, 256), kSMs * 16), 256, 0,
                   (cudaStream_t)stream, out, rows, width, seed, row0);
  SG_CHECK_LAUNCH("k_fill_uniform");
  return SG_OK;
}

}  // namespace sg
