// Exchange helpers for the push-to-owner / push-from-owner rounds
// (engine.py:121-156, scatter_shuffle_forward engine.py:591-630).
//
// Layer-l payload slots are holder-major ("pair slots": holder s's send buffer
// is slots [ref_off[s], ref_off[s+1]), ordered by owner then gid), receive
// slots are owner-major (owner o's buffer is [recv_off[o], recv_off[o+1]),
// ordered by sender then gid). xfer[slot] gives the receive slot. On one GPU
// (all devices in one process) the transport is one copy kernel; across GPUs
// the same buffers are handed to NCCL all-to-all-v (one message per peer,
// PAPER.md:820 "data coalescing").
#include "common.cuh"

namespace sg {
namespace {

__global__ void k_xfer(const SgMeta* __restrict__ meta, int l, const int32_t* __restrict__ xfer,
                       const float* __restrict__ in, float* __restrict__ out, int stride,
                       int forward) {
  SG_PDL_ENTRY();
  const int n = meta->npairs[l];
  const int64_t total = (int64_t)n * stride;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int slot = (int)(i / stride);
    const int c = (int)(i - (int64_t)slot * stride);
    const int rs = xfer[slot];
    if (forward) out[(int64_t)rs * stride + c] = in[i];
    else out[i] = in[(int64_t)rs * stride + c];
  }
}

__global__ void k_pack_from_owner(const SgMeta* __restrict__ meta, int l, int d,
                                  const int32_t* __restrict__ recv_row,
                                  const float* __restrict__ rows, int w, float* __restrict__ out,
                                  int stride) {
  SG_PDL_ENTRY();
  const int b = meta->recv_off[l][d], e = meta->recv_off[l][d + 1];
  const int64_t total = (int64_t)(e - b) * w;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i / w);
    const int c = (int)(i - (int64_t)k * w);
    const int rs = b + k;
    out[(int64_t)rs * stride + c] = rows[(int64_t)recv_row[rs] * w + c];
  }
}

__global__ void k_unpack_refs(const SgMeta* __restrict__ meta, int l, int d,
                              const int32_t* __restrict__ sendpos, const float* __restrict__ in,
                              int stride, int w, float* __restrict__ out) {
  SG_PDL_ENTRY();
  const int n = meta->n_ref[l][d];
  const int r0 = meta->ref_off[l][d];
  const int64_t total = (int64_t)n * w;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i / w);
    const int c = (int)(i - (int64_t)k * w);
    out[(int64_t)(r0 + k) * w + c] = in[(int64_t)sendpos[r0 + k] * stride + c];
  }
}

}  // namespace

extern "C" int sg_xfer_to_owner(const void* split_ws, const SgSplitLayout* lay, int32_t l,
                                const float* sendbuf, float* recvbuf, int32_t stride,
                                void* stream) {
  SG_REQUIRE(split_ws && lay, "xfer: null workspace");
  const char* base = (const char*)split_ws;
  const SgSplitLayout& y = *lay;
  const int64_t P = y.pbase[l + 1] - y.pbase[l];
  if (P <= 0) return SG_OK;
  ::sg::launch(k_xfer, clamp_grid(div_up(P * stride, 256), kSMs * 8), 256, 0, (cudaStream_t)stream, (const SgMeta*)(base + y.o_meta), l, (const int32_t*)(base + y.o_xfer) + y.pbase[l],
      sendbuf, recvbuf, stride, 1);
  SG_CHECK_LAUNCH("k_xfer(to_owner)");
  return SG_OK;
}

extern "C" int sg_xfer_from_owner(const void* split_ws, const SgSplitLayout* lay, int32_t l,
                                  const float* sendbuf_recv_layout, float* recvbuf_pair_layout,
                                  int32_t stride, void* stream) {
  SG_REQUIRE(split_ws && lay, "xfer: null workspace");
  const char* base = (const char*)split_ws;
  const SgSplitLayout& y = *lay;
  const int64_t P = y.pbase[l + 1] - y.pbase[l];
  if (P <= 0) return SG_OK;
  ::sg::launch(k_xfer, clamp_grid(div_up(P * stride, 256), kSMs * 8), 256, 0, (cudaStream_t)stream, (const SgMeta*)(base + y.o_meta), l, (const int32_t*)(base + y.o_xfer) + y.pbase[l],
      sendbuf_recv_layout, recvbuf_pair_layout, stride, 0);
  SG_CHECK_LAUNCH("k_xfer(from_owner)");
  return SG_OK;
}

extern "C" int sg_pack_from_owner(const void* split_ws, const SgSplitLayout* lay, int32_t l,
                                  int32_t d, const float* rows, int32_t w, float* out,
                                  int32_t stride, int64_t max_slots, void* stream) {
  SG_REQUIRE(split_ws && lay, "pack: null workspace");
  const char* base = (const char*)split_ws;
  const SgSplitLayout& y = *lay;
  if (max_slots <= 0) return SG_OK;
  ::sg::launch(k_pack_from_owner, clamp_grid(div_up(max_slots * w, 256), kSMs * 8), 256, 0,
                      (cudaStream_t)stream, (const SgMeta*)(base + y.o_meta), l, d,
                                              (const int32_t*)(base + y.o_recv_row) + y.pbase[l],
                                              rows, w, out, stride);
  SG_CHECK_LAUNCH("k_pack_from_owner");
  return SG_OK;
}

extern "C" int sg_unpack_refs(const void* split_ws, const SgSplitLayout* lay, int32_t l,
                              int32_t d, const float* recv_pair_layout, int32_t stride, int32_t w,
                              float* out, int64_t max_rows, void* stream) {
  SG_REQUIRE(split_ws && lay, "unpack: null workspace");
  const char* base = (const char*)split_ws;
  const SgSplitLayout& y = *lay;
  if (max_rows <= 0) return SG_OK;
  ::sg::launch(k_unpack_refs, clamp_grid(div_up(max_rows * w, 256), kSMs * 8), 256, 0,
                  (cudaStream_t)stream, (const SgMeta*)(base + y.o_meta), l, d,
                                          (const int32_t*)(base + y.o_sendpos) + y.pbase[l],
                                          recv_pair_layout, stride, w, out);
  SG_CHECK_LAUNCH("k_unpack_refs");
  return SG_OK;
}

}  // namespace sg
