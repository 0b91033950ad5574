// Host->device input pipeline for the captured training step
// (engine.CapturedStep.run_pipelined). The reference loads each iteration's
// inputs synchronously (engine.py:_load_inputs, :760-790); here a sample packed
// in pinned host memory crosses PCIe on a dedicated copy stream into one of two
// device staging slots while the previous step's graph runs, and the step's
// loss comes back through pinned memory read one step later.
//
//   copy stream : wait used[s] -> H2D host -> stage[s] -> record h2d[s]
//   main stream : wait h2d[s] -> D2D stage[s] -> graph inputs -> record used[s]
//                 -> graph replay -> D2H loss -> record done[s]
#include <algorithm>
#include <cstring>

#include "common.cuh"

namespace sg {
namespace {

struct Pipe {
  int64_t bytes = 0;  // staged input layout
  int64_t extra = 0;  // scratch after it (compact staging: the run starts)
  void* stage[2] = {nullptr, nullptr};
  float* loss_h = nullptr;  // pinned, 2 words
  cudaStream_t copy = nullptr;
  cudaEvent_t used[2] = {nullptr, nullptr}, h2d[2] = {nullptr, nullptr}, done[2] = {nullptr, nullptr};
};

void pipe_free(Pipe* p) {
  if (!p) return;
  for (int s = 0; s < 2; ++s) {
    if (p->stage[s]) cudaFree(p->stage[s]);
    if (p->used[s]) cudaEventDestroy(p->used[s]);
    if (p->h2d[s]) cudaEventDestroy(p->h2d[s]);
    if (p->done[s]) cudaEventDestroy(p->done[s]);
  }
  if (p->loss_h) cudaFreeHost(p->loss_h);
  if (p->copy) cudaStreamDestroy(p->copy);
  delete p;
}

}  // namespace

extern "C" void* sg_pipe_create2(int64_t bytes, int64_t extra) {
  if (bytes <= 0 || bytes % 16 || extra < 0) {
    set_error("pipe_create: bytes must be > 0 and a multiple of 16, extra >= 0");
    return nullptr;
  }
  Pipe* p = new Pipe();
  p->bytes = bytes;
  p->extra = extra;
  // highest priority: the compact form's expand kernel then takes the first
  // free SM slots between the running step's kernels instead of queueing
  // behind them (the next step's D2D waits on it)
  int lo_prio = 0, hi_prio = 0;
  cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
  bool ok = cudaStreamCreateWithPriority(&p->copy, cudaStreamNonBlocking, hi_prio) == cudaSuccess &&
            cudaHostAlloc((void**)&p->loss_h, 2 * sizeof(float), cudaHostAllocDefault) == cudaSuccess;
  for (int s = 0; ok && s < 2; ++s) {
    ok = cudaMalloc(&p->stage[s], (size_t)(bytes + extra)) == cudaSuccess &&
         cudaEventCreateWithFlags(&p->used[s], cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&p->h2d[s], cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&p->done[s], cudaEventDisableTiming) == cudaSuccess;
  }
  if (!ok) {
    set_error(std::string("pipe_create: ") + cudaGetErrorString(cudaGetLastError()));
    pipe_free(p);
    return nullptr;
  }
  return p;
}

extern "C" void* sg_pipe_create(int64_t bytes) { return sg_pipe_create2((bytes + 15) / 16 * 16, 0); }

extern "C" void sg_pipe_destroy(void* h) { pipe_free((Pipe*)h); }

// The pipe's copy stream (host-to-device copies; with direct staging also the
// next sample's split graph runs there).
extern "C" void* sg_pipe_copy_stream(void* h) { return h ? (void*)((Pipe*)h)->copy : nullptr; }

extern "C" int sg_pipe_stage(void* h, int32_t slot, const void* host_src, int64_t bytes, void* dev_dst,
                             void* stream) {
  Pipe* p = (Pipe*)h;
  SG_REQUIRE(p && (slot == 0 || slot == 1), "pipe_stage: bad handle/slot");
  SG_REQUIRE(bytes >= 0 && bytes <= p->bytes + p->extra, "pipe_stage: bytes exceed the staging slot");
  SG_REQUIRE(host_src && dev_dst, "pipe_stage: null buffer");
  cudaStream_t st = (cudaStream_t)stream;
  SG_CUDA(cudaStreamWaitEvent(p->copy, p->used[slot], 0));
  SG_CUDA(cudaMemcpyAsync(p->stage[slot], host_src, (size_t)bytes, cudaMemcpyHostToDevice, p->copy));
  SG_CUDA(cudaEventRecord(p->h2d[slot], p->copy));
  SG_CUDA(cudaStreamWaitEvent(st, p->h2d[slot], 0));
  SG_CUDA(cudaMemcpyAsync(dev_dst, p->stage[slot], (size_t)bytes, cudaMemcpyDeviceToDevice, st));
  SG_CUDA(cudaEventRecord(p->used[slot], st));
  return SG_OK;
}

namespace {
// Destination lists of a destination-grouped sample from per-destination run
// starts (the compact host->device form): layer l's starts follow layer l-1's
// (|V^l| words each, sizes from the staged header); one thread per destination
// writes its run of ed. Runs on the copy stream, in the shadow of the running step.
struct ExpandGeo {
  int64_t eoff[SG_MAXL];  // capacity offset of E^l in the es / ed regions (layer l at [l-1])
  int64_t o_ed;           // word offset of the ed region
  int64_t starts_off;     // word offset of the staged starts
  int L;
};

__global__ void __launch_bounds__(256) k_pipe_expand(int32_t* __restrict__ stage, const int32_t* __restrict__ starts,
                                                     ExpandGeo geo) {
  const int64_t* sizes = reinterpret_cast<const int64_t*>(stage);  // [nV (L+1) | nE (L)]
  int64_t off[SG_MAXL + 1];
  off[0] = 0;
  for (int l = 1; l <= geo.L; ++l) off[l] = off[l - 1] + sizes[l];
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < off[geo.L];
       x += (int64_t)gridDim.x * blockDim.x) {
    int l = 1;
    while (x >= off[l]) ++l;
    const int64_t i = x - off[l - 1];
    const int b = starts[x];
    const int e = i + 1 < sizes[l] ? starts[x + 1] : (int)sizes[geo.L + l];
    int32_t* ed = stage + geo.o_ed + geo.eoff[l - 1];
    for (int k = b; k < e; ++k) ed[k] = (int32_t)i;
  }
}
}  // namespace

// Compact staging: H2D of the sample prefix (header, V, es) and of the
// per-destination run starts, the ed lists rebuilt on the copy stream, then
// the usual D2D of the full prefix into the graph's input buffer.
extern "C" int sg_pipe_stage_compact(void* h, int32_t slot, const void* host_prefix, int64_t prefix_bytes,
                                     const void* host_starts, int64_t starts_bytes, int32_t L,
                                     const int64_t* edge_off, int64_t o_ed, int64_t full_bytes, void* dev_dst,
                                     void* stream) {
  Pipe* p = (Pipe*)h;
  SG_REQUIRE(p && (slot == 0 || slot == 1), "pipe_stage_compact: bad handle/slot");
  SG_REQUIRE(L >= 1 && L <= SG_MAXL && edge_off, "pipe_stage_compact: bad geometry");
  SG_REQUIRE(prefix_bytes >= 0 && full_bytes >= prefix_bytes && full_bytes <= p->bytes && starts_bytes >= 0 &&
                 starts_bytes <= p->extra,
             "pipe_stage_compact: bytes exceed the staging slot");
  SG_REQUIRE(host_prefix && host_starts && dev_dst, "pipe_stage_compact: null buffer");
  cudaStream_t st = (cudaStream_t)stream;
  char* stage = (char*)p->stage[slot];
  SG_CUDA(cudaStreamWaitEvent(p->copy, p->used[slot], 0));
  SG_CUDA(cudaMemcpyAsync(stage, host_prefix, (size_t)prefix_bytes, cudaMemcpyHostToDevice, p->copy));
  SG_CUDA(cudaMemcpyAsync(stage + p->bytes, host_starts, (size_t)starts_bytes, cudaMemcpyHostToDevice, p->copy));
  ExpandGeo geo;
  memset(&geo, 0, sizeof(geo));
  geo.L = L;
  for (int l = 0; l < L; ++l) geo.eoff[l] = edge_off[l];
  geo.o_ed = o_ed;
  geo.starts_off = p->bytes / 4;
  if (starts_bytes > 0) {
    k_pipe_expand<<<clamp_grid(div_up(starts_bytes / 4, 256), kSMs), 256, 0, p->copy>>>(
        (int32_t*)stage, (const int32_t*)stage + geo.starts_off, geo);
    SG_CHECK_LAUNCH("k_pipe_expand");
  }
  SG_CUDA(cudaEventRecord(p->h2d[slot], p->copy));
  SG_CUDA(cudaStreamWaitEvent(st, p->h2d[slot], 0));
  SG_CUDA(cudaMemcpyAsync(dev_dst, stage, (size_t)full_bytes, cudaMemcpyDeviceToDevice, st));
  SG_CUDA(cudaEventRecord(p->used[slot], st));
  return SG_OK;
}

// Direct staging (one captured graph per slot, each reading its own input
// buffer): the H2D lands straight in the graph's input buffer `dev_dst` on the
// copy stream -- no device-to-device copy on the step's critical path. The
// copy into slot s waits for the graph that last read slot s (sg_pipe_release).
// host_starts / starts_bytes: the compact form (run starts into the slot's
// scratch, ed rebuilt into dev_dst by k_pipe_expand); starts_bytes == 0: the
// full layout in host_prefix.
extern "C" int sg_pipe_stage_direct(void* h, int32_t slot, const void* host_prefix, int64_t prefix_bytes,
                                    const void* host_starts, int64_t starts_bytes, int32_t L,
                                    const int64_t* edge_off, int64_t o_ed, void* dev_dst, void* stream) {
  Pipe* p = (Pipe*)h;
  SG_REQUIRE(p && (slot == 0 || slot == 1), "pipe_stage_direct: bad handle/slot");
  SG_REQUIRE(prefix_bytes >= 0 && prefix_bytes <= p->bytes && starts_bytes >= 0 && starts_bytes <= p->extra,
             "pipe_stage_direct: bytes exceed the staging slot");
  SG_REQUIRE(host_prefix && dev_dst && (starts_bytes == 0 || (host_starts && edge_off && L >= 1 && L <= SG_MAXL)),
             "pipe_stage_direct: null buffer / bad geometry");
  cudaStream_t st = (cudaStream_t)stream;
  SG_CUDA(cudaStreamWaitEvent(p->copy, p->used[slot], 0));
  SG_CUDA(cudaMemcpyAsync(dev_dst, host_prefix, (size_t)prefix_bytes, cudaMemcpyHostToDevice, p->copy));
  if (starts_bytes > 0) {
    char* scratch = (char*)p->stage[slot] + p->bytes;
    SG_CUDA(cudaMemcpyAsync(scratch, host_starts, (size_t)starts_bytes, cudaMemcpyHostToDevice, p->copy));
    ExpandGeo geo;
    memset(&geo, 0, sizeof(geo));
    geo.L = L;
    for (int l = 0; l < L; ++l) geo.eoff[l] = edge_off[l];
    geo.o_ed = o_ed;
    k_pipe_expand<<<clamp_grid(div_up(starts_bytes / 4, 256), kSMs), 256, 0, p->copy>>>(
        (int32_t*)dev_dst, (const int32_t*)scratch, geo);
    SG_CHECK_LAUNCH("k_pipe_expand");
  }
  SG_CUDA(cudaEventRecord(p->h2d[slot], p->copy));
  SG_CUDA(cudaStreamWaitEvent(st, p->h2d[slot], 0));
  return SG_OK;
}

// After the graph that reads slot `slot` is queued on `stream`: the slot's next
// H2D may begin once that graph has run.
extern "C" int sg_pipe_release(void* h, int32_t slot, void* stream) {
  Pipe* p = (Pipe*)h;
  SG_REQUIRE(p && (slot == 0 || slot == 1), "pipe_release: bad handle/slot");
  SG_CUDA(cudaEventRecord(p->used[slot], (cudaStream_t)stream));
  return SG_OK;
}

extern "C" int sg_pipe_finish(void* h, int32_t slot, const float* dev_loss, void* stream) {
  Pipe* p = (Pipe*)h;
  SG_REQUIRE(p && (slot == 0 || slot == 1) && dev_loss, "pipe_finish: bad handle/slot/pointer");
  cudaStream_t st = (cudaStream_t)stream;
  SG_CUDA(cudaMemcpyAsync(p->loss_h + slot, dev_loss, sizeof(float), cudaMemcpyDeviceToHost, st));
  SG_CUDA(cudaEventRecord(p->done[slot], st));
  return SG_OK;
}

extern "C" int sg_pipe_wait(void* h, int32_t slot, float* loss_out) {
  Pipe* p = (Pipe*)h;
  SG_REQUIRE(p && (slot == 0 || slot == 1) && loss_out, "pipe_wait: bad handle/slot/pointer");
  SG_CUDA(cudaEventSynchronize(p->done[slot]));
  *loss_out = p->loss_h[slot];
  return SG_OK;
}

// One async copy in any direction (UVA: pinned host <-> device, device <->
// device) on `stream`: the executor's parameter upload, sample load and
// gradient read-back, without a framework dispatch per copy.
extern "C" int sg_copy_async(void* dst, const void* src, int64_t bytes, void* stream) {
  SG_REQUIRE(bytes >= 0 && (bytes == 0 || (dst && src)), "copy_async: bad argument");
  if (bytes > 0) SG_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, (cudaStream_t)stream));
  return SG_OK;
}

// split_minibatch's direct path (a native-sampler sample in one pinned
// buffer, no host pack): after one H2D of [header | V | es | ed], its 3L+2
// segments are moved to their word offsets in the capacity layout (one kernel,
// blockIdx.y = segment). The segments are derived on the device from the int64
// sizes header the sample carries (stage[0 .. S)), so the host passes only the
// capacity geometry (cached per geometry): geo = [L, S, o_V, o_es, o_ed,
// voff[0..L+1], eoff[0..L]] (int64, host memory, read at launch). Lengths are
// clamped to the capacities.
namespace {
struct RelGeo {
  int32_t L;
  int64_t S, o_V, o_es, o_ed, voff[SG_MAXL + 2], eoff[SG_MAXL + 1];
};
__global__ void k_relayout_hdr(const int32_t* __restrict__ src, int32_t* __restrict__ dst, RelGeo g) {
  const int seg = blockIdx.y, L = g.L;
  const int64_t* sz = reinterpret_cast<const int64_t*>(src);  // [nV_0..nV_L, nE_1..nE_L]
  int64_t VS = 0, ES = 0;
  for (int l = 0; l <= L; ++l) VS += sz[l];
  for (int l = 0; l < L; ++l) ES += sz[L + 1 + l];
  int64_t so, dof, len;
  if (seg == 0) {
    so = 0; dof = 0; len = g.S;
  } else if (seg <= L + 1) {  // V^l
    const int l = seg - 1;
    so = g.S;
    for (int k = 0; k < l; ++k) so += sz[k];
    dof = g.o_V + g.voff[l];
    len = min(sz[l], g.voff[l + 1] - g.voff[l]);
  } else {  // E^l sources (seg < 2L+2), then destinations
    const bool d = seg >= 2 * L + 2;
    const int l = seg - (d ? 2 * L + 2 : L + 2);
    so = g.S + VS + (d ? ES : 0);
    for (int k = 0; k < l; ++k) so += sz[L + 1 + k];
    dof = (d ? g.o_ed : g.o_es) + g.eoff[l];
    len = min(sz[L + 1 + l], g.eoff[l + 1] - g.eoff[l]);
  }
  const int32_t* a = src + so;
  int32_t* b = dst + dof;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}
}  // namespace

// Compact form: src = [header | V | es | per-destination run starts of layers
// 1..L (|V^l| each)]; the destination lists are rebuilt from the starts into
// the capacity layout (blocks y >= 2L+2: one thread per destination writes its
// run), the other segments copied as in k_relayout_hdr.
__global__ void k_relayout_compact(const int32_t* __restrict__ src, int32_t* __restrict__ dst, RelGeo g) {
  const int seg = blockIdx.y, L = g.L;
  const int64_t* sz = reinterpret_cast<const int64_t*>(src);
  int64_t VS = 0, ES = 0;
  for (int l = 0; l <= L; ++l) VS += sz[l];
  for (int l = 0; l < L; ++l) ES += sz[L + 1 + l];
  if (seg < 2 * L + 2) {
    int64_t so, dof, len;
    if (seg == 0) {
      so = 0; dof = 0; len = g.S;
    } else if (seg <= L + 1) {
      const int l = seg - 1;
      so = g.S;
      for (int k = 0; k < l; ++k) so += sz[k];
      dof = g.o_V + g.voff[l];
      len = min(sz[l], g.voff[l + 1] - g.voff[l]);
    } else {
      const int l = seg - (L + 2);
      so = g.S + VS;
      for (int k = 0; k < l; ++k) so += sz[L + 1 + k];
      dof = g.o_es + g.eoff[l];
      len = min(sz[L + 1 + l], g.eoff[l + 1] - g.eoff[l]);
    }
    const int32_t* a = src + so;
    int32_t* b = dst + dof;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x)
      b[i] = a[i];
    return;
  }
  const int l = seg - (2 * L + 2);  // E^(l+1): destinations are V^(l+1) positions
  int64_t so = g.S + VS + ES;
  for (int k = 0; k < l; ++k) so += sz[k + 1];
  const int64_t nd = sz[l + 1], ne = min(sz[L + 1 + l], g.eoff[l + 1] - g.eoff[l]);
  const int32_t* st = src + so;
  int32_t* ed = dst + g.o_ed + g.eoff[l];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nd; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = st[i], e = i + 1 < nd ? (int64_t)st[i + 1] : ne;
    for (int64_t k = max(b, (int64_t)0); k < min(e, ne); ++k) ed[k] = (int32_t)i;
  }
}

extern "C" int sg_relayout_sample_compact(const int32_t* src, int32_t* dst, const int64_t* geo, int64_t max_len,
                                          void* stream) {
  SG_REQUIRE(src && dst && geo && geo[0] >= 1 && geo[0] <= SG_MAXL && geo[1] == 2 * (2 * geo[0] + 1),
             "relayout_sample_compact: bad argument");
  RelGeo g;
  memset(&g, 0, sizeof(g));
  g.L = (int32_t)geo[0];
  g.S = geo[1]; g.o_V = geo[2]; g.o_es = geo[3]; g.o_ed = geo[4];
  for (int l = 0; l <= g.L + 1; ++l) g.voff[l] = geo[5 + l];
  for (int l = 0; l <= g.L; ++l) g.eoff[l] = geo[5 + g.L + 2 + l];
  dim3 grid(clamp_grid(div_up(std::max<int64_t>(max_len, 1), 4 * 256), kSMs), 3 * g.L + 2);
  k_relayout_compact<<<grid, 256, 0, (cudaStream_t)stream>>>(src, dst, g);
  SG_CHECK_LAUNCH("k_relayout_compact");
  return SG_OK;
}

extern "C" int sg_relayout_sample_hdr(const int32_t* src, int32_t* dst, const int64_t* geo, int64_t max_len,
                                      void* stream) {
  SG_REQUIRE(src && dst && geo && geo[0] >= 1 && geo[0] <= SG_MAXL && geo[1] == 2 * (2 * geo[0] + 1),
             "relayout_sample_hdr: bad argument");
  RelGeo g;
  memset(&g, 0, sizeof(g));
  g.L = (int32_t)geo[0];
  g.S = geo[1]; g.o_V = geo[2]; g.o_es = geo[3]; g.o_ed = geo[4];
  for (int l = 0; l <= g.L + 1; ++l) g.voff[l] = geo[5 + l];
  for (int l = 0; l <= g.L; ++l) g.eoff[l] = geo[5 + g.L + 2 + l];
  dim3 grid(clamp_grid(div_up(std::max<int64_t>(max_len, 1), 4 * 256), kSMs), 3 * g.L + 2);
  k_relayout_hdr<<<grid, 256, 0, (cudaStream_t)stream>>>(src, dst, g);
  SG_CHECK_LAUNCH("k_relayout_hdr");
  return SG_OK;
}


}  // namespace sg
