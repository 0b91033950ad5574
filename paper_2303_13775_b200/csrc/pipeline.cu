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
#include <cstring>

#include "common.cuh"

namespace sg {
namespace {

struct Pipe {
  int64_t bytes = 0;
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

extern "C" void* sg_pipe_create(int64_t bytes) {
  if (bytes <= 0) {
    set_error("pipe_create: bytes must be > 0");
    return nullptr;
  }
  Pipe* p = new Pipe();
  p->bytes = bytes;
  bool ok = cudaStreamCreateWithFlags(&p->copy, cudaStreamNonBlocking) == cudaSuccess &&
            cudaHostAlloc((void**)&p->loss_h, 2 * sizeof(float), cudaHostAllocDefault) == cudaSuccess;
  for (int s = 0; ok && s < 2; ++s) {
    ok = cudaMalloc(&p->stage[s], (size_t)bytes) == cudaSuccess &&
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

extern "C" void sg_pipe_destroy(void* h) { pipe_free((Pipe*)h); }

extern "C" int sg_pipe_stage(void* h, int32_t slot, const void* host_src, int64_t bytes, void* dev_dst,
                             void* stream) {
  Pipe* p = (Pipe*)h;
  SG_REQUIRE(p && (slot == 0 || slot == 1), "pipe_stage: bad handle/slot");
  SG_REQUIRE(bytes >= 0 && bytes <= p->bytes, "pipe_stage: bytes exceed the staging slot");
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

}  // namespace sg
