// Shared definitions for the splitgnn-b200 CUDA library (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <string>
#include <utility>

#include "../../include/splitgnn_b200.h"

namespace sg {

extern std::atomic<unsigned long long> g_launches;
void set_error(const std::string& msg);

#define SG_LAUNCHED() (::sg::g_launches.fetch_add(1, std::memory_order_relaxed))

#define SG_CHECK_LAUNCH(name)                                                  \
  do {                                                                         \
    cudaError_t e__ = cudaGetLastError();                                      \
    if (e__ != cudaSuccess) {                                                  \
      ::sg::set_error(std::string(name) + ": " + cudaGetErrorString(e__));     \
      return SG_ERR_CUDA;                                                      \
    }                                                                          \
    SG_LAUNCHED();                                                             \
  } while (0)

#define SG_CUDA(call)                                                          \
  do {                                                                         \
    cudaError_t e__ = (call);                                                  \
    if (e__ != cudaSuccess) {                                                  \
      ::sg::set_error(std::string(#call) + ": " + cudaGetErrorString(e__));    \
      return SG_ERR_CUDA;                                                      \
    }                                                                          \
  } while (0)

#define SG_REQUIRE(cond, msg)                                                  \
  do {                                                                         \
    if (!(cond)) {                                                             \
      ::sg::set_error(msg);                                                    \
      return SG_ERR_ARG;                                                       \
    }                                                                          \
  } while (0)

constexpr int kSMs = 148;

// ---- programmatic dependent launch (PDL)
// Every library kernel is launched with programmatic stream serialisation
// allowed and starts with SG_PDL_ENTRY(): griddepcontrol.wait blocks until the
// preceding grid in the stream has completed and its writes are visible (so
// no kernel ever reads a predecessor's output early), then
// launch_dependents lets the NEXT grid be scheduled while this one runs. In a
// captured CUDA graph this turns each kernel->kernel edge into a programmatic
// edge: the successor's launch latency and block scheduling overlap the
// predecessor instead of following it. griddepcontrol.wait is a no-op for a
// grid launched without the attribute. SG_PDL=0 disables the attribute.
#define SG_PDL_ENTRY()                                        \
  do {                                                        \
    asm volatile("griddepcontrol.wait;" ::: "memory");        \
    asm volatile("griddepcontrol.launch_dependents;" :::);    \
  } while (0)

// Wait for the completion of the mbarrier phase with parity `parity`; traps
// after 2 s (%globaltimer) instead of hanging the device on a lost arrival.
__device__ __forceinline__ void sg_mbar_wait(uint32_t mbar_smem, uint32_t parity) {
  uint32_t done = 0;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (true) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(mbar_smem), "r"(parity)
        : "memory");
    if (done) return;
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 2000000000ull) __trap();
  }
}

extern bool g_pdl;

template <typename... KArgs, typename... Args>
inline void launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                   Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Raise a kernel's dynamic shared-memory limit to the sm_100 maximum once per
// process (never inside a later CUDA-graph capture).
template <auto K>
inline cudaError_t allow_max_smem() {
  static bool done = false;
  if (done) return cudaSuccess;
  done = true;
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, K);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)(227 * 1024 - fa.sharedSizeBytes));
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ReLU with NumPy semantics: np.maximum(x, 0) propagates NaN (fmaxf would
// return 0 and hide it from DEBUG_CHECK_FINITE, engine.py:49-55).
__device__ __forceinline__ float sg_relu(float x) { return x < 0.f ? 0.f : x; }

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

inline int div_up(long long a, long long b) { return (int)((a + b - 1) / b); }

inline int clamp_grid(long long want, int cap) {
  if (want < 1) return 1;
  return want > cap ? cap : (int)want;
}

// Device-side: find d in [0, g) with off[d] <= x < off[d+1] (off non-decreasing).
__device__ __forceinline__ int find_bucket(const int32_t* off, int g, int x) {
  int lo = 0, hi = g - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (off[mid] <= x) lo = mid; else hi = mid - 1;
  }
  return lo;
}

}  // namespace sg
