// Peer-memory transport for the push-to-owner / push-from-owner rounds
// (engine.py:121-156) when every device is its own process (one rank per GPU).
//
// Every rank runs the splitter on the replicated sample, so every rank knows
// the GLOBAL slot numbering of a layer: pair slots (holder-major) and receive
// slots (owner-major), xfer[pair slot] = receive slot. Each rank's exchange
// buffers are mapped into its peers' address spaces (CUDA IPC over
// NVLink/NVSwitch), so no sizes ever travel to the host and the multi-GPU
// step is one CUDA graph:
//
//   to_owner   (holder r)  k_peer_push: for r's pair slots p, write the row
//              into owner o's receive buffer at xfer[p] (o = bucket of xfer[p]
//              in recv_off) -- stores over NVLink, coalesced 16 B.
//   from_owner (holder r)  k_peer_pull: for r's pair slots p, read the row the
//              owner packed at receive slot xfer[p] from the owner's buffer.
//   signal     after the producing kernel (stream order: its writes are
//              complete), k_peer_signal stores this step's epoch into slot
//              [round][r] of every peer's flag array (st.release.sys).
//   wait       k_peer_wait spins (ld.acquire.sys) until every peer's slot of
//              this round holds the current epoch; the next kernel in the
//              stream (griddepcontrol.wait) sees the peers' data.
// The epoch is a device counter bumped once per step (k_peer_epoch), so flags
// are monotonic and never reset. A round's buffers are not reused within a
// step; across steps the gradient all-reduce is the barrier that orders a
// rank's next writes after its peers' reads.
#include <cstring>
#include <type_traits>

#include "common.cuh"

namespace sg {
namespace {

constexpr int kRounds = 32;
constexpr uint64_t kPeerTimeoutNs = 20ull * 1000 * 1000 * 1000;  // 20 s without a peer signal  // exchange rounds per step (SAGE 5, GAT 15 at L = 3)

struct PeerTable {
  int64_t p[SG_MAXG];
};

__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(int* p, int v) {
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <bool PUSH, int VEC>
__global__ void __launch_bounds__(256) k_peer_move(const SgMeta* __restrict__ meta, int l, int rank, int g,
                                                   const int32_t* __restrict__ xfer, PeerTable peer,
                                                   float* __restrict__ local, int stride) {
  SG_PDL_ENTRY();
  using T = typename std::conditional<VEC == 4, float4, float>::type;
  const int p0 = meta->ref_off[l][rank], p1 = meta->ref_off[l][rank + 1];
  const int sv = stride / VEC;  // VEC == 4: 16-byte rows
  const int64_t total = (int64_t)(p1 - p0) * sv;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i / sv), c = (int)(i - (int64_t)k * sv);
    const int p = p0 + k;
    const int rs = xfer[p];
    const int o = find_bucket(meta->recv_off[l], g, rs);
    T* remote = reinterpret_cast<T*>((float*)peer.p[o] + (int64_t)rs * stride) + c;
    T* mine = reinterpret_cast<T*>(local + (int64_t)p * stride) + c;
    if (PUSH) *remote = *mine;
    else *mine = *remote;
  }
}

__global__ void k_peer_signal(PeerTable flags, int rank, int g, int round, const int* __restrict__ epoch) {
  SG_PDL_ENTRY();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int e = *epoch;
  __threadfence_system();
  for (int o = 0; o < g; ++o)
    if (o != rank) st_release_sys((int*)flags.p[o] + round * SG_MAXG + rank, e);
}

__global__ void k_peer_wait(const int* __restrict__ my_flags, int rank, int g, int round,
                            const int* __restrict__ epoch, int* __restrict__ timeout) {
  SG_PDL_ENTRY();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int e = *epoch;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int s = 0; s < g; ++s) {
    if (s == rank) continue;
    while (ld_acquire_sys(my_flags + round * SG_MAXG + s) < e) {
      __nanosleep(256);
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > kPeerTimeoutNs) {
        // a peer is gone or wedged: record it and abort the context -- the
        // step must never continue on stale peer buffers
        atomicOr(timeout, 1);
        __threadfence_system();
        __trap();
      }
    }
  }
}

__global__ void k_peer_epoch(int* epoch) {
  SG_PDL_ENTRY();
  if (threadIdx.x == 0 && blockIdx.x == 0) *epoch += 1;
}

}  // namespace
}  // namespace sg

using namespace sg;

static PeerTable table_of(const int64_t* ptrs, int g) {
  PeerTable t;
  memset(&t, 0, sizeof(t));
  for (int i = 0; i < g; ++i) t.p[i] = ptrs[i];
  return t;
}

extern "C" int sg_peer_rounds(void) { return kRounds; }

extern "C" int sg_peer_exchange(const void* split_ws, const SgSplitLayout* lay, int32_t l, int32_t rank,
                                int32_t push, float* local, int32_t stride, const int64_t* peer_bufs,
                                void* stream) {
  SG_REQUIRE(split_ws && lay && local && peer_bufs, "peer_exchange: null argument");
  const SgSplitLayout& y = *lay;
  SG_REQUIRE(rank >= 0 && rank < y.g && l >= 1 && l <= y.L, "peer_exchange: bad rank/layer");
  SG_REQUIRE(stride >= 1, "peer_exchange: stride >= 1");
  const char* base = (const char*)split_ws;
  const int64_t P = y.pbase[l + 1] - y.pbase[l];
  if (P <= 0) return SG_OK;
  const PeerTable t = table_of(peer_bufs, y.g);
  const bool v4 = stride % 4 == 0;
  const int grid = clamp_grid(div_up(P * (v4 ? stride / 4 : stride), 256), kSMs * 4);
  const SgMeta* meta = (const SgMeta*)(base + y.o_meta);
  const int32_t* xfer = (const int32_t*)(base + y.o_xfer) + y.pbase[l];
  cudaStream_t st = (cudaStream_t)stream;
  if (push && v4) ::sg::launch(k_peer_move<true, 4>, grid, 256, 0, st, meta, l, rank, y.g, xfer, t, local, stride);
  else if (push) ::sg::launch(k_peer_move<true, 1>, grid, 256, 0, st, meta, l, rank, y.g, xfer, t, local, stride);
  else if (v4) ::sg::launch(k_peer_move<false, 4>, grid, 256, 0, st, meta, l, rank, y.g, xfer, t, local, stride);
  else ::sg::launch(k_peer_move<false, 1>, grid, 256, 0, st, meta, l, rank, y.g, xfer, t, local, stride);
  SG_CHECK_LAUNCH("k_peer_move");
  return SG_OK;
}

extern "C" int sg_peer_signal(const int64_t* peer_flags, int32_t rank, int32_t g, int32_t round,
                              const int32_t* epoch, void* stream) {
  SG_REQUIRE(peer_flags && epoch && round >= 0 && round < kRounds && g >= 1 && g <= SG_MAXG,
             "peer_signal: bad argument");
  ::sg::launch(k_peer_signal, 1, 32, 0, (cudaStream_t)stream, table_of(peer_flags, g), rank, g, round, epoch);
  SG_CHECK_LAUNCH("k_peer_signal");
  return SG_OK;
}

extern "C" int sg_peer_wait(const int32_t* my_flags, int32_t rank, int32_t g, int32_t round,
                            const int32_t* epoch, int32_t* timeout, void* stream) {
  SG_REQUIRE(my_flags && epoch && timeout && round >= 0 && round < kRounds, "peer_wait: bad argument");
  ::sg::launch(k_peer_wait, 1, 32, 0, (cudaStream_t)stream, my_flags, rank, g, round, epoch, timeout);
  SG_CHECK_LAUNCH("k_peer_wait");
  return SG_OK;
}

extern "C" int sg_peer_epoch(int32_t* epoch, void* stream) {
  SG_REQUIRE(epoch, "peer_epoch: null");
  ::sg::launch(k_peer_epoch, 1, 32, 0, (cudaStream_t)stream, epoch);
  SG_CHECK_LAUNCH("k_peer_epoch");
  return SG_OK;
}

// ---- gradient all-reduce + SGD over peer memory (allreduce_and_step,
// engine.py:633-647). Each rank stages its flat gradient (+ loss slot) into
// one of two shared slots chosen by epoch parity, signals, waits, then every
// rank sums ALL ranks' slots in rank order (identical, deterministic result
// on every rank) and applies the SGD step. The parity double buffer plus the
// wait make this round the step barrier that orders the next step's writes
// into peer buffers after every peer's reads of this step.
namespace sg {
namespace {

__global__ void k_peer_grad_stage(const float* __restrict__ g, float* __restrict__ slots, int64_t n1,
                                  int64_t slot_stride, const int* __restrict__ epoch) {
  SG_PDL_ENTRY();
  float* dst = slots + (int64_t)(*epoch & 1) * slot_stride;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n1; k += (int64_t)gridDim.x * blockDim.x)
    dst[k] = g[k];
}

__global__ void k_peer_allreduce_sgd(PeerTable slots, int g, int64_t n, int64_t n1, int64_t slot_stride,
                                     const int* __restrict__ epoch, float* __restrict__ params,
                                     float* __restrict__ gout, float scale, double lr,
                                     const int64_t* __restrict__ nt) {
  SG_PDL_ENTRY();
  if (nt) scale = (float)(lr / (double)max(*nt, (int64_t)1));  // the sample's own target count
  const int64_t off = (int64_t)(*epoch & 1) * slot_stride;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n1; k += (int64_t)gridDim.x * blockDim.x) {
    float s = ((const float*)slots.p[0])[off + k];
    for (int r = 1; r < g; ++r) s += ((const float*)slots.p[r])[off + k];
    if (gout) gout[k] = s;
    if (k < n) params[k] -= scale * s;
  }
}

}  // namespace
}  // namespace sg

extern "C" int sg_peer_grad_stage(const float* grads, float* my_slots, int64_t n1, int64_t slot_stride,
                                  const int32_t* epoch, void* stream) {
  SG_REQUIRE(grads && my_slots && epoch && n1 > 0 && slot_stride >= n1, "peer_grad_stage: bad argument");
  ::sg::launch(k_peer_grad_stage, clamp_grid(div_up(n1, 256), kSMs), 256, 0, (cudaStream_t)stream, grads, my_slots,
               n1, slot_stride, epoch);
  SG_CHECK_LAUNCH("k_peer_grad_stage");
  return SG_OK;
}

extern "C" int sg_peer_allreduce_sgd(const int64_t* peer_slots, int32_t g, int64_t n, int64_t n1,
                                     int64_t slot_stride, const int32_t* epoch, float* params, float* grads_out,
                                     float scale, void* stream) {
  SG_REQUIRE(peer_slots && epoch && params && g >= 1 && g <= SG_MAXG && n1 >= n, "peer_allreduce_sgd: bad argument");
  ::sg::launch(k_peer_allreduce_sgd, clamp_grid(div_up(n1, 256), kSMs), 256, 0, (cudaStream_t)stream,
               table_of(peer_slots, g), (int)g, n, n1, slot_stride, epoch, params, grads_out, scale, 0.0,
               (const int64_t*)nullptr);
  SG_CHECK_LAUNCH("k_peer_allreduce_sgd");
  return SG_OK;
}

extern "C" int sg_peer_allreduce_sgd_nt(const int64_t* peer_slots, int32_t g, int64_t n, int64_t n1,
                                        int64_t slot_stride, const int32_t* epoch, float* params,
                                        float* grads_out, double lr, const int64_t* num_targets, void* stream) {
  SG_REQUIRE(peer_slots && epoch && params && num_targets && g >= 1 && g <= SG_MAXG && n1 >= n,
             "peer_allreduce_sgd_nt: bad argument");
  ::sg::launch(k_peer_allreduce_sgd, clamp_grid(div_up(n1, 256), kSMs), 256, 0, (cudaStream_t)stream,
               table_of(peer_slots, g), (int)g, n, n1, slot_stride, epoch, params, grads_out, 0.f, lr, num_targets);
  SG_CHECK_LAUNCH("k_peer_allreduce_sgd");
  return SG_OK;
}
