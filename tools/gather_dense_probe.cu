// Diagnostic (not product code): the HBM ceiling of gathering each UNIQUE
// layer-0 row once (the transform-before-aggregate dense pass), two ways:
//   k_reg<U, L>  : one warp per row group, U rows in flight per warp, L lanes x 16 B per row
//   k_bulk<T, S> : cp.async.bulk of each row into a T-row x S-stage smem ring,
//                  one producer thread per CTA, consumers sum the staged rows
// Built by tools/gather_dense_probe.py (nvcc -> .so, ctypes).
#include <cuda_runtime.h>
#include <stdint.h>

template <int U, int L>
__global__ void __launch_bounds__(256) k_reg(const float4* __restrict__ tab, const int* __restrict__ idx, int n,
                                            int S4, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int base = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * U; base < n; base += nw * U) {
    float4 t[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int i = base + k;
      const int r = i < n ? __ldg(idx + i) : 0;
      t[k] = (i < n && lane < L) ? __ldg(tab + (size_t)r * S4 + lane) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      float s = t[k].x + t[k].y + t[k].z + t[k].w;
#pragma unroll
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0 && base + k < n) out[base + k] = s;
    }
  }
}

__device__ __forceinline__ void mbar_init(uint32_t a, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint32_t a, int bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t par) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(a), "r"(par)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, int bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}

// T rows per stage, S stages, RB bytes per row (<= 512, multiple of 16); 4 warps: warp 0 lanes issue copies
template <int T, int S>
__global__ void __launch_bounds__(128) k_bulk(const float* __restrict__ tab, const int* __restrict__ idx, int n,
                                             int stride, int RB, float* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t full[S], empty[S];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init((uint32_t)__cvta_generic_to_shared(&full[s]), 1);
      mbar_init((uint32_t)__cvta_generic_to_shared(&empty[s]), 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int ntiles = (n + T - 1) / T;
  const uint32_t smb = (uint32_t)__cvta_generic_to_shared(sm);
  // producer: warp 0 (all lanes issue copies of their rows), runs ahead up to S tiles
  // consumer: all 4 warps
  int it = 0;
  int prod_it = 0;
  int prod_tile = blockIdx.x;
  auto produce = [&](int tile, int pit) {
    const int s = pit % S;
    const uint32_t fb = (uint32_t)__cvta_generic_to_shared(&full[s]);
    if (pit >= S) mbar_wait((uint32_t)__cvta_generic_to_shared(&empty[s]), ((pit / S) - 1) & 1);
    const int r0 = tile * T;
    const int nr = min(T, n - r0);
    if (lane == 0) mbar_expect(fb, nr * RB);
    __syncwarp();
    for (int k = lane; k < nr; k += 32) {
      const int r = __ldg(idx + r0 + k);
      bulk_g2s(smb + (uint32_t)((s * T + k) * 512), tab + (size_t)r * stride, RB, fb);
    }
  };
  if (w == 0) {
    for (int k = 0; k < S && prod_tile < ntiles; ++k) {
      produce(prod_tile, prod_it);
      prod_tile += gridDim.x;
      ++prod_it;
    }
  }
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int s = it % S;
    mbar_wait((uint32_t)__cvta_generic_to_shared(&full[s]), (it / S) & 1);
    const int r0 = tile * T;
    const int nr = min(T, n - r0);
    for (int k = w; k < nr; k += 4) {
      const float* row = (const float*)(sm + (s * T + k) * 512);
      float v = 0.f;
      for (int c = lane; c < RB / 4; c += 32) v += row[c];
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) out[r0 + k] = v;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive((uint32_t)__cvta_generic_to_shared(&empty[s]));
    if (w == 0 && prod_tile < ntiles) {
      produce(prod_tile, prod_it);
      prod_tile += gridDim.x;
      ++prod_it;
    }
  }
}

extern "C" int probe_reg(int variant, const float* tab, const int* idx, int n, int S4, float* out, int blocks) {
  switch (variant) {
    case 0: k_reg<4, 25><<<blocks, 256>>>((const float4*)tab, idx, n, S4, out); break;
    case 1: k_reg<8, 25><<<blocks, 256>>>((const float4*)tab, idx, n, S4, out); break;
    case 2: k_reg<4, 32><<<blocks, 256>>>((const float4*)tab, idx, n, S4, out); break;
    case 3: k_reg<8, 32><<<blocks, 256>>>((const float4*)tab, idx, n, S4, out); break;
    case 4: k_reg<16, 25><<<blocks, 256>>>((const float4*)tab, idx, n, S4, out); break;
    case 5: k_reg<2, 25><<<blocks, 256>>>((const float4*)tab, idx, n, S4, out); break;
  }
  return (int)cudaGetLastError();
}

extern "C" int probe_bulk(int variant, const float* tab, const int* idx, int n, int stride, int RB, float* out,
                          int blocks) {
  switch (variant) {
    case 0: {
      const int smem = 32 * 4 * 512;
      cudaFuncSetAttribute(k_bulk<32, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      k_bulk<32, 4><<<blocks, 128, smem>>>(tab, idx, n, stride, RB, out);
      break;
    }
    case 1: {
      const int smem = 32 * 8 * 512;
      cudaFuncSetAttribute(k_bulk<32, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      k_bulk<32, 8><<<blocks, 128, smem>>>(tab, idx, n, stride, RB, out);
      break;
    }
    case 2: {
      const int smem = 64 * 3 * 512;
      cudaFuncSetAttribute(k_bulk<64, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      k_bulk<64, 3><<<blocks, 128, smem>>>(tab, idx, n, stride, RB, out);
      break;
    }
    case 3: {
      const int smem = 16 * 6 * 512;
      cudaFuncSetAttribute(k_bulk<16, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      k_bulk<16, 6><<<blocks, 128, smem>>>(tab, idx, n, stride, RB, out);
      break;
    }
  }
  return (int)cudaGetLastError();
}

// Projection-shaped gathers at the projection's occupancy: tile = 128 rows x 25
// chunks, 256 threads, NLD = 13 float4 per thread, all in flight. pattern 0: a
// warp instruction covers 8 rows x 4 chunks (the plane-friendly mapping);
// pattern 1: a warp instruction covers one row's 25 chunks (row-contiguous).
template <int PAT>
__global__ void __launch_bounds__(256, 1) k_tile(const float4* __restrict__ tab, const int* __restrict__ idx, int n,
                                                int S4, float* __restrict__ out) {
  const int tid = threadIdx.x;
  const int ntiles = (n + 127) / 128;
  float acc = 0.f;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    float4 R[13];
#pragma unroll
    for (int j = 0; j < 13; ++j) {
      int m, c;
      if (PAT == 0) {
        const int i = tid + 256 * j, rest = i >> 3;
        c = rest % 26;
        m = (rest / 26) * 8 + (i & 7);
      } else {
        const int warp = tid >> 5, lane = tid & 31;
        m = warp * 16 + j + (j >= 13 ? 0 : 0);  // rows warp*16 .. +12 (13 of 16 rows, enough for the probe)
        c = lane;
      }
      const int r = t * 128 + m;
      R[j] = (m < 128 && c < 25 && r < n) ? __ldg(tab + (size_t)idx[r] * S4 + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int j = 0; j < 13; ++j) acc += R[j].x + R[j].y + R[j].z + R[j].w;
  }
  out[blockIdx.x * 256 + tid] = acc;
}

extern "C" int probe_tile(int pat, const float* tab, const int* idx, int n, int S4, float* out, int blocks) {
  if (pat == 0) k_tile<0><<<blocks, 256>>>((const float4*)tab, idx, n, S4, out);
  else k_tile<1><<<blocks, 256>>>((const float4*)tab, idx, n, S4, out);
  return (int)cudaGetLastError();
}
