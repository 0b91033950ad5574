// Diagnostic (not product code): one tcgen05.mma.kind::tf32 (M = 128, N = 64,
// K = 8 * KS) from shared memory in K-major or MN-major SWIZZLE_NONE layouts,
// D read back from TMEM, to pin the operand layouts against numpy
// (tools/umma_probe.py).
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t mkdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
         (1ull << 46);
}

// A: [M=128][K] row-major fp32 in global, B: [K][N=64] row-major in global, D: [128][64]
// amaj/bmaj: 0 = K-major, 1 = MN-major; lbo/sbo overrides for the MN-major operand (bytes)
extern "C" __global__ void k_probe(const float* A, const float* B, float* D, int KS, int amaj, int bmaj,
                                   int a_lbo, int a_sbo, int b_lbo, int b_sbo, int swapdesc) {
  constexpr int M = 128, N = 64;
  __shared__ __align__(128) uint32_t As[M * 32];
  __shared__ __align__(128) uint32_t Bs[N * 32];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_s;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int K = 8 * KS;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_s)), "n"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // A element (m, k)
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    int off;  // in 4-byte words
    if (amaj == 0) off = (k / 4) * (M * 4) + (m / 8) * 32 + (m % 8) * 4 + (k % 4);  // K-major: LBO = M*16 B, SBO = 128
    else off = (k / 8) * (a_lbo / 4) + (m / 4) * (a_sbo / 4) + (k % 8) * 4 + (m % 4);  // MN-major
    As[off] = __float_as_uint(A[m * K + k]) & 0xffffe000u;
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int k = i / N, n = i % N;
    int off;
    if (bmaj == 0) off = (k / 4) * (N * 4) + (n / 8) * 32 + (n % 8) * 4 + (k % 4);
    else off = (k / 8) * (b_lbo / 4) + (n / 4) * (b_sbo / 4) + (k % 8) * 4 + (n % 4);
    Bs[off] = __float_as_uint(B[k * N + n]) & 0xffffe000u;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_s;
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)amaj << 15) | ((uint32_t)bmaj << 16) |
                           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    for (int ks = 0; ks < KS; ++ks) {
      uint64_t da, db;
      if (amaj == 0) da = mkdesc(su32(As) + ks * 2 * M * 16, M * 16, 128);
      else da = swapdesc ? mkdesc(su32(As) + ks * a_lbo, a_sbo, a_lbo) : mkdesc(su32(As) + ks * a_lbo, a_lbo, a_sbo);
      if (bmaj == 0) db = mkdesc(su32(Bs) + ks * 2 * N * 16, N * 16, 128);
      else db = swapdesc ? mkdesc(su32(Bs) + ks * b_lbo, b_sbo, b_lbo) : mkdesc(su32(Bs) + ks * b_lbo, b_lbo, b_sbo);
      const uint32_t acc = ks > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
          "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mbar))
                 : "memory");
  }
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
          : "=r"(done)
          : "r"(su32(&mbar)), "r"(0)
          : "memory");
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int ch = warp >> 2;
  uint32_t v[32];
  const uint32_t taddr = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + 32 * ch;
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  const int m = 32 * (warp & 3) + (tid & 31);
  for (int q = 0; q < 32; ++q) D[m * N + 32 * ch + q] = __uint_as_float(v[q]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(64));
}

extern "C" int probe(const float* A, const float* B, float* D, int KS, int amaj, int bmaj, int a_lbo, int a_sbo,
                     int b_lbo, int b_sbo, int swapdesc) {
  k_probe<<<1, 256>>>(A, B, D, KS, amaj, bmaj, a_lbo, a_sbo, b_lbo, b_sbo, swapdesc);
  cudaError_t e = cudaDeviceSynchronize();
  return (int)e;
}
