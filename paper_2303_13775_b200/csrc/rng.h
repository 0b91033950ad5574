// Counter-based hashing RNG shared by host (generator, sampler) and device
// (synthetic features): splitmix64 finaliser over (seed, a, b). Results depend
// only on the counters, never on thread count or launch shape.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define SG_HD __host__ __device__ __forceinline__
#else
#define SG_HD inline
#endif

SG_HD uint64_t sg_mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

SG_HD uint64_t sg_hash3(uint64_t seed, uint64_t a, uint64_t b) {
  return sg_mix64(sg_mix64(sg_mix64(seed) ^ a) ^ (b * 0xD1B54A32D192ED03ull));
}

// U[0,1) with 24 random bits: exactly representable in fp32 and fp64.
SG_HD float sg_uniform24(uint64_t seed, uint64_t a, uint64_t b) {
  return (float)(sg_hash3(seed, a, b) >> 40) * (1.0f / 16777216.0f);
}

SG_HD double sg_uniform53(uint64_t h) { return (double)(h >> 11) * (1.0 / 9007199254740992.0); }

// Unbiased-enough bounded draw (Lemire multiply-shift, 64-bit source).
SG_HD uint64_t sg_bounded(uint64_t h, uint64_t bound) {
#ifdef __CUDA_ARCH__
  return __umul64hi(h, bound);
#else
  return (uint64_t)(((unsigned __int128)h * bound) >> 64);
#endif
}
