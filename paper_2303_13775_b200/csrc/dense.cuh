// Generic register-tiled FP32 GEMMs (dense.cu) used by the layer kernels
// outside their fast-path widths.
#pragma once
#include "common.cuh"

namespace sg {

// Row bases are DEVICE values (the split's own_off entries live in the
// SgMeta descriptor, so a captured graph serves every sample): a row index is
// (*base_dev) + add + r.
struct DenseRows {
  int mode;                  // 0: base + r   1: map[base + r]   2: SAGE self row of owned row base + r
  const int32_t* base_dev;   // may be null (base 0)
  int64_t add;
  const int32_t* map;        // mode 1; mode 2: layer-1 src_row applied after the self-row lookup
  const int32_t* selfrow;    // mode 2: *prev0_dev + selfrow[voff_l + base + r]
  const int32_t* prev0_dev;
  int64_t voff_l;
};

struct GemmArgs {
  const int32_t* R_dev;      // live row count (device)
  int K, N;
  const float* A;
  int64_t lda;
  DenseRows ar;
  const float* amask;        // A(r, k) zeroed where amask[(out_row(r)) * lda_mask + k] <= 0
  int64_t lda_mask;
  const float* B;
  int64_t ldb;
  int bt;                    // B(k, n) = bt ? B[n * ldb + k] : B[k * ldb + n]
  float* C;                  // row out_row(r) = (*c_base_dev) + r
  int64_t ldc;
  const int32_t* c_base_dev;
  int accum, relu;
  const float* bias;         // [N]
  const float* rdiv;         // C row scaled by 1 / rdiv[out_row(r)]
};

struct TnArgs {
  const int32_t* R_dev;
  int K, N, ones;            // ones: virtual column K of A == 1 (bias gradient)
  const float* A;
  int64_t lda;
  DenseRows ar;
  const float* G;            // row (*g_base_dev) + r
  int64_t ldg;
  const int32_t* g_base_dev;
  const float* gmask;        // G(r, n) zeroed where gmask[same index] <= 0
  float* P;                  // [nsplit][pstride], this GEMM at column offset p_off
  int64_t pstride, p_off;
  int nsplit;
};

int dense_gemm_rows(const GemmArgs& a, int64_t max_rows, cudaStream_t st);
int dense_gemm_tn_partial(const TnArgs& a, cudaStream_t st);

}  // namespace sg
