// Classifier loss, deterministic gradient reduction and the SGD step.
//
//   sg_cls_loss        classifier_loss (models.py:287-302) for the owned target
//                      rows of one device: logits, summed softmax-CE, d_h and
//                      per-block partials of dW_cls, db_cls and the loss.
//   sg_reduce_partials per-block partials -> gradients in ascending block
//                      order (replaces float atomics: run-to-run bit-identical)
//   sg_sum_sgd         allreduce_and_step (engine.py:633-647): device-order sum
//                      then p -= lr/num_targets * g (ModelParams.sgd_step,
//                      models.py:95-99).
#include <algorithm>
#include <cstring>

#include "common.cuh"

namespace sg {
namespace {

constexpr int LTR = 8;  // rows per tile (small: the batch is only ~1K rows)
constexpr int LMAXACC = 24;

struct LossArgs {
  int L, d, hid, ncls;
  int64_t voff_L;
  const int32_t* V;
  const int32_t* grouped;
  const int32_t* labels;
  const float* h;
  const float* w;  // [hid][ncls]
  const float* b;
  float* d_h;
  float* partial;
  int w_smem;  // stage W in shared memory (else read it through L1/L2)
};

__global__ void __launch_bounds__(256) k_cls_loss(const SgMeta* __restrict__ meta, LossArgs a) {
  // W staged before the PDL wait (parameters are not written by the preceding kernel)
  extern __shared__ float smem[];
  const int hid = a.hid, C = a.ncls, cp = C + 1;
  float* w_s = smem;                // [hid][C] when staged
  float* h_s = w_s + (a.w_smem ? hid * C : 0);  // [LTR][hid]
  float* lg_s = h_s + LTR * hid;    // [LTR][C+1]  logits, then d_logits
  int* y_s = (int*)(lg_s + LTR * cp);
  float* loss_s = (float*)(y_s + LTR);
  if (a.w_smem)
    for (int i = threadIdx.x; i < hid * C; i += blockDim.x) w_s[i] = a.w[i];
  SG_PDL_ENTRY();
  const float* Wm = a.w_smem ? w_s : a.w;
  const int n = meta->n_own[a.L][a.d];
  const int own0 = meta->own_off[a.L][a.d];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwc = hid * C;
  const int64_t ntot = (int64_t)nwc + C + 1;
  float* out = a.partial + (int64_t)blockIdx.x * ntot;
  float ab = 0.f, al = 0.f;
  const int ntiles = (n + LTR - 1) / LTR;
  // dW_cls slots in passes of 256 * LMAXACC (one pass unless hid * C > 6144);
  // d_h, db and the loss are produced in pass 0
  for (int slot0 = 0; slot0 < nwc; slot0 += 256 * LMAXACC) {
  const bool first = slot0 == 0;
  float aw[LMAXACC];
#pragma unroll
  for (int k = 0; k < LMAXACC; ++k) aw[k] = 0.f;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < LTR * hid; idx += blockDim.x) {
      const int rr = idx / hid, j = idx - rr * hid;
      const int q = tile * LTR + rr;
      h_s[idx] = q < n ? a.h[(int64_t)(own0 + q) * hid + j] : 0.f;
    }
    if (threadIdx.x < LTR) {
      const int q = tile * LTR + threadIdx.x;
      int y = -1;
      if (q < n) {
        const int p = a.grouped[a.voff_L + own0 + q];
        y = a.labels[a.V[a.voff_L + p]];
      }
      y_s[threadIdx.x] = y;
      loss_s[threadIdx.x] = 0.f;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < LTR * C; idx += blockDim.x) {
      const int rr = idx / C, c = idx - rr * C;
      float acc = a.b[c];
      for (int j = 0; j < hid; ++j) acc = fmaf(h_s[rr * hid + j], Wm[j * C + c], acc);
      lg_s[rr * cp + c] = acc;
    }
    __syncthreads();
    for (int rr = warp; rr < LTR; rr += 8) {  // one warp per row
      const int y = y_s[rr];
      if (y < 0) {
        for (int c = lane; c < C; c += 32) lg_s[rr * cp + c] = 0.f;
        continue;
      }
      float m = -INFINITY;
      for (int c = lane; c < C; c += 32) m = fmaxf(m, lg_s[rr * cp + c]);
#pragma unroll
      for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      float s = 0.f;
      for (int c = lane; c < C; c += 32) s += expf(lg_s[rr * cp + c] - m);
#pragma unroll
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      const float ly = lg_s[rr * cp + y];
      __syncwarp();
      const float inv = 1.0f / s;
      for (int c = lane; c < C; c += 32) {
        float p = expf(lg_s[rr * cp + c] - m) * inv;
        if (c == y) p -= 1.0f;
        lg_s[rr * cp + c] = p;
      }
      if (lane == 0) loss_s[rr] = (m + logf(s)) - ly;
    }
    __syncthreads();
    // d_h = d_logits @ W^T
    for (int idx = threadIdx.x; first && idx < LTR * hid; idx += blockDim.x) {
      const int rr = idx / hid, j = idx - rr * hid;
      const int q = tile * LTR + rr;
      if (q >= n) continue;
      float acc = 0.f;
      for (int c = 0; c < C; ++c) acc = fmaf(lg_s[rr * cp + c], Wm[j * C + c], acc);
      a.d_h[(int64_t)(own0 + q) * hid + j] = acc;
    }
#pragma unroll
    for (int k = 0; k < LMAXACC; ++k) {
      const int idx = slot0 + threadIdx.x + 256 * k;
      if (idx < nwc) {
        const int j = idx / C, c = idx - j * C;
        float s = aw[k];
        for (int rr = 0; rr < LTR; ++rr) s = fmaf(h_s[rr * hid + j], lg_s[rr * cp + c], s);
        aw[k] = s;
      }
    }
    if (first && threadIdx.x < C)
      for (int rr = 0; rr < LTR; ++rr) ab += lg_s[rr * cp + threadIdx.x];
    if (first && threadIdx.x == 0)
      for (int rr = 0; rr < LTR; ++rr) al += loss_s[rr];
  }
#pragma unroll
  for (int k = 0; k < LMAXACC; ++k) {
    const int idx = slot0 + threadIdx.x + 256 * k;
    if (idx < nwc) out[idx] = aw[k];
  }
  }
  if (threadIdx.x < C) out[nwc + threadIdx.x] = ab;
  if (threadIdx.x == 0) out[nwc + C] = al;
}

constexpr int MAXJOBS = 48;
struct Jobs {
  int64_t v[4 * MAXJOBS];
};
struct DevPtrs {
  int64_t v[SG_MAXG];
};

// Block = 32 output columns x 8 warps; warp w sums partial rows b = w, w+8, ...
// (8 loads in flight), then the 8 warp sums are added in warp order. With a
// parameter pointer (sgd job), the summed gradient g of the first n_sgd
// columns also takes the SGD step p -= scale * g in the same pass (g = 1:
// allreduce_and_step has nothing to sum, engine.py:633-647).
struct SgdJobs {
  int64_t param[MAXJOBS];
  int64_t n_sgd[MAXJOBS];
  float scale;
  double lr;                  // with nt: scale = lr / *nt, computed on the device
  const int64_t* nt;          // device num_targets of the step's sample (nullable)
};

__global__ void __launch_bounds__(256) k_reduce_partials(Jobs jobs, SgdJobs sj) {
  SG_PDL_ENTRY();
  __shared__ float red[8][33];
  const int jb = blockIdx.y;
  const float* p = (const float*)jobs.v[4 * jb + 0];
  const int nb = (int)jobs.v[4 * jb + 1];
  const int64_t n = jobs.v[4 * jb + 2];
  float* out = (float*)jobs.v[4 * jb + 3];
  float* prm = (float*)sj.param[jb];
  const int64_t n_sgd = sj.n_sgd[jb];
  // lr / num_targets (allreduce_and_step, engine.py:633-647) in double, as the
  // host computes it, from the sample's own target count
  const float scale = sj.nt ? (float)(sj.lr / (double)max(*sj.nt, (int64_t)1)) : sj.scale;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t k0 = (int64_t)blockIdx.x * 32; k0 < n; k0 += (int64_t)gridDim.x * 32) {
    const int64_t k = k0 + lane;
    float s[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) s[u] = 0.f;
    if (k < n) {
      int b = warp;
      for (; b + 56 < nb; b += 64) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = p[(int64_t)(b + 8 * u) * n + k];
#pragma unroll
        for (int u = 0; u < 8; ++u) s[u] += v[u];
      }
      for (; b < nb; b += 8) s[0] += p[(int64_t)b * n + k];
    }
    __syncthreads();
    red[warp][lane] = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
    __syncthreads();
    if (warp == 0 && k < n) {
      float t = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) t += red[w][lane];
      out[k] = t;
      if (prm && k < n_sgd) prm[k] -= scale * t;
    }
  }
}

__global__ void k_sum_sgd(float* __restrict__ params, float* __restrict__ gout, DevPtrs gptrs,
                          int ndev, int64_t n, float scale) {
  SG_PDL_ENTRY();
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    float s = ((const float*)gptrs.v[0])[k];
    for (int d = 1; d < ndev; ++d) s += ((const float*)gptrs.v[d])[k];
    if (gout) gout[k] = s;
    params[k] -= scale * s;
  }
}

// sg_sum_sgd with n1 >= n summed columns (the loss slot rides along) and the
// scale lr / *nt computed on the device.
__global__ void k_sum_sgd_nt(float* __restrict__ params, float* __restrict__ gout, DevPtrs gptrs,
                             int ndev, int64_t n, int64_t n1, double lr, const int64_t* __restrict__ nt) {
  SG_PDL_ENTRY();
  const float scale = (float)(lr / (double)max(*nt, (int64_t)1));
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n1;
       k += (int64_t)gridDim.x * blockDim.x) {
    float s = ((const float*)gptrs.v[0])[k];
    for (int d = 1; d < ndev; ++d) s += ((const float*)gptrs.v[d])[k];
    if (gout) gout[k] = s;
    if (k < n) params[k] -= scale * s;
  }
}

}  // namespace

extern "C" int sg_cls_loss(const void* split_ws, const SgSplitLayout* lay, int32_t d,
                           const int32_t* V, const int32_t* labels, const float* h, int32_t hid,
                           int32_t ncls, const float* w_cls, const float* b_cls, float* d_h,
                           float* partial, int32_t nblocks, int64_t max_rows, void* stream) {
  SG_REQUIRE(split_ws && lay, "cls_loss: null workspace");
  const char* base = (const char*)split_ws;
  const SgSplitLayout& y = *lay;
  SG_REQUIRE(d >= 0 && d < y.g, "cls_loss: bad device");
  SG_REQUIRE(hid >= 1 && ncls >= 1 && ncls <= 256, "cls_loss: classes must be 1..256");
  SG_REQUIRE(nblocks >= 1, "cls_loss: nblocks >= 1");
  (void)max_rows;
  LossArgs a;
  memset(&a, 0, sizeof(a));
  a.L = y.L;
  a.d = d;
  a.hid = hid;
  a.ncls = ncls;
  a.voff_L = y.voff[y.L];
  a.V = V;
  a.grouped = (const int32_t*)(base + y.o_grouped);
  a.labels = labels;
  a.h = h;
  a.w = w_cls;
  a.b = b_cls;
  a.d_h = d_h;
  a.partial = partial;
  const size_t smem_rest = sizeof(float) * ((size_t)LTR * hid + (size_t)LTR * (ncls + 1) + 2 * LTR);
  const size_t smem_w = sizeof(float) * (size_t)hid * ncls;
  a.w_smem = smem_rest + smem_w <= 96 * 1024;  // else W is read through L1/L2
  const size_t smem = smem_rest + (a.w_smem ? smem_w : 0);
  SG_REQUIRE(smem <= 227 * 1024, "cls_loss: hidden too large for shared memory");
  cudaStream_t st = (cudaStream_t)stream;
  SG_CUDA(allow_max_smem<k_cls_loss>());
  ::sg::launch(k_cls_loss, nblocks, 256, smem, st, (const SgMeta*)(base + y.o_meta), a);
  SG_CHECK_LAUNCH("k_cls_loss");
  return SG_OK;
}

static int reduce_partials(const int64_t* jobs, int stride, int32_t n_jobs, int64_t max_n, float scale,
                           void* stream, double lr = 0.0, const int64_t* nt = nullptr) {
  if (n_jobs <= 0 || max_n <= 0) return SG_OK;
  SG_REQUIRE(jobs != nullptr, "reduce_partials: null job table");
  for (int j0 = 0; j0 < n_jobs; j0 += MAXJOBS) {
    const int nj = std::min(MAXJOBS, n_jobs - j0);
    Jobs jb;
    SgdJobs sj;
    memset(&jb, 0, sizeof(jb));
    memset(&sj, 0, sizeof(sj));
    sj.scale = scale;
    sj.lr = lr;
    sj.nt = nt;
    for (int j = 0; j < nj; ++j) {
      const int64_t* r = jobs + (int64_t)stride * (j0 + j);
      for (int f = 0; f < 4; ++f) jb.v[4 * j + f] = r[f];
      if (stride >= 6) {
        sj.param[j] = r[4];
        sj.n_sgd[j] = r[5];
      }
    }
    dim3 grid(clamp_grid(div_up(max_n, 32), kSMs * 2), nj);
    ::sg::launch(k_reduce_partials, grid, 256, 0, (cudaStream_t)stream, jb, sj);
    SG_CHECK_LAUNCH("k_reduce_partials");
  }
  return SG_OK;
}

extern "C" int sg_reduce_partials(const int64_t* jobs, int32_t n_jobs, int64_t max_n,
                                  void* stream) {
  return reduce_partials(jobs, 4, n_jobs, max_n, 0.f, stream);
}

extern "C" int sg_reduce_partials_sgd(const int64_t* jobs, int32_t n_jobs, int64_t max_n, float scale,
                                      void* stream) {
  return reduce_partials(jobs, 6, n_jobs, max_n, scale, stream);
}

extern "C" int sg_reduce_partials_sgd_nt(const int64_t* jobs, int32_t n_jobs, int64_t max_n, double lr,
                                         const int64_t* num_targets, void* stream) {
  SG_REQUIRE(num_targets != nullptr, "reduce_partials_sgd_nt: null num_targets");
  return reduce_partials(jobs, 6, n_jobs, max_n, 0.f, stream, lr, num_targets);
}

extern "C" int sg_sum_sgd(float* params, float* grads_out, const int64_t* grad_ptrs,
                          int32_t n_dev, int64_t n, float scale, void* stream) {
  SG_REQUIRE(params && grad_ptrs && n_dev >= 1 && n_dev <= SG_MAXG, "sum_sgd: bad arguments");
  if (n <= 0) return SG_OK;
  DevPtrs gp;
  memset(&gp, 0, sizeof(gp));
  for (int d = 0; d < n_dev; ++d) gp.v[d] = grad_ptrs[d];
  ::sg::launch(k_sum_sgd, clamp_grid(div_up(n, 256), kSMs * 4), 256, 0, (cudaStream_t)stream, params, grads_out, gp, n_dev, n, scale);
  SG_CHECK_LAUNCH("k_sum_sgd");
  return SG_OK;
}

extern "C" int sg_sum_sgd_nt(float* params, float* grads_out, const int64_t* grad_ptrs, int32_t n_dev,
                             int64_t n, int64_t n1, double lr, const int64_t* num_targets, void* stream) {
  SG_REQUIRE(params && grad_ptrs && num_targets && n_dev >= 1 && n_dev <= SG_MAXG && n1 >= n,
             "sum_sgd_nt: bad arguments");
  if (n1 <= 0) return SG_OK;
  DevPtrs gp;
  memset(&gp, 0, sizeof(gp));
  for (int d = 0; d < n_dev; ++d) gp.v[d] = grad_ptrs[d];
  ::sg::launch(k_sum_sgd_nt, clamp_grid(div_up(n1, 256), kSMs * 4), 256, 0, (cudaStream_t)stream, params, grads_out,
               gp, n_dev, n, n1, lr, num_targets);
  SG_CHECK_LAUNCH("k_sum_sgd_nt");
  return SG_OK;
}

}  // namespace sg
