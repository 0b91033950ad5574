// Last GraphSAGE layer + classifier loss + the layer's row-local backward in
// ONE kernel (single-device split, g == 1).
//
// The final layer's rows are the targets; every quantity of its backward that
// does not cross an edge is row-local, so one CTA per 8-row tile runs
//   aggregation (engine.py:180-195) -> update, no ReLU (:212-226)
//   -> logits + summed softmax-CE + d_logits (models.py:287-302)
//   -> d_h = d_logits W_cls^T -> d_pre = d_h (final layer, engine.py:237)
//   -> dW_cls/db_cls/loss and dW_self/dW_neigh/db per-CTA partials
//      (engine.py:238-241), d_self = d_pre W_self^T, d_sums = d_pre W_neigh^T / N
//      (:242-244)
// with every intermediate in shared memory. The partials use the layouts of
// k_cls_loss and k_sage_wgrad, so sg_reduce_partials adds them in CTA order
// (deterministic). Replaces four launches (aggregate, linear, loss, wgrad).
#include <cstring>

#include "common.cuh"

namespace sg {
namespace {

constexpr int FTR = 8;  // rows per tile: one warp per row

struct FinalArgs {
  int L, d, w, dout, C;
  int64_t eoff_li, rbase_li, voff_l;
  const int32_t* rowbeg;
  const int32_t* rowend;
  const int32_t* lsrc;
  const int32_t* selfrow;
  const int32_t* src_row;
  const int32_t* grouped;
  const int32_t* V;
  const int32_t* labels;
  const float* h_prev;
  const float* ws;
  const float* wn;
  const float* bias;
  const float* wc;
  const float* bc;
  float* mean;
  float* counts;
  float* h;
  float* d_self;
  float* d_sums;
  float* part_cls;
  float* part_lay;
  // combine mode (g > 1): local partial + holders' partials (ascending sender)
  const float* sums;
  const float* recv;
  const int32_t* contrib;
  int stride, g;
};

__global__ void __launch_bounds__(256) k_sage_final(const SgMeta* __restrict__ meta, FinalArgs a) {
  // weights staged and accumulators zeroed before the PDL wait (nothing here
  // is written by the preceding kernel; parameters change only at step end)
  extern __shared__ __align__(16) float smem[];
  const int w = a.w, dout = a.dout, C = a.C, K = 2 * w, cp = C + 1;
  const int nwd = w * dout, nwc = dout * C;
  const int ncls = nwc + C + 1, nlay = 2 * nwd + dout;
  // every region starts on a 16-byte boundary (float4 row stores into A_s)
  auto r4 = [](int x) { return (x + 3) & ~3; };
  float* Ws = smem;                  // [w][dout]
  float* Wn = Ws + r4(nwd);          // [w][dout]
  float* bs = Wn + r4(nwd);          // [dout]
  float* Wc = bs + r4(dout);         // [dout][C]
  float* bcs = Wc + r4(nwc);         // [C]
  float* A_s = bcs + r4(C);          // [FTR][2w]  hs | mean
  float* h_s = A_s + FTR * K;        // [FTR][dout]
  float* lg = h_s + r4(FTR * dout);  // [FTR][C+1]  logits -> d_logits
  float* dp = lg + r4(FTR * cp);     // [FTR][dout] d_pre
  float* cnt = dp + r4(FTR * dout);  // [FTR] 1/N
  float* lossr = cnt + FTR;          // [FTR]
  int* ys = (int*)(lossr + FTR);
  float* acc_c = (float*)(ys + FTR);  // [ncls]
  float* acc_l = acc_c + r4(ncls);    // [nlay]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < nwd; i += 256) {
    Ws[i] = a.ws[i];
    Wn[i] = a.wn[i];
  }
  for (int i = tid; i < nwc; i += 256) Wc[i] = a.wc[i];
  for (int i = tid; i < C; i += 256) bcs[i] = a.bc[i];
  for (int i = tid; i < dout; i += 256) bs[i] = a.bias[i];
  for (int i = tid; i < ncls; i += 256) acc_c[i] = 0.f;
  for (int i = tid; i < nlay; i += 256) acc_l[i] = 0.f;
  const int l = a.L, d = a.d;
  const int n = meta->n_own[l][d];
  const int own0 = meta->own_off[l][d];
  const int prev0 = meta->own_off[l - 1][d];
  const int64_t rb = a.rbase_li + own0;
  // aggregation team: LPR lanes span the row (float4 each), EG edge groups
  const int w4 = w >> 2;
  const int LPR = w4 <= 4 ? 4 : w4 <= 8 ? 8 : w4 <= 16 ? 16 : 32;
  const int EG = 32 / LPR;
  const int eg = lane / LPR, lr = lane - eg * LPR;
  const int ntiles = (n + FTR - 1) / FTR;
  // also before the wait: the first tile's row bounds, this edge group's first
  // source index and the row's label -- all from the split / sample, which the
  // preceding kernel (the layer below, l >= 2) does not write. For l == 1 the
  // predecessor may be the split itself: no prefetch.
  const bool pre = l >= 2 && !a.sums;
  int b_pre = 0, e_pre = 0, rr_pre = -1, y_pre = -1;
  if (pre && blockIdx.x < ntiles) {
    const int q = blockIdx.x * FTR + warp;
    if (q < n) {
      b_pre = a.rowbeg[rb + q];
      e_pre = a.rowend[rb + q];
      if (b_pre + eg < e_pre) rr_pre = prev0 + a.lsrc[a.eoff_li + b_pre + eg];
      if (lane == 0) y_pre = a.labels[a.V[a.voff_l + a.grouped[a.voff_l + own0 + q]]];
    }
  }
  SG_PDL_ENTRY();
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const bool first_tile = pre && tile == (int)blockIdx.x;
    const int r0 = tile * FTR;
    const int rows = min(FTR, n - r0);
    __syncthreads();  // previous tile done with the smem rows
    // ---- aggregation: warp `warp` owns row r0 + warp
    {
      const int r = warp;
      if (r < rows) {
        const int q = r0 + r;
        const int b = a.sums ? 0 : (first_tile ? b_pre : a.rowbeg[rb + q]);
        const int e = a.sums ? 0 : (first_tile ? e_pre : a.rowend[rb + q]);
        const int64_t G = own0 + q;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        const bool colok = lr < w4;
        float cntf = (float)(e - b);
        if (a.sums) {  // combine mode: eg == 0 lanes hold the row, the xor tree adds zeros
          float N = a.counts[G];
          if (eg == 0 && colok) acc = *reinterpret_cast<const float4*>(a.sums + G * w + 4 * lr);
          const int32_t* cb = a.contrib + (int64_t)a.g * a.voff_l + G * a.g;
          for (int s = 0; s < a.g; ++s) {
            const int rs = cb[s];
            if (rs < 0) continue;
            const float* rrow = a.recv + (int64_t)rs * a.stride;
            if (eg == 0 && colok) {
              const float4 t = *reinterpret_cast<const float4*>(rrow + 4 * lr);
              acc.x += t.x; acc.y += t.y; acc.z += t.z; acc.w += t.w;
            }
            N += rrow[w];
          }
          cntf = N;
        } else {
          for (int j = b + eg; j < e; j += EG) {
            int rr = (first_tile && j == b + eg) ? rr_pre : prev0 + a.lsrc[a.eoff_li + j];
            if (a.src_row) rr = a.src_row[rr];
            if (colok) {
              const float4 v = __ldg(reinterpret_cast<const float4*>(a.h_prev + (int64_t)rr * w + 4 * lr));
              acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
            }
          }
        }
        for (int o = LPR; o < 32; o <<= 1) {
          acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
          acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
          acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
          acc.w += __shfl_xor_sync(0xffffffffu, acc.w, o);
        }
        if (eg == 0 && colok) {
          int rs = prev0 + a.selfrow[a.voff_l + G];
          if (a.src_row) rs = a.src_row[rs];
          const float4 hv = __ldg(reinterpret_cast<const float4*>(a.h_prev + (int64_t)rs * w + 4 * lr));
          const float inv = 1.0f / cntf;
          const float4 mn = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
          *reinterpret_cast<float4*>(A_s + r * K + 4 * lr) = hv;
          *reinterpret_cast<float4*>(A_s + r * K + w + 4 * lr) = mn;
          *reinterpret_cast<float4*>(a.mean + G * w + 4 * lr) = mn;
          if (lr == 0) {
            a.counts[G] = cntf;
            cnt[r] = inv;
          }
        }
        if (lane == 0) {
          if (first_tile) {
            ys[r] = y_pre;
          } else {
            const int p = a.grouped[a.voff_l + own0 + q];
            ys[r] = a.labels[a.V[a.voff_l + p]];
          }
        }
      } else {
        for (int k = lane; k < K; k += 32) A_s[r * K + k] = 0.f;
        if (lane == 0) {
          cnt[r] = 0.f;
          ys[r] = -1;
        }
      }
    }
    __syncthreads();
    // ---- update (final layer: no ReLU)
    for (int idx = tid; idx < FTR * dout; idx += 256) {
      const int r = idx / dout, j = idx - r * dout;
      float v = bs[j];
      const float* ar = A_s + r * K;
      for (int k = 0; k < w; ++k) v = fmaf(ar[k], Ws[k * dout + j], v);
      for (int k = 0; k < w; ++k) v = fmaf(ar[w + k], Wn[k * dout + j], v);
      if (r >= rows) v = 0.f;
      h_s[idx] = v;
      if (r < rows) a.h[(int64_t)(own0 + r0 + r) * dout + j] = v;
    }
    __syncthreads();
    // ---- logits
    for (int idx = tid; idx < FTR * C; idx += 256) {
      const int r = idx / C, c = idx - r * C;
      float v = bcs[c];
      for (int j = 0; j < dout; ++j) v = fmaf(h_s[r * dout + j], Wc[j * C + c], v);
      lg[r * cp + c] = v;
    }
    __syncthreads();
    // ---- softmax-CE, one warp per row
    {
      const int r = warp;
      const int y = ys[r];
      if (y < 0) {
        for (int c = lane; c < C; c += 32) lg[r * cp + c] = 0.f;
        if (lane == 0) lossr[r] = 0.f;
      } else {
        float m = -INFINITY;
        for (int c = lane; c < C; c += 32) m = fmaxf(m, lg[r * cp + c]);
#pragma unroll
        for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        float s = 0.f;
        for (int c = lane; c < C; c += 32) s += expf(lg[r * cp + c] - m);
#pragma unroll
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        const float ly = lg[r * cp + y];
        __syncwarp();
        const float inv = 1.0f / s;
        for (int c = lane; c < C; c += 32) {
          float pr = expf(lg[r * cp + c] - m) * inv;
          if (c == y) pr -= 1.0f;
          lg[r * cp + c] = pr;
        }
        if (lane == 0) lossr[r] = (m + logf(s)) - ly;
      }
    }
    __syncthreads();
    // ---- d_pre = d_logits W_cls^T; classifier partials
    for (int idx = tid; idx < FTR * dout; idx += 256) {
      const int r = idx / dout, j = idx - r * dout;
      float v = 0.f;
      for (int c = 0; c < C; ++c) v = fmaf(lg[r * cp + c], Wc[j * C + c], v);
      dp[idx] = v;
    }
    for (int slot = tid; slot < ncls; slot += 256) {
      float v = acc_c[slot];
      if (slot < nwc) {
        const int j = slot / C, c = slot - j * C;
        for (int r = 0; r < FTR; ++r) v = fmaf(h_s[r * dout + j], lg[r * cp + c], v);
      } else if (slot < nwc + C) {
        const int c = slot - nwc;
        for (int r = 0; r < FTR; ++r) v += lg[r * cp + c];
      } else {
        for (int r = 0; r < FTR; ++r) v += lossr[r];
      }
      acc_c[slot] = v;
    }
    __syncthreads();
    // ---- layer partials and the rows' input gradients
    for (int slot = tid; slot < nlay; slot += 256) {
      float v = acc_l[slot];
      if (slot < 2 * nwd) {
        const int kk = slot / dout, j = slot - kk * dout;  // kk < w: hs, else mean
        for (int r = 0; r < FTR; ++r) v = fmaf(A_s[r * K + kk], dp[r * dout + j], v);
      } else {
        const int j = slot - 2 * nwd;
        for (int r = 0; r < FTR; ++r) v += dp[r * dout + j];
      }
      acc_l[slot] = v;
    }
    for (int idx = tid; idx < rows * w; idx += 256) {
      const int r = idx / w, k = idx - r * w;
      float s1 = 0.f, s2 = 0.f;
      for (int j = 0; j < dout; ++j) {
        s1 = fmaf(dp[r * dout + j], Ws[k * dout + j], s1);
        s2 = fmaf(dp[r * dout + j], Wn[k * dout + j], s2);
      }
      const int64_t G = own0 + r0 + r;
      if (a.d_self) a.d_self[G * w + k] = s1;
      if (a.d_sums) a.d_sums[G * w + k] = s2 * cnt[r];
    }
  }
  __syncthreads();
  for (int i = tid; i < ncls; i += 256) a.part_cls[(int64_t)blockIdx.x * ncls + i] = acc_c[i];
  for (int i = tid; i < nlay; i += 256) a.part_lay[(int64_t)blockIdx.x * nlay + i] = acc_l[i];
}

}  // namespace
}  // namespace sg

using namespace sg;

static int final_impl(const void* split_ws, const SgSplitLayout* lay, int32_t d, const float* h_prev,
                      const int32_t* src_row, int32_t w, int32_t dout, int32_t ncls, const float* w_self,
                      const float* w_neigh, const float* bias, const float* w_cls, const float* b_cls,
                      const int32_t* V, const int32_t* labels, const float* sums, const float* recv,
                      int32_t recv_stride, float* mean, float* counts, float* h, float* d_self, float* d_sums,
                      float* part_cls, float* part_lay, int32_t nblocks, int64_t max_rows, void* stream) {
  SG_REQUIRE(split_ws && lay, "sage_final_fused: null workspace");
  const char* base = (const char*)split_ws;
  const SgSplitLayout& y = *lay;
  SG_REQUIRE(d >= 0 && d < y.g, "sage_final_fused: bad device");
  SG_REQUIRE(sums != nullptr || y.g == 1, "sage_final_fused: aggregate mode is single-device only");
  SG_REQUIRE(y.g == 1 || (recv && recv_stride % 4 == 0 && recv_stride >= w + 1),
             "sage_final_combine: recv stride must be a multiple of 4 and >= w + 1");
  SG_REQUIRE(w % 4 == 0 && w <= 128 && dout >= 1 && dout <= 64 && ncls >= 1 && ncls <= 1024,
             "sage_final_fused: needs w % 4 == 0, w <= 128, dout <= 64, classes <= 1024");
  SG_REQUIRE(nblocks >= 1, "sage_final_fused: nblocks >= 1");
  (void)max_rows;  // n_own is read on the device; an idle device still writes zero partials
  const int L = y.L;
  FinalArgs a;
  memset(&a, 0, sizeof(a));
  a.L = L; a.d = d; a.w = w; a.dout = dout; a.C = ncls;
  a.eoff_li = y.eoff[L - 1]; a.rbase_li = y.rbase[L - 1]; a.voff_l = y.voff[L];
  a.rowbeg = (const int32_t*)(base + y.o_rowbeg);
  a.rowend = (const int32_t*)(base + y.o_rowend);
  a.lsrc = (const int32_t*)(base + y.o_lsrc);
  a.selfrow = (const int32_t*)(base + y.o_selfrow);
  a.grouped = (const int32_t*)(base + y.o_grouped);
  a.src_row = src_row; a.V = V; a.labels = labels; a.h_prev = h_prev;
  a.ws = w_self; a.wn = w_neigh; a.bias = bias; a.wc = w_cls; a.bc = b_cls;
  a.mean = mean; a.counts = counts; a.h = h; a.d_self = d_self; a.d_sums = d_sums;
  a.part_cls = part_cls; a.part_lay = part_lay;
  a.sums = sums; a.recv = recv; a.stride = recv_stride; a.g = (sums && y.g > 1) ? y.g : 0;
  a.contrib = (const int32_t*)(base + y.o_contrib);
  const size_t nwd = (size_t)w * dout, nwc = (size_t)dout * ncls;
  auto r4 = [](size_t x) { return (x + 3) & ~(size_t)3; };
  const size_t floats = 2 * r4(nwd) + r4(dout) + r4(nwc) + r4(ncls) + FTR * 2 * (size_t)w +
                        r4(FTR * (size_t)dout) + r4(FTR * (size_t)(ncls + 1)) + r4(FTR * (size_t)dout) +
                        3 * FTR + r4(nwc + ncls + 1) + (2 * nwd + dout);
  const size_t smem = floats * sizeof(float);
  SG_REQUIRE(smem <= 200 * 1024, "sage_final_fused: layer too wide for shared memory");
  SG_CUDA(allow_max_smem<k_sage_final>());
  ::sg::launch(k_sage_final, nblocks, 256, smem, (cudaStream_t)stream, (const SgMeta*)(base + y.o_meta), a);
  SG_CHECK_LAUNCH("k_sage_final");
  return SG_OK;
}

extern "C" int sg_sage_final_fused(const void* split_ws, const SgSplitLayout* lay, int32_t d,
                                   const float* h_prev, const int32_t* src_row, int32_t w,
                                   int32_t dout, int32_t ncls, const float* w_self,
                                   const float* w_neigh, const float* bias, const float* w_cls,
                                   const float* b_cls, const int32_t* V, const int32_t* labels,
                                   float* mean, float* counts, float* h, float* d_self,
                                   float* d_sums, float* part_cls, float* part_lay,
                                   int32_t nblocks, int64_t max_rows, void* stream) {
  return final_impl(split_ws, lay, d, h_prev, src_row, w, dout, ncls, w_self, w_neigh, bias, w_cls, b_cls, V,
                    labels, nullptr, nullptr, 0, mean, counts, h, d_self, d_sums, part_cls, part_lay, nblocks,
                    max_rows, stream);
}

extern "C" int sg_sage_final_combine(const void* split_ws, const SgSplitLayout* lay, int32_t d,
                                     const float* h_prev, const int32_t* src_row, int32_t w, int32_t dout,
                                     int32_t ncls, const float* w_self, const float* w_neigh, const float* bias,
                                     const float* w_cls, const float* b_cls, const int32_t* V,
                                     const int32_t* labels, const float* sums, const float* recv,
                                     int32_t recv_stride, float* mean, float* counts, float* h, float* d_self,
                                     float* d_sums, float* part_cls, float* part_lay, int32_t nblocks,
                                     int64_t max_rows, void* stream) {
  SG_REQUIRE(sums && counts, "sage_final_combine: null sums/counts");
  return final_impl(split_ws, lay, d, h_prev, src_row, w, dout, ncls, w_self, w_neigh, bias, w_cls, b_cls, V,
                    labels, sums, recv, recv_stride, mean, counts, h, d_self, d_sums, part_cls, part_lay, nblocks,
                    max_rows, stream);
}
