"""Diagnostic (not product code): the practical HBM ceiling of the layer-1
access pattern -- rows of a 2.45M x F fp32 table gathered by index and summed
per destination (16 per destination) -- with a deliberately simple kernel
that keeps many independent 128-bit loads in flight (one warp per
destination, 16 rows x 8 float4 per lane in flight). Compiled at run time
with torch's inline extension; reports GB/s of row bytes read.

  python tools/gather_roof.py
"""
import torch
from torch.utils.cpp_extension import load_inline

SRC = r"""
#include <cuda_runtime.h>
#include <torch/extension.h>
template <int F4>
__global__ void __launch_bounds__(256) k_gather(const float4* __restrict__ tab, const int* __restrict__ idx,
                                               float4* __restrict__ out, int ndst, int deg, int S4) {
  const int lane = threadIdx.x & 31;
  for (int v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < ndst; v += (gridDim.x * blockDim.x) >> 5) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const int r = lane < deg ? idx[v * deg + lane] : 0;
    float4 t[16];
    const bool ok = lane < F4;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int rr = __shfl_sync(0xffffffffu, r, k);
      t[k] = (k < deg && ok) ? __ldg(tab + (size_t)rr * S4 + lane) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) { acc.x += t[k].x; acc.y += t[k].y; acc.z += t[k].z; acc.w += t[k].w; }
    if (ok) out[(size_t)v * F4 + lane] = acc;
  }
}
// 512-byte line-aligned window per row (4 full 128 B lines, all 32 lanes),
// rotated into column order with shuffles: unpadded 400 B rows, full-line loads
__global__ void __launch_bounds__(256) k_gather_win(const float4* __restrict__ tab, int64_t n4,
                                                   const int* __restrict__ idx, float4* __restrict__ out,
                                                   int ndst, int deg) {
  const int lane = threadIdx.x & 31;
  for (int v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < ndst; v += (gridDim.x * blockDim.x) >> 5) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const int r = lane < deg ? idx[v * deg + lane] : 0;
    float4 t[16];
    int sh[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int rr = __shfl_sync(0xffffffffu, r, k);
      const int64_t f = (int64_t)rr * 25;
      const int64_t a0 = f & ~(int64_t)7;
      sh[k] = (int)(f - a0);
      const int64_t ai = a0 + lane;
      t[k] = (k < deg && ai < n4) ? __ldg(tab + ai) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int src = (lane + sh[k]) & 31;
      acc.x += __shfl_sync(0xffffffffu, t[k].x, src);
      acc.y += __shfl_sync(0xffffffffu, t[k].y, src);
      acc.z += __shfl_sync(0xffffffffu, t[k].z, src);
      acc.w += __shfl_sync(0xffffffffu, t[k].w, src);
    }
    if (lane < 25) out[(size_t)v * 25 + lane] = acc;
  }
}
void gather_win(torch::Tensor tab, torch::Tensor idx, torch::Tensor out, int64_t deg, int64_t blocks) {
  auto st = at::cuda::getCurrentCUDAStream();
  k_gather_win<<<blocks, 256, 0, st>>>((const float4*)tab.data_ptr(), tab.numel() / 4, idx.data_ptr<int>(),
                                      (float4*)out.data_ptr(), out.size(0), (int)deg);
}
void gather(torch::Tensor tab, torch::Tensor idx, torch::Tensor out, int64_t deg, int64_t blocks) {
  const int ndst = out.size(0);
  const int F4 = out.size(1) / 4;
  const int S4 = tab.size(1) / 4;
  auto st = at::cuda::getCurrentCUDAStream();
  if (F4 == 25) k_gather<25><<<blocks, 256, 0, st>>>((const float4*)tab.data_ptr(), idx.data_ptr<int>(),
                                                  (float4*)out.data_ptr(), ndst, (int)deg, S4);
  else k_gather<32><<<blocks, 256, 0, st>>>((const float4*)tab.data_ptr(), idx.data_ptr<int>(),
                                          (float4*)out.data_ptr(), ndst, (int)deg, S4);
}
"""
CPP = ("void gather(torch::Tensor tab, torch::Tensor idx, torch::Tensor out, int64_t deg, int64_t blocks);\n"
       "void gather_win(torch::Tensor tab, torch::Tensor idx, torch::Tensor out, int64_t deg, int64_t blocks);")


def main():
    mod = load_inline("gather_roof", CPP, cuda_sources=SRC.replace("#include <torch/extension.h>",
                      "#include <torch/extension.h>\n#include <ATen/cuda/CUDAContext.h>"),
                      functions=["gather", "gather_win"], extra_cuda_cflags=["-O3", "-gencode", "arch=compute_100a,code=sm_100a"],
                      verbose=False)
    dev = torch.device("cuda")
    n = 2_449_029
    flush = torch.empty(256 << 18, device=dev)
    for F, S, win in ((100, 100, False), (100, 100, True), (100, 128, False), (128, 128, False)):
        tab = torch.rand(n, S, device=dev)
        for dist in ("uniform", "powerlaw"):
            ndst, deg = 27_000, 16
            if dist == "uniform":
                idx = torch.randint(0, n, (ndst * deg,), device=dev, dtype=torch.int32)
            else:  # Zipf-like reuse, as sampled neighbourhoods have
                r = torch.rand(ndst * deg, device=dev)
                idx = (n * r.pow(3.0)).to(torch.int32).clamp_(0, n - 1)
                idx = idx[torch.randperm(idx.numel(), device=dev)]
            out = torch.empty(ndst, F, device=dev)
            for blocks in (148 * 8,):
                ts = []
                for _ in range(10):
                    flush.zero_()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    (mod.gather_win if win else mod.gather)(tab, idx, out, deg, blocks)
                    e1.record()
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1))
                t = sorted(ts[2:])[len(ts[2:]) // 2]
                byts = ndst * deg * F * 4
                print(f"F={F} stride={S} win={win} {dist:8s}: {t * 1e3:.1f} us, row bytes {byts / 1e6:.0f} MB -> "
                      f"{byts / t / 1e6:.0f} GB/s")
        del tab


if __name__ == "__main__":
    main()
