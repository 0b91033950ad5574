"""H2D of a ~5 MB packed sample: torch pinned tensor vs cudaHostAlloc'd memory
(ctypes into libcudart) vs pageable, synchronous wall time per copy."""
import ctypes as C
import time

import numpy as np
import torch

n = 1_214_287
dst = torch.empty(n, dtype=torch.int32, device="cuda")
pin = torch.empty(n, dtype=torch.int32).pin_memory()
pin2 = torch.empty(n, dtype=torch.int32, pin_memory=True)
page = torch.empty(n, dtype=torch.int32)
print("is_pinned", pin.is_pinned(), pin[:n - 5].is_pinned(), pin2.is_pinned())
cudart = C.CDLL("libcudart.so") if False else None
try:
    import glob
    cands = glob.glob("/usr/local/cuda/lib64/libcudart.so*") + glob.glob(
        "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/cuda_runtime/lib/libcudart.so*")
    cudart = C.CDLL(cands[0])
except Exception as e:
    print("no cudart", e)


def t(fn, k=20):
    torch.cuda.synchronize()
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
        torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / k
    return f"{dt * 1e3:.3f} ms ({4 * n / dt / 1e9:.1f} GB/s)"


print("torch pinned      ", t(lambda: dst.copy_(pin, non_blocking=True)))
print("torch pinned slice", t(lambda: dst[:n - 5].copy_(pin[:n - 5], non_blocking=True)))
print("torch pin_memory=T", t(lambda: dst.copy_(pin2, non_blocking=True)))
print("torch pageable    ", t(lambda: dst.copy_(page)))
if cudart is not None:
    p = C.c_void_p()
    assert cudart.cudaHostAlloc(C.byref(p), C.c_size_t(4 * n), 0) == 0
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    print("cudaHostAlloc     ", t(lambda: cudart.cudaMemcpyAsync(C.c_void_p(dst.data_ptr()), p, C.c_size_t(4 * n), 1, st)))
    big = torch.empty(64 << 20, dtype=torch.int32).pin_memory()
    bd = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize(); t0 = time.perf_counter(); bd.copy_(big, non_blocking=True); torch.cuda.synchronize()
    print("256 MB pinned", f"{256 / 1024 / (time.perf_counter() - t0):.1f} GB/s")

# the same copies right after the host rewrote the buffer (split_minibatch packs
# each sample into its pinned slot, then copies it)
src = np.random.default_rng(0).integers(0, 1 << 30, n).astype(np.int32)
for name, buf in (("pin_memory()", pin), ("pin_memory=True", pin2)):
    def go(b=buf):
        b.numpy()[:] = src
        dst.copy_(b, non_blocking=True)
    print(f"rewrite+copy {name:16s}", t(go))
    def only_write(b=buf):
        b.numpy()[:] = src
    print(f"rewrite only {name:16s}", t(only_write))
