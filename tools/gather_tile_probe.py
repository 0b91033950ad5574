"""Diagnostic (not product code): gathers shaped like the tcgen05 projection tile
(128 rows x 25 chunks, 13 float4 per thread) at 1/2/4 CTAs per SM, plane-friendly
(8 rows x 4 chunks per warp instruction) vs row-contiguous lane mapping."""
import ctypes, os, subprocess, torch
HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_gather_dense_probe.so")
subprocess.check_call(["nvcc", "-O3", "-shared", "-Xcompiler", "-fPIC", "-gencode", "arch=compute_100a,code=sm_100a", "-o", SO, os.path.join(HERE, "gather_dense_probe.cu")])
lib = ctypes.CDLL(SO)
P, I = ctypes.c_void_p, ctypes.c_int
dev = torch.device("cuda:0")
n_tab = 2_449_029
for stride in (100, 128):
    tab = torch.rand(n_tab, stride, device=dev)
    flush = torch.empty(64 << 20, device=dev)
    n = 185_000
    idx = torch.randperm(n_tab, device=dev)[:n].to(torch.int32)
    out = torch.empty(148 * 4 * 256, device=dev)
    for pat in (0, 1):
        for mult in (1, 2, 4):
            ts = []
            for _ in range(7):
                flush.fill_(1.0)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); lib.probe_tile(I(pat), P(tab.data_ptr()), P(idx.data_ptr()), I(n), I(stride // 4), P(out.data_ptr()), I(148 * mult)); b.record()
                torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
            us = sorted(ts)[3]
            print(f"stride {stride*4}B pattern {pat} CTAs/SM {mult}: {us:6.1f} us  {n*400/us/1e3:6.0f} GB/s useful")
