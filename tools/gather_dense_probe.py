"""Diagnostic (not product code): HBM ceiling of a once-per-unique-row gather
(180K random rows of a 2.45M x 128-float table, 400 useful bytes per row), by
register loads and by cp.async.bulk rings.  See gather_dense_probe.cu.

  python tools/gather_dense_probe.py
"""
import ctypes
import os
import subprocess

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_gather_dense_probe.so")
if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(os.path.join(HERE, "gather_dense_probe.cu")):
    subprocess.check_call(["nvcc", "-O3", "-shared", "-Xcompiler", "-fPIC", "-gencode",
                           "arch=compute_100a,code=sm_100a", "-o", SO, os.path.join(HERE, "gather_dense_probe.cu")])
lib = ctypes.CDLL(SO)
P = ctypes.c_void_p
I = ctypes.c_int


def main():
    dev = torch.device("cuda:0")
    n_tab, stride = 2_449_029, 128
    tab = torch.rand(n_tab, stride, device=dev)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    for n in (180_000, 1_000_000):
        idx = torch.randperm(n_tab, device=dev)[:n].to(torch.int32)
        # sorted indices too (the dense pass can visit V^0 rows in any order)
        idx_sorted = torch.sort(idx).values
        out = torch.empty(n, device=dev)
        ref = tab[idx.long(), :100].sum(1)

        def timeit(fn, reps=10):
            ts = []
            for _ in range(reps):
                flush.fill_(1.0)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                fn()
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b) * 1e3)
            ts.sort()
            return ts[len(ts) // 2]

        print(f"--- n = {n} rows, useful bytes {n * 400 / 1e6:.1f} MB")
        for order, ix in (("random", idx), ("sorted", idx_sorted)):
            for v, name in ((5, "reg U2 L25"), (0, "reg U4 L25"), (1, "reg U8 L25"), (4, "reg U16 L25"),
                            (2, "reg U4 L32"), (3, "reg U8 L32")):
                for blocks in (148 * 8, 148 * 16):
                    f = lambda: lib.probe_reg(I(v), P(tab.data_ptr()), P(ix.data_ptr()), I(n), I(stride // 4),
                                              P(out.data_ptr()), I(blocks))
                    us = timeit(f)
                    print(f"{order:6s} {name:12s} blocks {blocks:5d}: {us:7.1f} us  {n * 400 / us / 1e3:6.0f} GB/s useful")
            for v, name, bl in ((0, "bulk T32 S4", 3), (1, "bulk T32 S8", 1), (2, "bulk T64 S3", 2), (3, "bulk T16 S6", 4)):
                for rb in (400, 512):
                    for mult in (bl, bl * 2):
                        blocks = 148 * mult
                        f = lambda: lib.probe_bulk(I(v), P(tab.data_ptr()), P(ix.data_ptr()), I(n), I(stride), I(rb),
                                                   P(out.data_ptr()), I(blocks))
                        us = timeit(f)
                        print(f"{order:6s} {name:12s} RB {rb} blocks {blocks:5d}: {us:7.1f} us  "
                              f"{n * 400 / us / 1e3:6.0f} GB/s useful")
            if order == "random":
                lib.probe_bulk(I(0), P(tab.data_ptr()), P(idx.data_ptr()), I(n), I(stride), I(400), P(out.data_ptr()),
                               I(148 * 3))
                torch.cuda.synchronize()
                print("bulk check max err", (out - ref).abs().max().item())
                lib.probe_reg(I(0), P(tab.data_ptr()), P(idx.data_ptr()), I(n), I(stride // 4), P(out.data_ptr()),
                              I(148 * 8))
                torch.cuda.synchronize()
                print("reg check max err", (out - ref).abs().max().item())


if __name__ == "__main__":
    main()
