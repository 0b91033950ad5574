"""Diagnostic (not product code): pin tcgen05 kind::tf32 operand layouts
(K-major / MN-major, LBO vs SBO meaning) against numpy. See umma_probe.cu."""
import ctypes, os, subprocess
import numpy as np
import torch
HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_umma_probe.so")
subprocess.check_call(["nvcc", "-O2", "-shared", "-Xcompiler", "-fPIC", "-gencode", "arch=compute_100a,code=sm_100a",
                       "-o", SO, os.path.join(HERE, "umma_probe.cu")])
lib = ctypes.CDLL(SO)
P, I = ctypes.c_void_p, ctypes.c_int
rng = np.random.default_rng(0)
for KS in (1, 4):
    K = 8 * KS
    A = rng.standard_normal((128, K)).astype(np.float32)
    B = rng.standard_normal((K, 64)).astype(np.float32)
    tr = lambda x: (x.view(np.uint32) & np.uint32(0xffffe000)).view(np.float32)
    ref = tr(A).astype(np.float64) @ tr(B).astype(np.float64)
    At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    for amaj, bmaj, al, asb, bl, bsb, sw in [(0, 0, 0, 0, 0, 0, 0),
                                         (1, 0, 4096, 128, 0, 0, 0), (1, 0, 4096, 128, 0, 0, 1),
                                         (0, 1, 0, 0, 2048, 128, 0), (0, 1, 0, 0, 2048, 128, 1),
                                         (1, 1, 4096, 128, 2048, 128, 0), (1, 1, 4096, 128, 2048, 128, 1)]:
        D = torch.zeros(128, 64, device="cuda")
        rc = lib.probe(P(At.data_ptr()), P(Bt.data_ptr()), P(D.data_ptr()), I(KS), I(amaj), I(bmaj), I(al), I(asb),
                       I(bl), I(bsb), I(sw))
        torch.cuda.synchronize()
        d = D.cpu().numpy().astype(np.float64)
        err = np.abs(d - ref).max() / np.abs(ref).max()
        print(f"KS={KS} amaj={amaj} bmaj={bmaj} A(lbo={al},sbo={asb}) B(lbo={bl},sbo={bsb}) swap={sw} rc={rc} "
              f"rel err {err:.2e} |D|max {np.abs(d).max():.3f}")
