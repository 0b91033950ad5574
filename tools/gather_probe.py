"""Practical roofline for the layer-1 access pattern: random 400-byte row
gathers from a 2.45M x 100 fp32 table (torch index_select, L2 flushed)."""
import torch

dev = torch.device("cuda", 0)
flush = torch.empty(256 * 2**20 // 4, device=dev)
for n, w in ((2_449_029, 100), (2_449_029, 128)):
    tab = torch.rand(n, w, device=dev)
    for rows in (179_000, 344_000, 2_000_000):
        idx = torch.randint(0, n, (rows,), device=dev)
        out = torch.empty(rows, w, device=dev)
        ts = []
        for it in range(8):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.index_select(tab, 0, idx, out=out)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = sorted(ts[2:])[len(ts[2:]) // 2]
        by = rows * w * 4 * 2 + rows * 8
        print(f"w={w} rows={rows}: {t*1e3:.1f} us  {by/t/1e6:.0f} GB/s (read+write+idx)  read-only {rows*w*4/t/1e6:.0f} GB/s")
    big = torch.empty(n, w, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); big.copy_(tab); e1.record(); torch.cuda.synchronize()
    print(f"contiguous copy {2*n*w*4/e0.elapsed_time(e1)/1e6:.0f} GB/s")
    del tab, big
