"""Host-side cost of one async copy call (pinned H2D small / large, D2H) and
of a small kernel launch through the C ABI. GPU box: python tools/h2d_call_probe.py"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2303_13775_b200 import _lib  # noqa: E402

st = torch.cuda.current_stream().cuda_stream
small_h = torch.empty(4096, dtype=torch.float32, pin_memory=True)
big_h = torch.empty(650_000, dtype=torch.int32, pin_memory=True)
small_d = torch.empty(4096, dtype=torch.float32, device="cuda")
big_d = torch.empty(650_000, dtype=torch.int32, device="cuda")
fill = torch.empty(1, dtype=torch.float32, device="cuda")


def tm(f, k=300):
    for _ in range(30):
        f()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(k):
        f()
    t = time.perf_counter() - t
    torch.cuda.synchronize()
    return 1e6 * t / k


print("H2D 16 KB  %.1f us" % tm(lambda: _lib.call("sg_copy_async", small_d.data_ptr(), small_h.data_ptr(), 16384, st)))
print("H2D 2.6 MB %.1f us" % tm(lambda: _lib.call("sg_copy_async", big_d.data_ptr(), big_h.data_ptr(), 2_600_000, st), 50))
print("D2H 16 KB  %.1f us" % tm(lambda: _lib.call("sg_copy_async", small_h.data_ptr(), small_d.data_ptr(), 16384, st)))
print("D2D 2.6 MB %.1f us" % tm(lambda: _lib.call("sg_copy_async", big_d.data_ptr(), big_d.data_ptr() + 4, 2_000_000, st)))
print("stream_ptr %.1f us" % tm(lambda: _lib.stream_ptr()))
print("kernel     %.1f us" % tm(lambda: _lib.call("sg_fill_uniform", fill.data_ptr(), 1, 1, 1, 0, st)))
print("stream_ptr (raw) %.1f us; equal to torch's: %s" % (
    tm(lambda: _lib.stream_ptr()), _lib.stream_ptr() == torch.cuda.current_stream().cuda_stream))
s2 = torch.cuda.Stream()
with torch.cuda.stream(s2):
    print("inside a side stream: equal %s" % (_lib.stream_ptr() == s2.cuda_stream))
