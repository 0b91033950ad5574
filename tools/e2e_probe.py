"""Diagnostic: where the end-to-end (pinned host sample -> loss) time goes
for the captured C2 step. Not a bench line."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2303_13775_b200 as sg  # noqa: E402
from paper_2303_13775_b200 import _lib  # noqa: E402
from paper_2303_13775_b200.engine import CapturedStep, PinnedSample, capacities_for  # noqa: E402


def timed(fn, n):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n, (time.perf_counter() - t) * 1e3 / n


def main():
    dev = torch.device("cuda:0")
    graph, labels, train, _ = bench.build_workload(16)
    K = 30
    samples, _ = bench.make_samples(graph, train, K + 2, bench.BATCH, 16)
    pm = sg.range_partition(graph.num_vertices, 1)
    cache = sg.full_cache(pm)
    feats = sg.FeatureStore.synthetic(graph.num_vertices, bench.FEAT, seed=1)
    lab = torch.from_numpy(labels).to(dev)
    params = sg.init_params("graphsage", bench.FEAT, bench.HIDDEN, bench.CLASSES, 3, seed=0)
    dp = sg.DeviceParams.from_host(params)
    cap_nV, cap_nE = capacities_for(samples)
    rec = os.environ.get("PROBE_EVENTS") or False
    cs = CapturedStep(dp, pm, cache, feats, lab, cap_nV, cap_nE, 1e-3, dev, record_events=rec)
    cs.capture(samples[0])
    print("record_events", rec)
    pinned = [PinnedSample(s, cs.inp) for s in samples[2:]]
    nb = pinned[0].h2d_bytes
    print("h2d bytes", nb, "words", cs.inp.words)

    def replays():
        for _ in range(K):
            cs.graph.replay()
    print("replay only   (dev ms, wall ms) per step", timed(replays, K))

    stage = torch.empty(cs.inp.words, dtype=torch.int32, device=dev)
    def h2d_only():
        for p in pinned:
            stage[:p.buf.numel()].copy_(p.buf, non_blocking=True)
    print("h2d only torch (dev ms, wall ms)", timed(h2d_only, K))

    def d2d_only():
        for p in pinned:
            cs.inp.buf[:p.buf.numel()].copy_(stage[:p.buf.numel()], non_blocking=True)
    print("d2d only torch (dev ms, wall ms)", timed(d2d_only, K))

    def pipe():
        cs.run_pipelined(pinned)
    pipe()
    print("native pipeline (dev ms, wall ms)", timed(pipe, K), cs.pipe_stats)

    def seq():
        for p in pinned:
            cs.inp.buf[:p.buf.numel()].copy_(p.buf, non_blocking=True)
            cs.graph.replay()
            float(cs.out[dp.n].item())
    print("sequential     (dev ms, wall ms)", timed(seq, K))

    def nosync():
        for p in pinned:
            cs.inp.buf[:p.buf.numel()].copy_(p.buf, non_blocking=True)
            cs.graph.replay()
    print("h2d+replay nosync (dev ms, wall ms)", timed(nosync, K))

    lib = _lib.load()
    h = cs._pipe
    st = _lib.stream_ptr()
    dst = _lib.ptr(cs.inp.buf)
    def stage_only():
        for i, p in enumerate(pinned):
            _lib.check(lib.sg_pipe_stage(h, i & 1, p.buf.data_ptr(), p.h2d_bytes, dst, st))
    print("native stage only (dev ms, wall ms)", timed(stage_only, K))
    def stage_replay():
        for i, p in enumerate(pinned):
            _lib.check(lib.sg_pipe_stage(h, i & 1, p.buf.data_ptr(), p.h2d_bytes, dst, st))
            cs.graph.replay()
    print("native stage+replay nosync (dev ms, wall ms)", timed(stage_replay, K))
    print("current stream handle", st)


if __name__ == "__main__":
    main()
