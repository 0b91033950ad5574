"""Determinism probe: replay ONE sample from the SAME parameters several times
and compare loss + updated parameters bitwise (eager SplitStep and the
captured graph). Usage: python tools/det_probe.py [c2|c3] [reps]."""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    bench.select_config(cfg)
    import paper_2303_13775_b200 as sg
    from paper_2303_13775_b200.engine import CapturedStep, capacities_for

    dev = torch.device("cuda", 0)
    threads = os.cpu_count() or 1
    graph, labels, train, _ = bench.build_workload(threads)
    pm = sg.range_partition(bench.N_NODES, 1)
    feats = sg.FeatureStore.synthetic(bench.N_NODES, bench.FEAT, bench.FEAT_SEED, device=dev,
                                      pad_rows=bench.KIND == "graphsage")
    cache = sg.full_cache(pm)
    labels_dev = torch.from_numpy(labels).to(dev)
    samples, _ = bench.make_samples(graph, train, 14, bench.BATCH, threads)
    rec = os.environ.get("PROBE_EVENTS") or False
    params = sg.init_params(bench.KIND, bench.FEAT, bench.HIDDEN, bench.CLASSES, len(bench.FANOUTS),
                            seed=bench.RUN_SEED, heads=bench.HEADS)
    dp = sg.DeviceParams.from_host(params, dev)
    p0 = dp.flat.clone()
    cap_nV, cap_nE = capacities_for(samples)
    cs = CapturedStep(dp, pm, cache, feats, labels_dev, cap_nV, cap_nE, bench.LR / bench.BATCH, dev,
                      record_events=rec)
    cs.capture(samples[0])
    bad = 0
    for mode in ("graph", "graph-no-flush"):
        ref = None
        for r in range(reps):
            dp.flat.copy_(p0)
            if mode == "graph":
                torch.empty(64 * 2**20, dtype=torch.float32, device=dev).zero_()
            cs.run(samples[1])
            torch.cuda.synchronize()
            out = (dp.flat.detach().cpu().numpy().copy(), cs.out.detach().cpu().numpy().copy())
            if ref is None:
                ref = out
                print(f"{mode}: loss {float(out[1][dp.n]):.6f}, non-finite params {int((~np.isfinite(out[0])).sum())}")
                continue
            dpar = np.flatnonzero(out[0] != ref[0])
            dout = np.flatnonzero(out[1] != ref[1])
            if len(dpar) or len(dout):
                bad += 1
                print(f"{mode} rep {r}: {len(dpar)} params differ (first {dpar[:8]}), "
                      f"{len(dout)} out words differ; max |dp| {np.abs(out[0] - ref[0]).max():.3e}")
        print(f"{mode}: {reps} reps done")
    print("DETERMINISTIC" if bad == 0 else f"NONDETERMINISTIC ({bad} mismatching reps)")
    # a training sequence over different samples: first step with non-finite parameters
    dp.flat.copy_(p0)
    for i, smp in enumerate(samples[2:]):
        cs.run(smp)
        loss = float(cs.out.reshape(-1)[dp.n])
        torch.cuda.synchronize()
        f = dp.flat.detach().cpu().numpy()
        badi = np.flatnonzero(~np.isfinite(f))
        if len(badi) or not np.isfinite(loss):
            names = sorted({dp.names[int(np.searchsorted(dp.offsets, j, side="right")) - 1]
                            if j < dp.n else "<extra>" for j in badi})
            print(f"step {i}: loss {loss}, {len(badi)} non-finite params in {names}")
            break
        print(f"step {i}: loss {loss:.6f} finite")


if __name__ == "__main__":
    main()
