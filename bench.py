"""Benchmark: split-parallel GraphSAGE training step on an ogbn-products-shaped
synthetic power-law graph (BASELINE.json configs[1], "C2").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One process per GPU (torchrun for N>1): split parts g = N, rank r owns part r
(range partition, fully cached feature shard), NCCL all-to-all-v for the
push-to-owner / push-from-owner rounds and an NCCL all-reduce of gradients.
A step = split + layer-0 gather + 3-layer forward + loss + backward + gradient
reduction + SGD for one 1024-target mini-batch (samples are produced ahead by
the native sampler, as in the paper's methodology).
Metric: aggregated edges/s = sum_l |E^l| per sample / step time (engine.py:799-800).

--impl reference times the reference CPU algorithm (oracle/ NumPy port) on
this host, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Workloads (BASELINE.json configs, SURVEY §8 shapes). C2 is the headline.
CONFIGS = {
    "c2": dict(kind="graphsage", heads=1, n=2_449_029, m=61_859_140, feat=100, classes=47,
               train_frac=0.0803, p_local=0.92,
               desc="C2 GraphSAGE-3L mean, products-shape synthetic power-law (2.45M nodes / "
                    "61.9M edges, F=100, 47 classes)"),
    "c3": dict(kind="gat", heads=4, n=2_449_029, m=61_859_140, feat=100, classes=47,
               train_frac=0.0803, p_local=0.92,
               desc="C3 GAT-3L 4 heads x 16 (concat), products-shape synthetic power-law "
                    "(2.45M nodes / 61.9M edges, F=100, 47 classes)"),
    "c5": dict(kind="exchange", heads=1, n=0, m=0, feat=100, classes=0, train_frac=0.0, p_local=0.0,
               desc="C5 push-to-owner / push-from-owner exchange microbench: remote-partial rows per "
                    "peer swept 2^8..2^20, width 101 (push-to-owner, d_in+1) and 100 (push-from-owner) fp32"),
    "c4": dict(kind="graphsage", heads=1, n=111_059_956, m=1_615_685_872, feat=128, classes=172,
               train_frac=0.0109, p_local=0.95,
               desc="C4 GraphSAGE-3L mean, papers100M-shape synthetic power-law (111M nodes / "
                    "1.62B edges, F=128, 172 classes), whole feature table resident"),
}
CFG_NAME = "c2"
KIND, HEADS = "graphsage", 1
N_NODES = 2_449_029
N_EDGES = 61_859_140
FEAT = 100
CLASSES = 47
HIDDEN = 16
FANOUTS = [15, 10, 5]
BATCH = 1024
TRAIN_FRAC = 0.0803
P_LOCAL = 0.92
DESC = CONFIGS["c2"]["desc"]
LR = 0.1
GRAPH_SEED, FEAT_SEED, LABEL_SEED, TRAIN_SEED, RUN_SEED = 0, 1, 2, 3, 0


def _trace(what, x):
    """SG_BENCH_TRACE=1: checksums of intermediate state on stderr (determinism checks)."""
    if os.environ.get("SG_BENCH_TRACE") != "1":
        return
    if hasattr(x, "detach"):
        a = x.detach().float().cpu().numpy()
        bad = np.flatnonzero(~np.isfinite(a))
        x = (float(np.abs(a).sum()), int(a.view(np.uint32).astype(np.uint64).sum() % (1 << 32)), len(a),
             f"non-finite {len(bad)} at {bad[:6].tolist()}")
    print(f"[trace] {what}: {x}", file=sys.stderr, flush=True)


def select_config(name):
    global CFG_NAME, KIND, HEADS, N_NODES, N_EDGES, FEAT, CLASSES, TRAIN_FRAC, P_LOCAL, DESC
    c = CONFIGS[name]
    CFG_NAME, KIND, HEADS = name, c["kind"], c["heads"]
    N_NODES, N_EDGES, FEAT, CLASSES = c["n"], c["m"], c["feat"], c["classes"]
    TRAIN_FRAC, P_LOCAL, DESC = c["train_frac"], c["p_local"], c["desc"]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--batch", type=int, default=BATCH)
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no clocks/baseline)")
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    return ap.parse_args()


def build_workload(threads):
    import paper_2303_13775_b200 as sg
    t = time.time()
    graph = sg.generate_powerlaw(N_NODES, N_EDGES, blocks=64, p_local=P_LOCAL, gamma=2.1,
                                 seed=GRAPH_SEED, threads=threads)
    labels = sg.synthetic_labels(N_NODES, CLASSES, LABEL_SEED)
    perm = np.random.default_rng(TRAIN_SEED).permutation(N_NODES)
    train = np.sort(perm[: int(np.ceil(TRAIN_FRAC * N_NODES))])
    return graph, labels, train, time.time() - t


def make_samples(graph, train, k, batch, threads):
    import paper_2303_13775_b200 as sg
    sampler = sg.NativeSampler(graph, threads=threads)
    ss = np.random.SeedSequence([RUN_SEED, 0])
    batches = sg.epoch_batches(train, batch, np.random.default_rng(ss.spawn(1)[0]))
    out = []
    global PLAN
    PLAN = []
    for i in range(k):
        tg = batches[i % len(batches)]
        seed = int(np.random.default_rng(ss.spawn(1)[0]).integers(0, 2**63 - 1))
        out.append(sampler.sample(tg, FANOUTS, seed))
        PLAN.append((tg, seed))
    return out, len(batches)


PLAN = []  # (targets, seed) of every pre-sampled step, for the on-GPU sampling pipeline


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


def sage_fwd_bytes(E, R, w):
    """SURVEY §8(d) SpMM-forward algorithmic bytes (per-edge source-row model)."""
    return 4 * w * E + 4 * E + 4 * (R + 1) + 4 * (w + 1) * R


def sage_fused_fwd_bytes(E, R, w, dout):
    """Fused single-device layer (SpMM + update): the SpMM's per-edge source
    rows, edge and row indices, then per destination row the self row read,
    mean / self-row / count / output writes (the sums never leave the chip)."""
    return 4 * w * E + 4 * E + 4 * (R + 1) + 4 * w * R + 4 * (2 * w + 1 + dout) * R


def gat_agg_bytes(E, R, dh, H):
    """SURVEY §8(d) GAT forward scores+softmax+aggregation bytes, per head:
    E*20 (src/dst index, s_src, t_dst, e) + E*(12 + 4 dh) (e, index, alpha, z
    row) + R*(4 dh + 8) (num, m, den)."""
    return H * (20 * E + (12 + 4 * dh) * E + (4 * dh + 8) * R)


def gat_project_bytes(n0, n1, w, D, H):
    """GAT layer-1 projection (k_gat_project_mma), per launch: per V^0 row the
    gathered feature row (4w) and its row index (4), z (4D) and s (4H) written,
    grouped (4); per V^1 self row rank (4) and t (4H) written."""
    return n0 * (4 * w + 4 + 4 * D + 4 * H + 4) + n1 * (4 + 4 * H)


def cpu_baseline(graph, labels, samples, pm_assign, g, n_iter=2):
    """Reference algorithm (oracle NumPy port) on this host, 1 thread, on the
    first n_iter samples of the same workload: split + forward + backward +
    all-reduce/SGD, float64."""
    from threadpoolctl import threadpool_limits

    import paper_2303_13775_b200 as sg
    from oracle.coop_oracle import CoopRun, reduce_and_sgd
    from oracle.model_oracle import glorot_params
    from oracle.split_oracle import split_sample
    if KIND == "gat" and HEADS > 1:
        from oracle.multihead_oracle import multihead_run
        params = {k: np.asarray(v, dtype=np.float64) for k, v in
                  sg.init_params("gat", FEAT, HIDDEN, CLASSES, len(FANOUTS), seed=RUN_SEED,
                                 heads=HEADS).tensors().items()}
    else:
        params = glorot_params(KIND, FEAT, HIDDEN, CLASSES, len(FANOUTS), seed=RUN_SEED)
    edges = 0
    t_total = 0.0
    with threadpool_limits(limits=1):
        for smp in samples[:n_iter]:
            # compact the gids the sample touches (sorted, so gid order is kept)
            V = [np.asarray(v, dtype=np.int64) for v in smp.layer_vertices]
            uniq = np.unique(V[0])
            Vc = [np.searchsorted(uniq, v) for v in V]
            Ec = [(np.asarray(s, np.int64), np.asarray(d, np.int64)) for s, d in smp.layer_edges]
            X = sg.synthetic_features(0, FEAT, FEAT_SEED, row_ids=uniq).astype(np.float64)
            asn = pm_assign[uniq]
            lab = np.asarray(labels, dtype=np.int64)[uniq]
            t0 = time.perf_counter()
            splits, plan = split_sample(Vc, Ec, asn, g, None)
            if KIND == "gat" and HEADS > 1:  # per-head composition of the reference layer (g=1)
                _, gr, _ = multihead_run(Vc, Ec, params, X, lab, HEADS)
                grads = [gr]
            else:
                run = CoopRun(params, splits, plan, X, lab)
                _, grads = run.run()
            reduce_and_sgd(params, grads, LR, len(V[-1]))
            t_total += time.perf_counter() - t0
            edges += smp.total_edges
    return edges / t_total, t_total, n_iter, edges


def run_reference_arm(args, rank, world):
    import torch  # noqa: F401
    if rank != 0:
        return
    select_config(args.config)
    if KIND == "exchange":
        print(json.dumps({"impl": "reference", "unavailable": "the reference exchanges in-process with "
                          "NumPy copies (engine.py:121-156); there is no transport to microbenchmark"}))
        return
    threads = os.cpu_count() or 1
    graph, labels, train, _ = build_workload(threads)
    samples, _ = make_samples(graph, train, args.warmup + args.steps, args.batch, threads)
    g = args.gpus
    pm_assign = (np.arange(N_NODES, dtype=np.int64) * g) // N_NODES
    cpu_baseline(graph, labels, samples[: args.warmup], pm_assign, g, n_iter=args.warmup)
    rate, secs, n_it, edges = cpu_baseline(graph, labels, samples[args.warmup:], pm_assign, g,
                                           n_iter=args.steps)
    line = {
        "impl": "reference", "metric": "aggregated_edges_per_s", "value": rate, "unit": "edges/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / n_it, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C2 GraphSAGE-3L mean, products-shape synthetic (2.45M/61.9M, F=100), "
                               f"batch {args.batch}, fanout {FANOUTS}, g={g}", "model": "graphsage-3l-h16",
                   "global_batch": args.batch},
        "cpu_baseline": {"value": rate, "unit": "edges/s", "cores": 1, "kind": "port",
                         "sample": f"{n_it} {CFG_NAME.upper()} iterations (batch {args.batch}), oracle NumPy port of "
                                   "split_minibatch+SplitExecutor+allreduce_and_step, float64, 1 thread"},
        "e2e": {"value": rate, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_exchange_bench(args, rank, world, local):
    """C5: the split exchange's transport (NcclTransport: one all-to-all-v per
    round, engine.py:121-156 / PAPER.md:820) on uniform synthetic plans, rows
    per peer swept; bytes sent per GPU / device time (max over ranks) against
    NVLink 5 (900 GB/s per direction). At N = 1 there is no peer link: the
    line reports NCCL's self-copy through the same call, marked as such."""
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world,
                            init_method=None if "MASTER_ADDR" in os.environ else "tcp://127.0.0.1:29512")
    sweep = []
    for width in (101, 100):
        for lg in range(8, 21, 2):
            rows = 1 << lg
            if rows * width * 4 * world > 8 << 30:
                break
            send = torch.rand(rows * world, width, device=dev)
            recv = torch.empty_like(send)
            splits = [rows * width] * world
            for _ in range(args.warmup):
                dist.all_to_all_single(recv.view(-1), send.view(-1), splits, splits)
            dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.steps):
                dist.all_to_all_single(recv.view(-1), send.view(-1), splits, splits)
            e1.record()
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            # bytes each GPU sends to its peers (N = 1: the self-copy reads and writes its block)
            peer_bytes = rows * width * 4 * (world - 1) if world > 1 else 2 * rows * width * 4
            sweep.append({"rows_per_peer": rows, "width": width, "bytes_sent_per_gpu": peer_bytes,
                          "us": ms * 1e3, "GBps_per_gpu": peer_bytes / (ms * 1e-3) / 1e9})
            del send, recv
    best = max(sweep, key=lambda r: r["GBps_per_gpu"])
    if rank == 0:
        line = {"metric": "exchange_GBps_per_gpu", "value": best["GBps_per_gpu"], "unit": "GB/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": best["us"] / 1e3,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic",
                "config": {"workload": DESC, "config_id": "c5", "parallelism": f"split{world}",
                           "peer_link": "NVLink 5 / NVSwitch" if world > 1 else "none (N=1: NCCL self-copy)"},
                "roofline": {"bound": "nvlink" if world > 1 else "hbm",
                             "achieved": best["GBps_per_gpu"], "peak": 900.0 if world > 1 else 6551.7,
                             "unit": "GB/s", "frac": best["GBps_per_gpu"] / (900.0 if world > 1 else 6551.7),
                             "traffic": None},
                "sweep": sweep}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference_arm(args, rank, world)
    select_config(args.config)
    if KIND == "exchange":
        return run_exchange_bench(args, rank, world, local)

    import torch
    import torch.distributed as dist

    import paper_2303_13775_b200 as sg
    from paper_2303_13775_b200 import _lib
    from paper_2303_13775_b200.engine import SplitStep

    # SG_BENCH_HOST_STAGED=1: every rank on cuda:0, payloads staged through host
    # memory over gloo -- exercises the N > 1 code path on a single-GPU box
    # (the numbers are not NVLink numbers and are marked as such).
    staged = os.environ.get("SG_BENCH_HOST_STAGED") == "1" and world > 1
    if staged:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if staged:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def allreduce(t, op=None):
        op = dist.ReduceOp.SUM if op is None else op
        if not staged:
            dist.all_reduce(t, op=op)
            return
        c = t.cpu()
        dist.all_reduce(c, op=op)
        t.copy_(c)
    g = world
    threads = max(1, (os.cpu_count() or 1) // max(1, world))
    graph, labels, train, gen_s = build_workload(threads)
    pm = sg.range_partition(N_NODES, g)
    part_rows = pm.device_vertices(rank)
    feats = sg.FeatureStore.synthetic(N_NODES, FEAT, FEAT_SEED,
                                      row_ids=None if g == 1 else part_rows, device=dev,
                                      pad_rows=KIND == "graphsage")  # whole 128 B lines per row
    cache = sg.full_cache(pm)
    labels_dev = torch.from_numpy(labels).to(dev)
    n_steps = args.warmup + args.steps
    samples, iters_per_epoch = make_samples(graph, train, n_steps, args.batch, threads)
    params = sg.init_params(KIND, FEAT, HIDDEN, CLASSES, len(FANOUTS), seed=RUN_SEED, heads=HEADS)
    dp = sg.DeviceParams.from_host(params, dev)
    # N > 1: the peer-memory transport (IPC-mapped buffers, device flags; the
    # rank step is one CUDA graph) unless SG_TRANSPORT=nccl asks for the eager
    # NCCL all-to-all-v path.
    use_peer = g > 1 and os.environ.get("SG_TRANSPORT", "peer") == "peer"
    if g == 1:
        transport = sg.LocalTransport()
    elif use_peer:
        try:  # CUDA IPC between the ranks' GPUs; every rank must succeed
            transport = sg.PeerTransport(rank, world, device=dev)
            ok = 1
        except Exception as exc:  # noqa: BLE001 - reported, then the NCCL path runs
            print(f"[rank {rank}] peer transport unavailable ({exc}); using NCCL", file=sys.stderr)
            ok = 0
        flag = torch.tensor([ok], dtype=torch.int32, device=dev if not staged else "cpu")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 0:
            use_peer = False
            transport = sg.NcclTransport(rank, world, stage_on_host=staged)
    else:
        transport = sg.NcclTransport(rank, world, stage_on_host=staged)
    # device-resident inputs
    dev_samples = []
    for s in samples:
        V, es, ed = s.packed()
        dev_samples.append((torch.from_numpy(V).to(dev), torch.from_numpy(es).to(dev),
                            torch.from_numpy(ed).to(dev), s.sizes()))
    flush = torch.empty(256 * 2**20 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    exact = g > 1

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    edges = sum(samples[i].total_edges for i in range(args.warmup, n_steps))
    agg_ms, step_ms, roof_ms = [], [], []
    phases = {}
    clocks = ClockSampler(local)
    if g == 1 or use_peer:
        # ---- the whole (rank) step is one captured CUDA graph ----------------------
        from paper_2303_13775_b200.engine import CapturedStep, RankCapturedStep, capacities_for
        cap_nV, cap_nE = capacities_for(samples)

        def make_step(scale, record_events=False):
            if g == 1:
                return CapturedStep(dp, pm, cache, feats, labels_dev, cap_nV, cap_nE, scale, dev,
                                    record_events=record_events)
            return RankCapturedStep(dp, pm, cache, feats, labels_dev, cap_nV, cap_nE, scale, rank, transport,
                                    dev, record_events=record_events)
        cs = make_step(LR / args.batch, record_events="agg")
        cs.capture(samples[0])                     # eager warm-up step 0 + capture
        _trace("params after capture", dp.flat)
        agg_in_graph = True
        for i in range(1, args.warmup):
            cs.run(samples[i])
        barrier()
        l0 = _lib.launch_count()
        with clocks:
            t_wall = time.perf_counter()
            for i in range(args.warmup, n_steps):
                flush.zero_()
                cs.inp.load(samples[i])            # H2D outside the device-resident timing
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                cs.replay()
                e1.record()
                e1.synchronize()
                step_ms.append(e0.elapsed_time(e1))
                ev = cs.step.events
                try:
                    agg_ms.append(ev["agg1_start"][0].elapsed_time(ev["agg1_end"][0]))
                    if "roof1_start" in ev:
                        roof_ms.append(ev["roof1_start"][0].elapsed_time(ev["roof1_end"][0]))
                except Exception:
                    agg_in_graph = False
            barrier()
            t_wall = time.perf_counter() - t_wall
        _trace("params after timed", dp.flat)
        # diagnostic (untimed): a second capture with an event around every phase
        diag = make_step(0.0, record_events="all")
        diag.capture(samples[0])
        nd = min(5, args.steps)
        for i in range(args.warmup, args.warmup + nd):
            flush.zero_()
            diag.run(samples[i])
            torch.cuda.synchronize()
            for k, v in diag.step.phase_ms().items():
                phases[k] = phases.get(k, 0.0) + v / nd
        # graph replays launch the captured kernels: count them from one eager step
        # (which also times the layer-1 SpMM with events if the in-graph
        # event nodes were not readable)
        per_step_launches = _lib.launch_count()
        cs.inp.load(samples[n_steps - 1])
        cs._body()
        torch.cuda.synchronize()
        per_step_launches = _lib.launch_count() - per_step_launches
        if not agg_ms:
            ev = cs.step.events
            agg_ms.append(ev["agg1_start"][0].elapsed_time(ev["agg1_end"][0]))
        launches = per_step_launches * args.steps
        my_ms = sum(step_ms)
        # ---- end to end: host sample -> pinned -> H2D -> graph -> D2H loss ----------
        barrier()
        _trace("params before e2e", dp.flat)
        losses = []
        h2d = 0
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        # the user-facing captured step (no timing-event nodes in the graph),
        # fed from the sampler's output in pinned host memory (packed untimed)
        del diag
        ce = make_step(LR / args.batch)
        ce.capture(samples[0])
        # compact staging (run starts instead of per-edge destinations) unless SG_PIPE_COMPACT=0
        pinned = ce.prepare_pinned(samples[args.warmup:n_steps], compact=os.environ.get("SG_PIPE_COMPACT", "1") != "0")
        ce.run_pipelined(pinned[:2])  # allocate the staging buffers (untimed)
        barrier()
        e0.record()
        t_e2e = time.perf_counter()
        losses, h2d, d2h = ce.run_pipelined(pinned)
        t_e2e = time.perf_counter() - t_e2e
        _trace("e2e losses", losses)
        e1.record()
        barrier()
        e2e_ms = e0.elapsed_time(e1)
        # ---- end to end from host TARGETS: the GPU sampler inside the graph ------------
        e2e_s = None
        pipe_stats = getattr(ce, "pipe_stats", None)
        if g == 1 and all(len(t) == args.batch for t, _ in PLAN):
            from paper_2303_13775_b200.engine import SampledCapturedStep
            del ce
            gs = sg.GpuSampler(graph, device=dev)
            cz = SampledCapturedStep(gs, FANOUTS, args.batch, dp, pm, cache, feats, labels_dev, cap_nV, cap_nE,
                                     LR / args.batch, dev)
            cz.capture_targets(*PLAN[0])
            pz = cz.pin_targets(PLAN[args.warmup:n_steps])
            cz.run_pipelined_targets(pz[:2])
            barrier()
            z0, z1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            z0.record()
            zl, zh2d, zd2h = cz.run_pipelined_targets(pz)
            z1.record()
            barrier()
            cz.check()
            zms = z0.elapsed_time(z1)
            e2e_s = {"value": edges / (zms / 1e3), "unit": "edges/s", "h2d_bytes_per_step": zh2d // args.steps,
                     "d2h_bytes_per_step": zd2h // args.steps, "ms_per_step": zms / args.steps,
                     "what": "host targets + seed -> GPU sampler (bit-identical to the native sampler) + split + "
                             "train + SGD in one CUDA graph -> loss to host; includes sampling, which `value` "
                             "and the CPU reference exclude"}
    else:
        t_e2e, ce, e2e_s, pipe_stats = None, None, None, None
        # ---- one rank per GPU: eager step, NCCL all-to-all-v + all-reduce ---------
        def one_step(i, record_events=False):
            V, es, ed, (nV, nE) = dev_samples[i]
            ds = sg.DeviceSplit(V, es, ed, nV, nE, pm, cache, True, dev)
            step = SplitStep(dp, ds, feats, labels_dev, devices=[rank], transport=transport,
                             exact=True, record_events=record_events)
            step.run()
            gbuf = step.grads[rank]
            allreduce(gbuf)
            ptrs_h = np.asarray([gbuf.data_ptr()], dtype=np.int64)
            _lib.call("sg_sum_sgd", _lib.ptr(dp.flat), None, _lib.ptr(ptrs_h), 1, dp.n,
                      LR / len(samples[i].targets), _lib.stream_ptr())
            return step, gbuf

        for i in range(args.warmup):
            one_step(i)
        barrier()
        keep = []
        l0 = _lib.launch_count()
        with clocks:
            barrier()
            t_wall = time.perf_counter()
            for i in range(args.warmup, n_steps):
                flush.zero_()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                step, gbuf = one_step(i, record_events=True)
                e1.record()
                keep.append((e0, e1, step))
            barrier()
            t_wall = time.perf_counter() - t_wall
        launches = _lib.launch_count() - l0
        for e0, e1, step in keep:
            step_ms.append(e0.elapsed_time(e1))
            agg_ms.append(step.events["agg1_start"][0].elapsed_time(step.events["agg1_end"][0]))
        my_ms = sum(step_ms)
        barrier()
        losses, h2d = [], 0
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(args.warmup, n_steps):
            smp = samples[i]
            ds = sg.DeviceSplit.from_sample(smp, pm, cache, dev)
            step = SplitStep(dp, ds, feats, labels_dev, devices=[rank], transport=transport, exact=True)
            step.run()
            gbuf = step.grads[rank]
            allreduce(gbuf)
            ptrs_h = np.asarray([gbuf.data_ptr()], dtype=np.int64)
            _lib.call("sg_sum_sgd", _lib.ptr(dp.flat), None, _lib.ptr(ptrs_h), 1, dp.n,
                      LR / len(smp.targets), _lib.stream_ptr())
            losses.append(float(gbuf[dp.n].item()) / len(smp.targets))
            V, es, ed = smp.packed()
            h2d += V.nbytes + es.nbytes + ed.nbytes
        e1.record()
        barrier()
        e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([my_ms, e2e_ms], device=dev)
        allreduce(t, op=dist.ReduceOp.MAX)
        my_ms, e2e_ms = float(t[0].item()), float(t[1].item())
    value = edges / (my_ms / 1e3)
    e2e = edges / (e2e_ms / 1e3)

    if rank == 0:
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
            peak_src = "measured"
        except Exception:
            peak_src = "fallback"
        hbm = float(peaks.get("hbm_gbs", 6650.0))
        s0 = samples[args.warmup]
        nV, nE = s0.sizes()
        # dominant kernel: layer-1 SpMM (agg) of this rank's split
        E1 = np.mean([samples[i].sizes()[1][0] for i in range(args.warmup, n_steps)]) / g
        R1 = np.mean([samples[i].sizes()[0][1] for i in range(args.warmup, n_steps)]) / g
        if KIND == "gat":
            alg = gat_agg_bytes(E1, R1, HIDDEN, HEADS)
        else:
            alg = sage_fused_fwd_bytes(E1, R1, FEAT, HIDDEN) if g == 1 else sage_fwd_bytes(E1, R1, FEAT)
        agg_avg = float(np.mean(agg_ms))
        achieved = alg / (agg_avg / 1e3) / 1e9
        def _traffic(kind):  # ncu DRAM bytes per launch of the roofline kernel, if captured
            tpath = os.path.join(ROOT, "profiles", f"{kind}_traffic_{CFG_NAME}.json")
            try:
                return json.load(open(tpath)).get("bytes_per_launch")
            except Exception:
                return None
        traffic = _traffic("agg1")
        roof_gat = None
        if KIND == "gat" and roof_ms:
            # C3's dominant forward kernel is the layer-1 projection, not the aggregation
            n0 = np.mean([samples[i].sizes()[0][0] for i in range(args.warmup, n_steps)]) / g
            pb = gat_project_bytes(n0, R1, FEAT, HIDDEN * HEADS, HEADS)
            pms = float(np.mean(roof_ms))
            roof_gat = {"bound": "hbm", "kernel": f"k_gat_project_tc layer 1 (tcgen05 kind::tf32 3xTF32, TMEM "
                                                  f"accumulator, F={FEAT} -> {HEADS}x{HIDDEN})",
                        "achieved": pb / (pms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                        "frac": pb / (pms / 1e3) / 1e9 / hbm, "traffic": _traffic("roof1"), "peak_source": peak_src,
                        "alg_bytes_per_launch": pb, "avg_launch_ms": pms, "share_of_step": pms / (my_ms / args.steps),
                        "tensor_flops_per_launch": 3 * 2 * n0 * FEAT * HIDDEN * HEADS}
        base = None
        if not args.no_cpu_baseline and not args.profile:
            rate, secs, n_it, _ = cpu_baseline(graph, labels, samples[args.warmup:], pm.assignment, g, 2)
            base = {"value": rate, "unit": "edges/s", "cores": 1, "kind": "port",
                    "sample": f"{n_it} {CFG_NAME.upper()} iterations (batch {args.batch}) through the oracle NumPy port of "
                              f"split_minibatch+SplitExecutor+allreduce_and_step, float64, 1 thread, {secs:.1f}s"}
        line = {
            "metric": "aggregated_edges_per_s", "value": value, "unit": "edges/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": my_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": f"{DESC}, batch {args.batch}, fanout {FANOUTS}, hidden 16, split parts g={g}, "
                                   "range partition, full feature cache",
                       "config_id": CFG_NAME,
                       "model": f"{KIND}-3l-h16" + (f"x{HEADS}" if HEADS > 1 else ""),
                       "global_batch": args.batch, "seq_len": None,
                       "parallelism": f"split{g}" + (" host-staged (gloo, one GPU): not an NVLink number"
                                                      if staged else ""),
                       "transport": "local" if g == 1 else ("peer (CUDA IPC, graph-captured rank step)"
                                                            if use_peer else "nccl all-to-all-v (eager)"),
                       "l2": "flushed between timed steps (256 MB write, "
                                                          "outside the per-step events)",
                       "epoch_iterations": iters_per_epoch,
                       "epoch_time_s": iters_per_epoch * my_ms / args.steps / 1e3,
                       "edges_per_step": edges / args.steps, "graph_gen_s": round(gen_s, 1),
                       "sample_sizes_first": {"V": nV, "E": nE}},
            "roofline_agg" if roof_gat else "roofline": {"bound": "hbm", "kernel": (f"k_gat_agg layer 1 (online softmax, {HEADS} heads)" if KIND == "gat"
                                                    else f"k_sage_agg_mean + k_sage_linear layer 1 (F={FEAT})" if g == 1
                                                    else f"k_sage_agg layer 1 (F={FEAT})"),
                         "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                         "traffic": traffic, "peak_source": peak_src,
                         "alg_bytes_per_launch": alg, "avg_launch_ms": agg_avg,
                         "share_of_step": agg_avg / (my_ms / args.steps)},
            **({"roofline": roof_gat} if roof_gat else {}),
            "e2e": {"value": e2e, "unit": "edges/s", "h2d_bytes_per_step": h2d // args.steps,
                    "d2h_bytes_per_step": 4, "ms_per_step": e2e_ms / args.steps,
                    "wall_ms_per_step": (t_e2e * 1e3 / args.steps) if g == 1 else None,
                    "host_us_per_step": pipe_stats if g == 1 else None},
            "e2e_with_sampling": e2e_s,
            "gpu_launches": int(launches),
            "phases_ms": {k: round(v, 5) for k, v in sorted(phases.items(), key=lambda x: -x[1])},
            "clocks": clocks.summary(),
            "wall_s_timed": t_wall,
            "loss_last": losses[-1] if losses else None,
        }
        if base is not None:
            line["cpu_baseline"] = base
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
