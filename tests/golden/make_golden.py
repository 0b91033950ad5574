"""Generate golden vectors by running the REAL reference (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports `splitgnn` from /root/reference/pkg/src (read-only, never copied)
and writes small .npz fixtures next to this file. The fixtures pin both the
oracle restatement (oracle/) and, on the GPU box, the CUDA path.

Feature matrices are rounded to float32 before the reference runs, so the
float64 reference and the fp32 GPU path see bit-identical inputs.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from golden_io import pack_dict, pack_sample, pack_splits  # noqa: E402

from splitgnn.engine import PhaseRunner, SplitExecutor, allreduce_and_step  # noqa: E402
from splitgnn.graph import community_labels, from_edges, generate_planted_partition  # noqa: E402
from splitgnn.metrics import IterationMetrics  # noqa: E402
from splitgnn.models import init_params, run_reference  # noqa: E402
from splitgnn.partition import PartitionMap, build_cache, partition_graph  # noqa: E402
from splitgnn.sampling import epoch_batches, sample_minibatch  # noqa: E402
from splitgnn.scheduler import split_cost, split_minibatch  # noqa: E402


def f32(graph):
    return graph.with_features(graph.features.astype(np.float32).astype(np.float64))


def split_to_dicts(splits):
    out = []
    for s in splits:
        out.append(dict(owned_gids=s.owned_gids, owned_pos=s.owned_pos, ref_gids=s.ref_gids,
                        ref_owner=s.ref_owner, edges_src=s.edges_src, edges_dst=s.edges_dst,
                        self_rows=s.self_rows, load_gids=s.load_gids))
    return out


def plan_to_dict(plan):
    return {k: (e.gids, e.holder_idx, e.owner_idx) for k, e in plan.entries.items()}


def save(name, out):
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path)} B)")


def pack_cache(out, cache):
    if cache is None:
        out["cache_ndev"] = np.int64(-1)
        return
    out["cache_ndev"] = np.int64(len(cache.cached))
    for d, ids in enumerate(cache.cached):
        out[f"cache_{d}"] = np.asarray(ids, dtype=np.int64)


def pack_params(out, params, prefix="P"):
    pack_dict(out, {k: v.copy() for k, v in params.tensors().items()}, prefix)


def split_case(out, sample, pm, cache):
    splits, plan = split_minibatch(sample, pm, cache)
    pack_sample(out, sample.layer_vertices, sample.layer_edges)
    out["assignment"] = pm.assignment.copy()
    out["g"] = np.int64(pm.num_devices)
    pack_cache(out, cache)
    pack_splits(out, split_to_dicts(splits), plan_to_dict(plan))
    rep = split_cost(sample, pm, pm.num_devices)
    out["cost_per_layer"] = np.asarray(rep.cost_per_layer, dtype=np.int64)
    out["edges_per_device"] = np.asarray(rep.edges_per_device, dtype=np.int64)
    out["local_edge_fraction"] = np.float64(rep.local_edge_fraction)
    out["edge_skew"] = np.float64(rep.edge_skew)
    out["pair_count"] = np.asarray([plan.pair_count(l) for l in range(1, sample.num_layers + 1)],
                                   dtype=np.int64)
    return splits, plan


def executor_case(out, kind, graph, pm, cache, sample, labels, params):
    """Reference split executor + single-device oracle on one sample."""
    splits, plan = split_case(out, sample, pm, cache)
    out["features"] = graph.features.astype(np.float32)
    out["labels"] = np.asarray(labels, dtype=np.int64)
    out["kind"] = np.array(kind)
    pack_params(out, params)
    loss_ref, grads_ref = run_reference(sample, params, graph.features, labels)
    rec = IterationMetrics(iteration=0, mode="split", num_devices=pm.num_devices)
    runner = PhaseRunner(pm.num_devices, 1)
    ex = SplitExecutor(params, splits, plan, graph.features, labels, runner, rec)
    loss_split, per_dev = ex.run()
    runner.close()
    out["loss_ref"] = np.float64(loss_ref)
    out["loss_split"] = np.float64(loss_split)
    out["peer_bytes"] = np.int64(rec.peer_bytes)
    pack_dict(out, grads_ref, "Gref")
    for d, gd in enumerate(per_dev):
        pack_dict(out, gd, f"G{d}")
    for d, st in enumerate(ex.states):
        for l in range(params.num_layers + 1):
            out[f"h_{d}_{l}"] = st.h[l]
        if kind == "gat":
            for l in range(1, params.num_layers + 1):
                out[f"alpha_{d}_{l}"] = st.layer[l]["alpha"]


def main():
    # A. splitter cases (test_scheduler.py:15-21 setup, with a cache)
    for seed in range(6):
        rng = np.random.default_rng(seed)
        g = generate_planted_partition(80, 4, 0.15, 0.03, 4, seed=seed)
        pm = PartitionMap(rng.integers(0, 4, 80), 4, 1.0)
        targets = rng.choice(80, size=10, replace=False)
        sample = sample_minibatch(g, targets, [3, 3], rng)
        cache = build_cache(g, pm, 0.2) if seed % 2 == 0 else None
        out = {}
        split_case(out, sample, pm, cache)
        save(f"split_random_{seed}", out)

    # B. executor cases (test_engine.py:21-41 setup)
    for kind in ("graphsage", "gat"):
        for seed in range(4):
            rng = np.random.default_rng(seed)
            g = f32(generate_planted_partition(60, 3, 0.2, 0.05, 5, seed=seed))
            pm = PartitionMap(rng.integers(0, 3, 60), 3, 1.0)
            targets = rng.choice(60, size=8, replace=False)
            sample = sample_minibatch(g, targets, [3, 3], rng)
            labels = rng.integers(0, 3, 60)
            params = init_params(kind, 5, 4, 3, 2, seed=seed + 50)
            out = {}
            executor_case(out, kind, g, pm, None, sample, labels, params)
            save(f"exec_{kind}_{seed}", out)

    # C. edge cases
    g = f32(from_edges(2, [0], [1], np.random.default_rng(3).random((2, 4))))
    pm = PartitionMap(np.array([0, 1]), 2, 1.0)
    sample = sample_minibatch(g, [1], [1], np.random.default_rng(0))
    out = {}
    executor_case(out, "graphsage", g, pm, None, sample, np.array([0, 1]),
                  init_params("graphsage", 4, 3, 2, 1, seed=5))
    save("edge_single_cross", out)

    g = f32(generate_planted_partition(20, 2, 0.4, 0.1, 2, seed=0))
    pm = PartitionMap(np.zeros(20, dtype=np.int64), 3, 2.0)
    sample = sample_minibatch(g, [1, 5], [2, 2], np.random.default_rng(1))
    out = {}
    executor_case(out, "gat", g, pm, None, sample, np.arange(20) % 2,
                  init_params("gat", 2, 4, 2, 2, seed=6))
    save("edge_all_on_one", out)

    rng = np.random.default_rng(51)
    g = f32(generate_planted_partition(60, 3, 0.2, 0.05, 5, seed=51))
    targets = rng.choice(60, size=8, replace=False)
    sample = sample_minibatch(g, targets, [3, 3], rng)
    labels = rng.integers(0, 3, 60)
    asn = np.zeros(60, dtype=np.int64)
    asn[::2] = 1
    asn[1::4] = 2
    pm = PartitionMap(asn, 4, 4.0)
    for kind in ("graphsage", "gat"):
        out = {}
        executor_case(out, kind, g, pm, None, sample, labels, init_params(kind, 5, 4, 3, 2, seed=52))
        save(f"edge_idle_device_{kind}", out)

    # D. 3-layer acceptance workload (test_acceptance.py:49-61), partitioned + cached
    graph = f32(generate_planted_partition(2000, 4, 0.02, 0.001, 16, seed=7))
    pm = partition_graph(graph, 4, 0.05, seed=7)
    cache = build_cache(graph, pm, 0.25)
    labels = community_labels(2000, 4)
    for kind in ("graphsage", "gat"):
        rng = np.random.default_rng([7, 0, 0])
        targets = epoch_batches(np.arange(2000), 256, np.random.default_rng([7, 0]))[0]
        sample = sample_minibatch(graph, targets, [5, 5, 5], rng)
        params = init_params(kind, 16, 16, 4, 3, seed=7)
        out = {}
        executor_case(out, kind, graph, pm, cache, sample, labels, params)
        save(f"workload3_{kind}", out)

    # E. loss curves over 50 split steps (engine.py:729-826 seed protocol)
    graph = f32(generate_planted_partition(600, 4, 0.03, 0.003, 8, seed=11))
    pm = partition_graph(graph, 3, 0.05, seed=11)
    cache = build_cache(graph, pm, 0.3)
    labels = community_labels(600, 4)
    for kind in ("graphsage", "gat"):
        params = init_params(kind, 8, 16, 4, 2, seed=12)
        out = {"features": graph.features.astype(np.float32), "labels": labels,
               "assignment": pm.assignment.copy(), "g": np.int64(3), "kind": np.array(kind),
               "lr": np.float64(0.1)}
        pack_cache(out, cache)
        pack_params(out, params, "P0")
        losses, nsteps, epoch = [], 0, 0
        runner = PhaseRunner(3, 1)
        while nsteps < 50:
            ss = np.random.SeedSequence([12, epoch])
            batches = epoch_batches(np.arange(600), 64, np.random.default_rng(ss.spawn(1)[0]))
            for targets in batches:
                if nsteps >= 50:
                    break
                brng = np.random.default_rng(ss.spawn(1)[0])
                sample = sample_minibatch(graph, targets, [4, 4], brng)
                sub = {}
                pack_sample(sub, sample.layer_vertices, sample.layer_edges)
                for k, v in sub.items():
                    out[f"it{nsteps}_{k}"] = v
                splits, plan = split_minibatch(sample, pm, cache)
                loss_sum, per_dev = SplitExecutor(params, splits, plan, graph.features, labels,
                                                  runner).run()
                allreduce_and_step(params, per_dev, 0.1, len(targets))
                losses.append(loss_sum / len(targets))
                nsteps += 1
            epoch += 1
        runner.close()
        out["steps"] = np.int64(nsteps)
        out["losses"] = np.asarray(losses)
        pack_params(out, params, "Pfinal")
        save(f"losscurve_{kind}", out)


if __name__ == "__main__":
    main()
