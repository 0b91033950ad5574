"""Golden fixtures for the reference's file formats, written by the UNMODIFIED
reference (run in the build container only; /root/reference does not travel):
  io_graph.splg   graph.save_binary_csr of a small random graph with features
  io_metrics.csv  metrics.emit_csv of two synthetic epochs (3 devices)
  io_metrics.npz  the records' field values, to rebuild them on our side
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_io_golden.py
"""
import os

import numpy as np
from splitgnn.graph import Graph, save_binary_csr
from splitgnn.metrics import EpochMetrics, IterationMetrics, emit_csv

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    rng = np.random.default_rng(0)
    n, m = 50, 300
    dst = np.sort(rng.integers(0, n, m))
    src = rng.integers(0, n, m)
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.add.at(offsets, dst + 1, 1)
    offsets = np.cumsum(offsets)
    feats = rng.random((n, 3))
    save_binary_csr(Graph(n, offsets, src.astype(np.int64), feats), os.path.join(HERE, "io_graph.splg"))
    recs, flat = [], {}
    for e in range(2):
        em = EpochMetrics(epoch=e, mode="split", num_devices=3)
        for i in range(4):
            it = IterationMetrics(iteration=i, mode="split", num_devices=3)
            it.host_bytes = int(rng.integers(0, 10**6))
            it.peer_bytes = int(rng.integers(0, 10**6))
            it.edges_per_device = rng.integers(0, 1000, 3).astype(np.int64)
            it.redundant_edges = int(rng.integers(0, 50))
            it.edge_skew = float(rng.random())
            it.local_edge_fraction = float(rng.random())
            it.sample_ms, it.split_ms, it.train_ms = (float(x) for x in rng.random(3) * 10)
            it.loss = float(rng.random() * 4)
            em.iterations.append(it)
            for k in ("host_bytes", "peer_bytes", "redundant_edges", "edge_skew", "local_edge_fraction",
                      "sample_ms", "split_ms", "train_ms", "loss"):
                flat[f"{e}_{i}_{k}"] = getattr(it, k)
            flat[f"{e}_{i}_edges_per_device"] = it.edges_per_device
        recs.append(em)
    emit_csv(recs, os.path.join(HERE, "io_metrics.csv"))
    np.savez(os.path.join(HERE, "io_metrics.npz"), offsets=offsets, src=src, feats=feats, **flat)


if __name__ == "__main__":
    main()
