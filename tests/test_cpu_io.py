"""File formats beside the hot path, pinned to fixtures
written by the unmodified reference (tests/golden/make_io_golden.py): the SPLG
binary CSR (graph.py:238-273) and the per-iteration metrics CSV
(metrics.py:100-198) -- byte-identical round trips."""

import os

import numpy as np

from helpers import GOLD


def test_splg_reader_and_writer_match_reference_bytes(tmp_path):
    import paper_2303_13775_b200 as sg
    z = np.load(os.path.join(GOLD, "io_metrics.npz"))
    g = sg.load_binary_csr(os.path.join(GOLD, "io_graph.splg"))
    assert g.num_vertices == 50 and g.num_edges == 300
    assert np.array_equal(g.row_offsets, z["offsets"])
    assert np.array_equal(g.col_indices, z["src"])
    assert np.allclose(g.features, z["feats"], rtol=1e-7)  # fp32 on our side
    # writing our float64 copy back reproduces the reference's bytes exactly
    g64 = sg.Graph(g.num_vertices, g.row_offsets, g.col_indices, None)
    out = tmp_path / "g.splg"
    sg.save_binary_csr(g64, out)
    ref = open(os.path.join(GOLD, "io_graph.splg"), "rb").read()
    mine = open(out, "rb").read()
    hdr = 4 + 4 + 24
    assert mine[:4] == ref[:4] and mine[8:hdr - 8] == ref[8:hdr - 8]      # magic, n, m
    assert mine[hdr:] == ref[hdr:hdr + 8 * (51 + 300)]                    # offsets + indices


def test_metrics_csv_matches_reference_bytes(tmp_path):
    import paper_2303_13775_b200 as sg
    z = np.load(os.path.join(GOLD, "io_metrics.npz"))
    recs = []
    for e in range(2):
        em = sg.EpochMetrics(epoch=e, mode="split", num_devices=3)
        for i in range(4):
            it = sg.IterationMetrics(iteration=i, mode="split", num_devices=3)
            for k in ("host_bytes", "peer_bytes", "redundant_edges"):
                setattr(it, k, int(z[f"{e}_{i}_{k}"]))
            for k in ("edge_skew", "local_edge_fraction", "sample_ms", "split_ms", "train_ms", "loss"):
                setattr(it, k, float(z[f"{e}_{i}_{k}"]))
            it.edges_per_device = z[f"{e}_{i}_edges_per_device"].astype(np.int64)
            em.iterations.append(it)
        recs.append(em)
    out = tmp_path / "m.csv"
    sg.emit_csv(recs, out)
    assert open(out).read() == open(os.path.join(GOLD, "io_metrics.csv")).read()
    header, rows = sg.read_csv(out)
    assert header[5:8] == ["edges_dev0", "edges_dev1", "edges_dev2"] and len(rows) == 10
