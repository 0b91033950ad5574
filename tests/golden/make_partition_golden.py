"""Pin the GPU partitioner's QUALITY to the reference's (build container only:
imports the unmodified reference from /root/reference/pkg/src).

Runs reference `partition_graph` (partition.py:298-349: multilevel heavy-edge
coarsening, greedy region growing, boundary refinement) on the graphs the
quality tests regenerate with NumPy, and records its cut sizes:

* the reference's own planted-partition fixture (test_partition.py:62-69:
  generate_planted_partition(4000, 4, 0.1, 0.001, 2, seed=3), g = 4, eps 0.05);
* the same planted graph with its vertex ids permuted (contiguous-id starting
  maps get no help from the id layout);
* an 8-block planted graph with shuffled block membership (tests/
  test_gpu_partition.py:_planted) at g = 2, 4, 8;
* a C1-shape-family block-planted power-law graph (oracle/workload.py
  generate_powerlaw, 50K nodes / 500K edges) at g = 2, 4, 8.

Writes tests/golden/partition_quality.json. Usage:
    python tests/golden/make_partition_golden.py
"""

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
sys.path.insert(0, os.path.join(HERE, ".."))
sys.path.insert(0, "/root/reference/pkg/src")

from splitgnn.graph import from_edges, generate_planted_partition  # noqa: E402
from splitgnn.partition import cut_size, partition_graph  # noqa: E402

from partition_graphs import permuted, planted_blocks, powerlaw_edges, reference_planted_edges  # noqa: E402


def main():
    out = {}

    g0 = generate_planted_partition(4000, 4, 0.1, 0.001, 2, seed=3)
    s0, d0 = g0.edge_arrays()
    s1, d1 = reference_planted_edges(4000, 4, 0.1, 0.001, seed=3)
    order0 = np.lexsort((s0, d0))
    order1 = np.lexsort((s1, d1))
    assert np.array_equal(s0[order0], s1[order1]) and np.array_equal(d0[order0], d1[order1]), \
        "restated generator differs from the reference's"
    cases = [("ref_planted", 4000, s1, d1, [4])]
    ps, pd = permuted(4000, s1, d1, seed=11)
    cases.append(("ref_planted_permuted", 4000, ps, pd, [4]))
    s2, d2 = planted_blocks()
    cases.append(("planted8_shuffled", 20000, s2, d2, [2, 4, 8]))
    s3, d3 = powerlaw_edges()
    cases.append(("powerlaw50k", 50000, s3, d3, [2, 4, 8]))
    for name, n, s, d, gs in cases:
        gr = from_edges(n, s, d)
        rec = {"n": n, "m": int(len(s)), "edge_checksum": int((s * 1000003 + d).sum() % (1 << 61)), "cut": {}}
        for g in gs:
            t = time.time()
            pm = partition_graph(gr, g, 0.05, seed=5)
            rec["cut"][str(g)] = int(cut_size(gr, pm))
            print(name, g, rec["cut"][str(g)], f"of {len(s)} ({time.time() - t:.1f}s)", flush=True)
        out[name] = rec
    with open(os.path.join(HERE, "partition_quality.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
