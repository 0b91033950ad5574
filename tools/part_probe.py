"""Partitioner quality probe: cut of partition_graph on the quality graphs under
SG_PART_TWO_HOP / SG_PART_HOST_REFINE variants, vs the reference's cuts
(tests/golden/partition_quality.json). Run on a GPU box:
    python tools/part_probe.py"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

if len(sys.argv) > 1 and sys.argv[1] == "--one":
    sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
    import time
    import paper_2303_13775_b200 as sg
    from test_gpu_partition import _quality_graph
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "partition_quality.json")))
    for name in sys.argv[2:]:
        n, s, d = _quality_graph(name)
        graph = sg.from_edges(n, s, d)
        for g, ref in gold[name]["cut"].items():
            t = time.time()
            pm = sg.partition_graph(graph, int(g), 0.05, seed=5)
            cut = sg.cut_size(graph, pm)
            print(f"{name} g={g}: cut {cut} ref {ref} ({cut / ref:.3f}x) {time.time() - t:.2f}s", flush=True)
    sys.exit(0)

for two_hop in ("1", "0"):
    for host in (str(1 << 18), "0"):
        env = dict(os.environ, SG_PART_TWO_HOP=two_hop, SG_PART_HOST_REFINE=host, SG_PART_TRACE="1")
        print(f"== two_hop={two_hop} host_refine_max={host}", flush=True)
        subprocess.run([sys.executable, __file__, "--one", "powerlaw50k", "planted8_shuffled"], env=env)
