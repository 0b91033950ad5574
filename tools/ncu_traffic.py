"""Write profiles/agg1_traffic_<cfg>.json from an ncu --set full report: DRAM bytes
(read + write) of the layer-1 aggregation launch (the largest launch of the
named kernel), which bench.py reports as roofline.traffic.

  python tools/ncu_traffic.py <report.ncu-rep> <kernel-substring> [out.json]
"""
import csv
import io
import json
import subprocess
import sys

rep, kname = sys.argv[1], sys.argv[2]
out = sys.argv[3] if len(sys.argv) > 3 else "profiles/agg1_traffic_c2.json"
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, units = rows[0], rows[1]
best = None
for r in rows[2:]:
    d = dict(zip(hdr, r))
    if kname not in d.get("Kernel Name", ""):
        continue
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = float(d["dram__bytes_read.sum"].replace(",", "")) * scale[units[hdr.index("dram__bytes_read.sum")]]
    wr = float(d["dram__bytes_write.sum"].replace(",", "")) * scale[units[hdr.index("dram__bytes_write.sum")]]
    if best is None or rd + wr > best[0]:
        best = (rd + wr, rd, wr, d["Kernel Name"], d["gpu__time_duration.sum"])
assert best, f"no launch of {kname} in {rep}"
json.dump({"bytes_per_launch": best[0], "read": best[1], "write": best[2], "kernel": best[3],
           "ncu_duration": best[4], "report": rep,
           "note": "dram__bytes_read.sum + dram__bytes_write.sum of the largest launch, ncu --set full, "
                   "cold L2 (ncu flushes caches between replays)"}, open(out, "w"), indent=1)
print(json.dumps(json.load(open(out))))
