"""Print per-launch kernel durations from an ncu --csv metrics dump on stdin:
   ncu --metrics gpu__time_duration.sum --csv ... | python tools/ncu_times.py [last_n]"""
import csv
import sys

rows = [r for r in csv.reader(sys.stdin) if len(r) > 5]
hdr = next((r for r in rows if "Kernel Name" in r), None)
if hdr is None:
    sys.exit("no ncu csv on stdin")
k, v = hdr.index("Kernel Name"), hdr.index("Metric Value")
data = [(r[k].split("(")[0].split("::")[-1], float(r[v].replace(",", ""))) for r in rows[rows.index(hdr) + 1:]
        if len(r) == len(hdr)]
n = int(sys.argv[1]) if len(sys.argv) > 1 else len(data)
tot = 0.0
for name, t in data[-n:]:
    tot += t
    print(f"{t / 1e3:9.1f} us  {name}")
print(f"{tot / 1e3:9.1f} us  total of the last {n}")
