"""Top stall-sampled SASS lines from an `ncu --page source --csv --print-source sass` export.
  python tools/ncu_hot.py export.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for start, r in enumerate(rows):
    if "Address" in r and "Source" in r:
        break
hdr = rows[start]
ia, isrc, iss = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


data = [r for r in rows[start + 1:] if len(r) == len(hdr) and r[ia] != "Address"]
tot = sum(num(r[iss]) for r in data) or 1.0
print("samples", tot)
idx = {id(r): i for i, r in enumerate(data)}
for r in sorted(data, key=lambda r: -num(r[iss]))[:n]:
    i = idx[id(r)]
    prev = data[i - 1][isrc][:60] if i else ""
    print(f"{num(r[iss]) / tot * 100:5.1f}%  {r[ia]}  {r[isrc][:80]:80s} | prev: {prev}")
