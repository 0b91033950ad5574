"""Summarise an `ncu --csv --metrics ...` log: per kernel-name launch count
and mean of each metric (diagnostic helper)."""
import csv
import sys
from collections import defaultdict


def main(path, top=40):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.reader(lines[start:]))
    hdr = rows[0]
    ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = defaultdict(dict)
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        per[int(r[ii])]["name"] = r[ki]
        try:
            per[int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
        except ValueError:
            pass
    agg = defaultdict(lambda: defaultdict(list))
    order = []
    for i in sorted(per):
        nm = per[i]["name"].split("(")[0][-70:]
        if nm not in agg:
            order.append(nm)
        for k, v in per[i].items():
            if k != "name":
                agg[nm][k].append(v)
    for nm in order[:int(top)]:
        d = agg[nm]
        cols = " ".join(f"{k.split('__')[-1][:22]}={sum(v)/len(v):.0f}" for k, v in d.items())
        print(f"{len(next(iter(d.values())))}x {nm}: {cols}")


if __name__ == "__main__":
    main(*sys.argv[1:])
