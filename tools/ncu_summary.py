"""Summarise ncu outputs into committed markdown under profiles/.

  python tools/ncu_summary.py launches <launches.csv> <out.md> [steps]
  python tools/ncu_summary.py full <report.ncu-rep> <out.md>
  python tools/ncu_summary.py step <launches.csv> <out.md>   (one training step)
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path, out, steps=None):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if "Kernel Name" in r)
    data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        name = d["Kernel Name"].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"].replace(",", ""))
    tot = sum(v for _, v in agg.values())
    with open(out, "w") as f:
        f.write(f"# ncu launch list: {path}\n\n`gpu__time_duration.sum`, --clock-control none, cold-cache and "
                "serialised (compare SHARES, not absolutes).\n\n")
        f.write(f"{len(data)} launches, total {tot/1e3:.1f} us")
        if steps:
            f.write(f" over {steps} steps")
        f.write("\n\n| launches | total us | share | kernel |\n|---:|---:|---:|---|\n")
        for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"| {c} | {v/1e3:.1f} | {100*v/tot:.1f}% | `{k}` |\n")


def launches_step(path, out, marker="k_meta_init"):
    """ONE training step out of a launch list: the last complete run of
    launches that starts at `marker` (every step's split begins with it) and
    ends before the next one; workload generation, sampling and warm-up
    launches are excluded."""
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if "Kernel Name" in r)
    data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
    names = [d["Kernel Name"].split("(")[0].split("::")[-1] for d in data]
    times = [float(d["Metric Value"].replace(",", "")) for d in data]
    starts = [i for i, n in enumerate(names) if n.startswith(marker)]
    if len(starts) < 2:
        raise SystemExit("fewer than two step markers")
    a, b = starts[-2], starts[-1]  # the last complete step
    tot = sum(times[a:b])
    with open(out, "w") as f:
        f.write(f"# one step from the ncu launch list {path}\n\n`gpu__time_duration.sum`, --clock-control none, "
                "cold-cache and serialised: the in-graph step overlaps the side-stream sort with the forward "
                "and is shorter; compare SHARES, not absolutes.\n\n")
        f.write(f"launches {a}..{b - 1} ({b - a} kernels), serialised total {tot / 1e3:.1f} us\n\n"
                "| # | us | share | kernel |\n|---:|---:|---:|---|\n")
        for k in range(a, b):
            f.write(f"| {k - a} | {times[k] / 1e3:.1f} | {100 * times[k] / tot:.1f}% | `{names[k]}` |\n")


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
           "smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]


def full(path, out):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    with open(out, "w") as f:
        f.write(f"# ncu --set full: {path}\n\n")
        for r in rows[2:]:
            f.write(f"## `{r[hdr.index('Kernel Name')][:120]}`\n\n| metric | value | unit |\n|---|---:|---|\n")
            for m in METRICS:
                if m in hdr:
                    i = hdr.index(m)
                    f.write(f"| {m} | {r[i]} | {units[i]} |\n")
            f.write("\n")


if __name__ == "__main__":
    if sys.argv[1] == "step":
        launches_step(sys.argv[2], sys.argv[3])
    elif sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
    else:
        full(sys.argv[2], sys.argv[3])
