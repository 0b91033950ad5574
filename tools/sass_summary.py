"""Per-kernel SASS instruction counts of the built library (the evidence that
tcgen05 / bulk-copy / HMMA / FFMA paths are what the kernels actually run):
    python tools/sass_summary.py > profiles/<tag>_sass_summary.md"""
import collections
import os
import re
import subprocess
import sys

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2303_13775_b200",
                   "libsplitgnn_b200.so")
KEYS = ["UTCHMMA", "UTCBAR", "LDTM", "UBLKCP", "HMMA", "FFMA", "LDGSTS", "LDG", "STG", "LDS", "STS", "SHFL",
        "ACQBULK", "PREEXIT", "ATOMS", "ATOMG", "RED"]
sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
counts = collections.defaultdict(collections.Counter)
cur = None
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    ins = re.search(r"/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]+)", line)
    if cur and ins and ins.group(1) in KEYS:
        counts[cur][ins.group(1)] += 1
names = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.splitlines()
rows = []
for mangled, d in zip(counts, names):
    d = d.replace("sg::(anonymous namespace)::", "").replace("(anonymous namespace)::", "").replace("sg::", "")
    d = re.sub(r"\(.*", "", d)
    rows.append((d, counts[mangled]))
out = sys.stdout
out.write(f"# SASS instruction counts: {os.path.basename(LIB)} (sm_100a, cuobjdump -sass)\n\n"
          "Static counts per kernel (not executed counts). UTCHMMA / UTCBAR / LDTM = tcgen05 MMA, commit, "
          "TMEM load; UBLKCP = cp.async.bulk; HMMA = mma.sync; ACQBULK / PREEXIT = griddepcontrol (PDL).\n\n")
out.write("| kernel | " + " | ".join(KEYS) + " |\n|---|" + "---:|" * len(KEYS) + "\n")
for d, c in sorted(rows):
    out.write(f"| `{d[:70]}` | " + " | ".join(str(c[k]) for k in KEYS) + " |\n")
