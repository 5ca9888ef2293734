"""Stall reasons per source region of one ncu --set full capture.

    python profiles/stall_by_region.py <prof.ncu-rep> <cubin> <mangled-kernel> [--loop A B]

Maps each SASS instruction of the source page to its innermost source line
(nvdisasm -gi line info), groups lines into regions (the enclosing lambda of
kernels.cu, or the header file), and sums ncu's per-instruction stall_*
sample columns.  --loop prints per-instruction samples for addresses A..B.
"""
import collections
import csv
import io
import re
import subprocess
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from sass_by_line import line_map  # noqa: E402

rep, cubin, fn = sys.argv[1:4]
src_rows = list(csv.reader(io.StringIO(subprocess.run(
    ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
    capture_output=True, text=True).stdout)))
hdr = src_rows[1]
rows = src_rows[2:]
lm = line_map(cubin, fn)
base = int(rows[0][0], 16)
kern = open(__file__.rsplit("/", 2)[0] + "/paper_2010_05371_b200/csrc/kernels.cu").read().splitlines()


def region(f, ln):
    if f != "kernels.cu":
        return f
    for k in range(ln - 1, max(0, ln - 250), -1):
        m = re.search(r"auto (\w+) = \[", kern[k])
        if m:
            return "k:" + m.group(1)
    return "k:?"


stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
agg = collections.defaultdict(lambda: collections.Counter())
for r in rows:
    off = int(r[0], 16) - base
    loc = lm.get(off)
    reg = region(*loc) if loc else "?"
    for i in stall_cols:
        agg[reg][hdr[i]] += int(r[i] or 0)
tot = sum(sum(c.values()) for c in agg.values())
for reg, c in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:8]:
    s = sum(c.values())
    top = ", ".join(f"{k[6:]} {v / s:.0%}" for k, v in c.most_common(6))
    print(f"{reg:14s} {s / tot:6.1%}  {top}")
