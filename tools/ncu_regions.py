"""Aggregate ncu per-instruction stall samples (--page source --csv) by source
line / inlined-call region, using nvdisasm -g line info of the same cubin.
    python tools/ncu_regions.py <src.csv> <nvdisasm_lines.txt> <kernel substring> [topN]"""
import csv
import re
import sys
from collections import Counter, defaultdict

src_csv, lines_txt, kern = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
rows = list(csv.reader(open(src_csv)))
hdr = rows[1]
col = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
base = int(data[0][0], 16)
samp = {}
for r in data:
    off = int(r[0], 16) - base
    samp[off] = (int(r[col["Warp Stall Sampling (All Samples)"]] or 0),
                 int(r[col["stall_no_inst"]] or 0), int(r[col["Instructions Executed"]] or 0))
lines = open(lines_txt).read().split("\n")
start = [i for i, l in enumerate(lines) if ".text." in l and kern in l and "//---" in l][0]
cur = ("?", 0)
ctx = ""
by_line = defaultdict(lambda: [0, 0, 0])
for l in lines[start + 1:]:
    if l.startswith("//---------------------"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)(.*)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        ctx = m.group(3)
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m:
        off = int(m.group(1), 16)
        if off in samp:
            a, n, e = samp[off]
            key = cur
            by_line[key][0] += a
            by_line[key][1] += n
            by_line[key][2] += e
tot = sum(v[0] for v in by_line.values())
totn = sum(v[1] for v in by_line.values())
print(f"total samples {tot}, no_instruction {totn}")
by_file = Counter()
for k, v in by_line.items():
    by_file[k[0]] += v[0]
print("by file:", by_file.most_common())
for k, v in sorted(by_line.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0]:8d} {v[1]:7d} {v[2]:12d}  {k[0]}:{k[1]}")
