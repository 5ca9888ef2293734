"""Stall-reason breakdown per address range of an ncu source-page CSV
(ncu -i rep --page source --csv --print-source sass -k <kernel>):
    python tools/ncu_stalls.py src.csv [lo-hi ...]   (hex offsets from the kernel start)"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
A = hdr.index("Address")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
seen, data = set(), []
for r in rows[2:]:
    if r[A] in seen:
        continue
    seen.add(r[A])
    try:
        data.append((int(r[A], 16), {k: int(r[hdr.index(k)] or 0) for k in reasons},
                     int(r[hdr.index("Instructions Executed")] or 0)))
    except ValueError:
        pass
data.sort()
base = data[0][0]
ranges = [tuple(int(x, 16) for x in a.split("-")) for a in sys.argv[2:]] or [(0, 1 << 40)]
for lo, hi in ranges:
    tot = {k: 0 for k in reasons}
    ins = 0
    for a, st, e in data:
        if lo <= a - base < hi:
            ins += e
            for k, v in st.items():
                tot[k] += v
    s = sum(tot.values())
    top = sorted(tot.items(), key=lambda kv: -kv[1])[:6]
    print(f"{lo:x}-{hi:x}: {s} samples, {ins / 1e6:.1f}M instrs: " +
          ", ".join(f"{k[6:]} {100 * v / max(s, 1):.0f}%" for k, v in top))
