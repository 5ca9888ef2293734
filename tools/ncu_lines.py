"""Per-source-line hot spots of an ncu source page (--print-source cuda --csv):
    python tools/ncu_lines.py src.csv [top]
Prints each file's share of warp-stall samples and executed instructions, and
the top lines by samples with their dominant stall reasons."""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
files, cur, hdr = {}, None, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Name" or r[0] == "File Path":
        cur = r[1]
        files.setdefault(cur, [])
        hdr = None
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or cur is None:
        continue
    d = dict(zip(hdr, r))
    try:
        w = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        e = int(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    st = {k[6:]: int(v or 0) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v}
    files[cur].append((w, e, int(d["Line No"]), d["Source"].strip(), st))
tw = sum(x[0] for v in files.values() for x in v) or 1
te = sum(x[1] for v in files.values() for x in v) or 1
for f, v in files.items():
    w = sum(x[0] for x in v)
    e = sum(x[1] for x in v)
    if w or e:
        print(f"{100 * w / tw:5.1f}% samples {100 * e / te:5.1f}% instrs  {f}")
allv = [(w, e, ln, src, st, f) for f, v in files.items() for (w, e, ln, src, st) in v]
allv.sort(key=lambda x: -x[0])
for w, e, ln, src, st, f in allv[:top]:
    s = sum(st.values()) or 1
    reasons = ", ".join(f"{k} {100 * c / s:.0f}%" for k, c in sorted(st.items(), key=lambda kv: -kv[1])[:3])
    print(f"{100 * w / tw:5.1f}% {100 * e / te:5.1f}%i {f.split('/')[-1]}:{ln:<5} {src[:60]:60s} | {reasons}")
