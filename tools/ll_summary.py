"""Summarise an ncu launch-list CSV (--metrics gpu__time_duration.sum --csv):
per kernel name, launch count and total / mean device time.
    python tools/ll_summary.py launches.csv [more.csv ...]"""
import csv
import sys
from collections import OrderedDict


def summary(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "nsecond")
        ms = v / 1e6 if unit.startswith("n") else (v / 1e3 if unit.startswith("u") else v)
        rows.append((r["Kernel Name"].split("(")[0], ms))
    agg = OrderedDict()
    for name, ms in rows:
        c, t = agg.get(name, (0, 0.0))
        agg[name] = (c + 1, t + ms)
    print(f"== {path}: {len(rows)} launches, {sum(t for _, t in rows):.3f} ms")
    for name, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"  {t:9.3f} ms  {c:5d} x {t / c:8.4f}  {name[:90]}")
    return rows


if __name__ == "__main__":
    for p in sys.argv[1:]:
        summary(p)
