"""Markdown table of the committed bench lines (profiles/r2_bench_*.json):
    python tools/bench_table.py"""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rows = [("cfg4", "cfg4 headline (1e8, m=1024, w=205)"), ("cfg3", "cfg3 (1e7, m=512, w=51)"),
        ("cfg3-nolb", "cfg3 EAPrunedDTW only"), ("cfg2", "cfg2 (1e6, m=128, w=6)"),
        ("cfg1", "cfg1 (1024 pairs, L=256, w=25, 2 cutoffs)"),
        ("cfg5", "cfg5 (1000 x 20000, L=512, unbounded)"),
        ("grid", "grid (4 lengths x 5 ratios on a 1e6 random_walk)")]
print("| Config | GPU / step (device-resident) | Throughput | e2e (public API, pinned host input) | "
      "roofline frac | reference CPU (cpu_baseline) |")
print("|---|---:|---:|---:|---:|---:|")
for key, name in rows:
    p = os.path.join(ROOT, "profiles", f"r2_bench_{key}.json")
    if not os.path.exists(p):
        continue
    d = json.load(open(p))
    cpu = d.get("cpu_baseline") or {}
    roof = d.get("roofline") or {}
    print(f"| {name} | {d['ms_per_step']:.3g} ms | {d['value']:.3g} {d['unit']} | "
          f"{d['e2e']['value']:.3g} | {roof.get('frac', float('nan')):.3f} ({roof.get('bound', '-')}) | "
          f"{cpu.get('value', float('nan')):.3g} on {cpu.get('cores', '-')} threads |")
p = os.path.join(ROOT, "profiles", "r2_bench_ref.json")
if os.path.exists(p):
    d = json.load(open(p))
    print(f"\nreference arm (cfg4, --impl reference): {d['value']:.3g} {d['unit']} on "
          f"{d['cpu_baseline']['cores']} threads")
