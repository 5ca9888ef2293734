"""Samples / instructions of the sweep per code region, from tools/ncu_regions.py
output (all lines):  python tools/ncu_region_table.py regions.txt"""
import re
import sys

REGIONS = [  # (file, first line, last line, name) -- line numbers of the build profiled
    ("dtw_f32.cuh", 215, 297, "FP32 strip engine: step loop + finish masks"),
    ("dtw_f32.cuh", 46, 46, "FP32 strip engine: step loop + finish masks"),  # fmin3f of the step
    ("dtw_f32.cuh", 0, 10**9, "FP32 strip engine: strip prologue / epilogue, probe"),
    ("dtw_warp.cuh", 0, 10**9, "dtw_warp.cuh (sq_cost of the corners, exact engine, record)"),
    ("screen.cuh", 0, 10**9, "phase-A lane screen"),
    ("kernels.cu", 1009, 1276, "run_dtw: setup, cumulative-bound row thresholds"),
    ("kernels.cu", 1364, 1431, "queue: claim / pop"),
    ("kernels.cu", 1432, 1601, "LB_Kim corner + layers"),
    ("kernels.cu", 1611, 1699, "LB_Keogh terms (lb_range)"),
    ("kernels.cu", 1700, 1783, "Keogh tier stage (pop, staging, push)"),
    ("kernels.cu", 1323, 1363, "stack push / pop"),
    ("kernels.cu", 1784, 1821, "phase-A stage + publish"),
    ("kernels.cu", 0, 10**9, "kernels.cu other"),
]
tot = [0, 0, 0]
acc = {}
for line in open(sys.argv[1]):
    m = re.match(r"\s*(\d+)\s+(\d+)\s+(\d+)\s+(\S+):(\d+)", line)
    if not m:
        continue
    s, n, i, f, l = int(m[1]), int(m[2]), int(m[3]), m[4], int(m[5])
    name = f
    for rf, a, b, nm in REGIONS:
        if f == rf and a <= l <= b:
            name = nm
            break
    if f == "sm_30_intrinsics.hpp":
        name = "shuffles / votes (sm_30_intrinsics.hpp)"
    r = acc.setdefault(name, [0, 0, 0])
    r[0] += s
    r[1] += n
    r[2] += i
    tot[0] += s
    tot[1] += n
    tot[2] += i
print(f"total: {tot[0]} stall samples ({100 * tot[1] / tot[0]:.1f}% no_instruction), "
      f"{tot[2] / 1e9:.2f} G warp instructions\n")
print("| region | samples | of which no_instruction | warp instructions |")
print("|---|---:|---:|---:|")
for name, r in sorted(acc.items(), key=lambda kv: -kv[1][0]):
    if r[0] * 1000 < tot[0]:
        continue
    print(f"| {name} | {100 * r[0] / tot[0]:.1f}% | {100 * r[1] / max(1, r[0]):.0f}% | "
          f"{r[2] / 1e9:.2f} G ({100 * r[2] / tot[2]:.1f}%) |")
