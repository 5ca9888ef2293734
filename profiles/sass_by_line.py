"""Attribute an ncu SASS-level source page to CUDA source lines.

    python profiles/sass_by_line.py <prof.ncu-rep> <cubin> <kernel-mangled-name> [top]

Uses `nvdisasm -gi` line info (build with -lineinfo) to map each SASS offset
to its innermost source line, then sums ncu's executed instructions and warp
stall samples per line.
"""
import collections
import csv
import re
import subprocess
import sys


def line_map(cubin, fn):
    txt = subprocess.run(["nvdisasm", "-gi", cubin], capture_output=True, text=True).stdout
    out = {}
    cur = None
    fresh = True  # the first location comment after an instruction is the innermost
    infn = False
    for ln in txt.splitlines():
        if ln.startswith(".text.") or ".text." in ln and ln.strip().endswith(":"):
            infn = fn in ln
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            if fresh:
                cur = (m.group(1).split("/")[-1], int(m.group(2)))
                fresh = False
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
        if m:
            fresh = True
            if infn and cur:
                out[int(m.group(1), 16)] = cur
    return out


def main():
    rep, cubin, fn = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    lm = line_map(cubin, fn)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    rows = list(csv.reader(raw))
    h = rows[1]
    data = [dict(zip(h, r)) for r in rows[2:]]
    base = int(data[0]["Address"], 16)
    ins = collections.Counter()
    smp = collections.Counter()
    for d in data:
        off = int(d["Address"], 16) - base
        key = lm.get(off, ("?", 0))
        ins[key] += int(d["Instructions Executed"] or 0)
        smp[key] += int(d["Warp Stall Sampling (All Samples)"] or 0)
    ti = sum(ins.values())
    ts = sum(smp.values())
    print(f"total warp instructions {ti:.4g}, samples {ts}")
    for k, v in ins.most_common(top):
        print(f"{100 * v / ti:6.2f}% instr {100 * smp[k] / ts:6.2f}% stall  {k[0]}:{k[1]}")


if __name__ == "__main__":
    main()
