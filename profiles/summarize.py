"""Summarise ncu outputs into the small text/JSON files committed under profiles/.

    python profiles/summarize.py launches <launches.csv> <out.md>
    python profiles/summarize.py report <prof.ncu-rep> <out.txt> [config-name]

`launches` turns a `--metrics gpu__time_duration.sum` launch list into a
per-kernel table (count, total, mean, share of the measured span);
`report` extracts the headline metrics of one `--set full` capture and, given a
config name, records the kernel's DRAM traffic in search_kernel_traffic.json
(read by bench.py for roofline.traffic).
"""
import collections
import csv
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
    "launch__grid_size", "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    # per-pipe utilisation: the DTW engines' min3 / compare / select / integer
    # work runs on the ALU pipe, the FP32 sub/mul/add on the FMA pipe
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.max.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
]


def launches(src, out):
    rows = [r for r in csv.reader(open(src)) if len(r) > 10]
    h = rows[0]
    agg = collections.OrderedDict()
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        ns = float(d["Metric Value"].replace(",", ""))
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ns
    total = sum(v[1] for v in agg.values())
    with open(out, "w") as f:
        f.write(f"# ncu launch list ({os.path.basename(src)}), cold-cache serialised times\n\n")
        f.write("| kernel | launches | total ms | mean ms | share |\n|---|---:|---:|---:|---:|\n")
        for k, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"| {k} | {n} | {ns / 1e6:.3f} | {ns / n / 1e6:.3f} | {ns / total:.1%} |\n")
    print(open(out).read())


def report(src, out, cfg=None):
    raw = subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout.splitlines()
    rows = list(csv.reader(raw))
    h, units, vals = rows[0], rows[1], rows[2]
    d = {k: (v, u) for k, u, v in zip(h, units, vals)}
    with open(out, "w") as f:
        f.write(f"# {os.path.basename(src)}: {d.get('Kernel Name', ('?',))[0]}\n")
        for k in KEYS:
            if k in d:
                f.write(f"{k} = {d[k][0]} {d[k][1]}\n")
    print(open(out).read())
    if cfg:
        def to_bytes(v, u):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[u]
            return float(v.replace(",", "")) * scale
        traffic = to_bytes(*d["dram__bytes_read.sum"]) + to_bytes(*d["dram__bytes_write.sum"])
        path = os.path.join(HERE, "search_kernel_traffic.json")
        pipes = os.path.join(HERE, "search_kernel_ncu.json")
        cur_p = json.load(open(pipes)) if os.path.exists(pipes) else {}

        def pct(k):
            return float(d[k][0].replace(",", "")) if k in d else None
        cur_p[cfg] = {
            "source": f"profiles/{os.path.basename(out)} (ncu --set full of {d.get('Kernel Name', ('?',))[0]})",
            "issue_slots_busy_pct": pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "alu_pipe_pct": pct("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
            "fma_pipe_pct": pct("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
            "fp64_pipe_active_pct": pct("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "lsu_pipe_pct": pct("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
            "warps_active_pct": pct("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "dram_bytes": to_bytes(*d["dram__bytes_read.sum"]) + to_bytes(*d["dram__bytes_write.sum"]),
        }
        json.dump(cur_p, open(pipes, "w"), indent=1)
        cur = json.load(open(path)) if os.path.exists(path) else {}
        cur[cfg] = traffic
        json.dump(cur, open(path, "w"), indent=1)
        print("traffic", cfg, traffic)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        report(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
