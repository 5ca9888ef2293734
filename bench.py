"""bench.py -- z-normalised subsequence NN1 search under windowed DTW on B200.

Contract (driver): ``python bench.py --gpus N --steps K --warmup W`` prints ONE
JSON line on rank 0.  N>1 is launched by torchrun (one process per GPU, NCCL).

Workload (BASELINE.json configs[3], "cfg4"): a seeded float64 random walk of
1e8 points (increments N(0,1)), a random-walk query of 1024 points, window
205 cells (ratio 205/1024), z-normalised, full LB_Kim -> LB_Keogh EQ/EC ->
EAPrunedDTW cascade.  One step = one complete search of the reference.
``--impl reference`` times the reference's own CPU implementation
(oracle/_ref, compiled unmodified from /root/reference) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (n, m, ratio, description)
    "cfg2": (1_000_000, 128, 0.05, "cfg2: N=1e6 ref, m=128, w=6 (5%), LB cascade"),
    "cfg3": (10_000_000, 512, 0.1, "cfg3: N=1e7 ref, m=512, w=51 (10%), LB cascade"),
    "cfg3-nolb": (10_000_000, 512, 0.1, "cfg3: N=1e7 ref, m=512, w=51, EAPrunedDTW only"),
    "cfg4": (100_000_000, 1024, 205 / 1024,
             "cfg4: N=1e8 ref, m=1024, w=205 (ratio 205/1024), LB cascade, shards 1/2/4/8"),
}
SEED_REF, SEED_QUERY = 20261019, 20261020
# batch configs (no subsequence search): (npairs or (nq, nd), length, window)
BATCH_CONFIGS = {
    "cfg1": "cfg1: 1024 pairs of z-normalised N(0,1) random walks, L=256, w=25 (10%), "
            "cutoff +inf and 1.05 x exact; pairwise EAPrunedDTW",
    "cfg5": "cfg5: 1000 queries x 20000 database series, z-normalised N(0,1) random walks, "
            "L=512, unbounded band, running cutoff per query; NN1",
}
# the reference CLI's bench grid (eapdtw_cli.cpp:110-142)
GRID = {"n": 1_000_000, "seed": 42, "lengths": (128, 256, 512, 1024),
        "ratios": (0.1, 0.2, 0.3, 0.4, 0.5), "concurrency": 4}
GRID_DESC = ("grid: the reference CLI's bench grid (eapdtw_cli.cpp:110-142) -- query lengths "
             "128/256/512/1024 x window ratios 0.1-0.5, EAPrunedDTW + LB cascade, 20 searches of "
             "a 1e6-point random_walk(seed 42) reference (the reference's uniform-step "
             "generator, io.cpp:124-137) with prefixes of a random_walk(1024, 43) query")
FP64_OPS_PER_CELL = 5  # DSUB, DMUL, DADD + 2 DSETP (min3) per counted cell
FP32_OPS_PER_CELL = 4  # FSUB, FMUL, FADD + 1 FMNMX3 per counted cell of the FP32 screen


def mixed_roofline(cells64, cells32, seconds, p64, p32, kernel):
    """Issue roofline over both DTW engines: achieved = FP ops / time; frac = the
    time the FP pipes would need at their measured peaks / the measured time
    (so peak = achieved / frac is the cell-mix-weighted peak)."""
    ops = FP64_OPS_PER_CELL * cells64 + FP32_OPS_PER_CELL * cells32
    busy = FP64_OPS_PER_CELL * cells64 / p64 + FP32_OPS_PER_CELL * cells32 / p32
    frac = busy / seconds
    achieved = ops / seconds
    bound = "fp32" if FP32_OPS_PER_CELL * cells32 / p32 > FP64_OPS_PER_CELL * cells64 / p64 else "fp64"
    return {"bound": bound, "achieved": achieved / 1e12, "peak": achieved / frac / 1e12 if frac else None,
            "unit": "TFLOP/s", "frac": frac, "traffic": None, "kernel": kernel,
            "cells_fp64": cells64, "cells_fp32": cells32,
            "peak_fp64": p64 / 1e12, "peak_fp32": p32 / 1e12,
            "note": "CUDA-core issue roofline: 5 FP64-pipe ops per counted cell of the exact "
                    "FP64 engine, 4 FP32 ops per counted cell of the FP32 screening engine; "
                    "peaks = DADD / FADD rates measured on this GPU in this run; frac = "
                    "(time at peak) / measured time"}


def band_cells(m: int, w: int) -> int:
    w = min(w, m - 1)
    return m * (2 * w + 1) - w * (w + 1)


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML
    (pynvml, every 10 ms, from a thread) when available, else nvidia-smi
    -lms 50.  __enter__ returns once the first sample is in, so even a short
    timed region is covered; __exit__ adds one last sample."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    # nvmlClocksEventReason* bits
    NVML_BITS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                 "sw_power_cap": 0x4}  # nvmlClocksEventReason* (pynvml constants)

    def __init__(self, device: int, poll: bool = True):
        self.device = device
        self.poll = poll  # False: one sample at entry and one at exit (no thread
        #                   competing with a launch loop of microsecond kernels)
        self.rows = []  # (sm_mhz, max_mhz, set of reasons)
        self.proc = None
        self.thread = None
        self.stop = threading.Event()
        self.nvml = None

    def _nvml_sample(self):
        nv, h = self.nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        self.rows.append((float(sm), float(mx),
                          {k for k, b in self.NVML_BITS.items() if bits & b}))

    def _nvml_loop(self):
        while not self.stop.is_set():
            try:
                self._nvml_sample()
            except Exception:
                return
            self.stop.wait(0.01)

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            idx = int(vis.split(",")[self.device]) if vis and vis.split(",")[0].isdigit() else self.device
            self.nvml = (nv, nv.nvmlDeviceGetHandleByIndex(idx))
            self._nvml_sample()
            if self.poll:
                self.thread = threading.Thread(target=self._nvml_loop, daemon=True)
                self.thread.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 5.0:
                time.sleep(0.01)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7 and parts[0].replace(".", "").isdigit():
                self.rows.append((float(parts[0]),
                                  float(parts[1]) if parts[1].replace(".", "").isdigit() else None,
                                  {names[k] for k in range(4) if parts[3 + k].lower().startswith("active")}))

    def __exit__(self, *exc):
        self.stop.set()
        if self.nvml is not None:
            try:
                self._nvml_sample()
            except Exception:
                pass
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [r[0] for r in self.rows]
        mx = [r[1] for r in self.rows if r[1]]
        reasons = sorted(set().union(*(r[2] for r in self.rows)))
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows),
                "source": "nvml" if self.nvml is not None else "nvidia-smi"}


def make_inputs(n: int, m: int):
    from paper_2010_05371_b200 import random_walk_normal
    ref = random_walk_normal(n, SEED_REF)
    q = random_walk_normal(m, SEED_QUERY)
    return ref, q


def search_config(cfgname: str, world: int, batches: int) -> dict:
    """The bench line's ``config`` for a search workload -- the SAME dict on
    both arms (ours and --impl reference), so the driver compares like with
    like."""
    n, m, ratio, desc = CONFIGS[cfgname]
    return {"workload": desc, "n": n, "m": m,
            "window_cells": int(np.floor(ratio * m)), "window_ratio": ratio,
            "parallelism": f"shards{world}",
            "l2": "inputs larger than L2 (800 MB reference vs 126 MB L2)"
            if n * 8 > 126e6 else "reference smaller than L2",
            "batches_per_search": batches if world > 1 else 1}


# The reference's similarity_search is sequential; the CPU
# arm shards candidate starts at multiples of 100000 (the stats reset
# interval, search.cpp:16), one unmodified similarity_search per host thread,
# merged by (distance, lowest index) -- bit-identical to the unsharded search
# (SURVEY Appendix C).  Each shard starts from ub = +inf like any call of the
# reference's API, so shards are 1e6 candidates long (10 reset segments): long
# enough for the reference's best-so-far to converge as it does in the full
# run (calibration against a full-size run: DESIGN.md section 6).
REF_SHARD = 1_000_000


def reference_shards(ncand: int, threads: int, step: int):
    """Candidate ranges [s0, s1) of one timed step: `threads` shards of
    REF_SHARD candidates, rotating through the whole reference step by step
    (so the K timed steps sample K x threads different stretches).  Small
    configurations (ncand <= threads x REF_SHARD) run whole, split into
    100000-aligned shards."""
    if ncand <= threads * REF_SHARD:
        per = max(100_000, -(-ncand // threads // 100_000) * 100_000)
        return [(s, min(ncand, s + per)) for s in range(0, ncand, per)]
    nsh = ncand // REF_SHARD  # whole shards only
    return [((step * threads + j) % nsh * REF_SHARD, (step * threads + j) % nsh * REF_SHARD
             + REF_SHARD) for j in range(threads)]


def reference_step(lib, ref, q, m, ratio, use_lb, shards, threads):
    """Run the unmodified reference over `shards` on `threads` host threads
    (ctypes releases the GIL); returns (seconds, candidates, best)."""
    from concurrent.futures import ThreadPoolExecutor

    def one(sh):
        s0, s1 = sh
        r = lib.similarity_search_threads(ref[s0:s1 + m - 1], q, ratio, 1, query_length=m,
                                          use_lb=use_lb, tighten=use_lb)
        return (float(r.distance_sq), int(r.location) + s0) if r.found else None
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        res = [r for r in ex.map(one, shards) if r is not None]
    dt = time.perf_counter() - t0
    return dt, sum(s1 - s0 for s0, s1 in shards), min(res) if res else None


def reference_inputs(n: int, m: int):
    """The bench inputs generated by the oracle's copy of the generator (the
    reference arm must not load the product library)."""
    import oracle
    o = oracle.Oracle()
    return o.random_walk_normal(n, SEED_REF), o.random_walk_normal(m, SEED_QUERY)


def run_reference_arm(args, cfgname):
    """--impl reference: the unmodified reference (oracle/_ref, compiled from
    /root/reference by oracle/Makefile) on the host cores, same workload,
    metric and config as our arm."""
    import oracle
    n, m, ratio, desc = CONFIGS[cfgname]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    use_lb = cfgname != "cfg3-nolb"
    threads = os.cpu_count() or 1
    lib = oracle.Reference()
    ref, q = reference_inputs(n, m)
    ncand = n - m + 1
    # warm-up steps are untimed: one 100000-candidate shard per thread
    warm = [(s, min(ncand, s + 100_000)) for s in range(0, min(ncand, threads * 100_000), 100_000)]
    for _ in range(args.warmup):
        reference_step(lib, ref, q, m, ratio, use_lb, warm, threads)
    times, cands, best = [], 0, None
    for k in range(args.steps):
        shards = reference_shards(ncand, threads, k)
        dt, c, b = reference_step(lib, ref, q, m, ratio, use_lb, shards, threads)
        times.append(dt)
        cands += c
        best = b if best is None or (b is not None and b < best) else best
    value = cands / sum(times)
    shards0 = reference_shards(ncand, threads, 0)
    whole = sum(s1 - s0 for s0, s1 in shards0) == ncand
    sample = ("the whole search per step" if whole else
              f"{len(shards0)} shards of {REF_SHARD} candidates per step, rotating through the "
              f"reference ({args.steps} steps: {cands} of {ncand} candidates)")
    line = {
        "impl": "reference", "metric": "subsequences searched/sec", "value": value,
        "unit": "subsequences/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": statistics.mean(times) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: seeded N(0,1) random walks (mt19937_64 + Box-Muller), "
                "no public dataset",
        "config": search_config(cfgname, world, args.batches),
        "cpu_baseline": {"value": value, "unit": "subsequences/s", "cores": threads,
                         "kind": "reference",
                         "sample": sample + "; unmodified similarity_search per shard on "
                                   f"{threads} host threads, shards 100000-aligned; "
                                   "warm-up steps: one 100000-candidate shard per thread"},
        "e2e": {"value": value, "unit": "subsequences/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "result_over_sample": None if best is None else {"location": best[1],
                                                         "distance_sq": best[0]},
    }
    print(json.dumps(line), flush=True)
    return 0


def apply_opts(ctx, args):
    for kv in args.opt:
        k, v = kv.split("=", 1)
        ctx.set_option(k, int(v))


def hbm_peak_gbs():
    """The measured HBM copy bandwidth (MEASURED_PEAKS.json, driver-written), else
    the profiling recipe's fallback for B200."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return {"value": float(json.load(f)["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    except (OSError, KeyError, ValueError):
        return {"value": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def committed_ncu(cfg):
    """(DRAM bytes per launch, pipe/issue utilisation) of cfg's dominant kernel
    from the committed ncu capture (profiles/summarize.py report ... cfg)."""
    out = []
    for name in ("search_kernel_traffic.json", "search_kernel_ncu.json"):
        try:
            out.append(json.load(open(os.path.join(ROOT, "profiles", name))).get(cfg))
        except Exception:
            out.append(None)
    return tuple(out)


def run_batch(args):
    """cfg1 (pairwise) and cfg5 (NN1) lines: pairs/s through the public batch API
    with host buffers, the device-resident kernel time from CUDA events."""
    import ctypes as C
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    cfg = args.config
    sharded = cfg == "cfg5" and (world > 1 or args.shard_nn1) and args.impl != "reference"
    if rank != 0 and not sharded:
        return 0  # cfg1 (and the reference arm) run on rank 0; cfg5 shards its database
    if args.impl == "reference":
        # the reference arm never loads the product library: the reference's
        # own znormalize and the oracle's copy of the generator
        import oracle
        zn, rwn = oracle.Reference().znormalize, oracle.Oracle().random_walk_normal
    else:
        import torch

        import paper_2010_05371_b200 as g
        from paper_2010_05371_b200 import _capi
        zn, rwn = g.znormalize, g.random_walk_normal
    if cfg == "cfg1":
        npairs, L, w = 1024, 256, 25
        a = np.stack([zn(rwn(L, 1000 + p)) for p in range(npairs)])
        b = np.stack([zn(rwn(L, 500000 + p)) for p in range(npairs)])
        units = npairs
        unit = "pairs/s"
    else:
        nq, nd, L = 1000, 20000, 512
        rng = np.random.default_rng(SEED_REF)
        qs = np.stack([zn(np.cumsum(rng.standard_normal(L))) for _ in range(nq)])
        db = np.stack([zn(np.cumsum(rng.standard_normal(L))) for _ in range(nd)])
        units = nq * nd
        unit = "query-series pairs/s"
    if sharded:
        return run_nn1_sharded(args, qs, db, rank, world)
    if args.impl == "reference":
        import oracle
        lib = oracle.Reference() if oracle.Reference.available() else None
        threads = os.cpu_count() or 1
        times = []
        for k in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            if cfg == "cfg1":
                exact, _ = lib.pairwise_threads(a, b, w, None, threads=threads)
                lib.pairwise_threads(a, b, w, exact * 1.05, threads=threads)
                n_units = 2 * npairs
            else:
                nqs = max(1, min(nq, threads * 2))  # bounded sample: a subset of queries
                lib.nn1_threads(qs[:nqs], db, oracle.UNBOUNDED, threads=threads)
                n_units = nqs * nd
            if k >= args.warmup:
                times.append(time.perf_counter() - t0)
        v = n_units / statistics.mean(times)
        line = {"impl": "reference", "metric": unit.replace("/s", " per second"), "value": v,
                "unit": unit, "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": statistics.mean(times) * 1e3, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic z-normalised N(0,1) random walks",
                "config": {"workload": BATCH_CONFIGS[cfg]},
                "cpu_baseline": {"value": v, "unit": unit, "cores": threads, "kind": "reference",
                                 "sample": "cfg1: all 1024 pairs x 2 cutoffs" if cfg == "cfg1"
                                 else f"{nqs} of the 1000 queries vs the full database"},
                "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0
    ctx = g.Context(0)
    apply_opts(ctx, args)
    # e2e inputs come from pinned host memory (the contract's H2D), as for cfg2-4
    if cfg == "cfg1":
        a = torch.from_numpy(a).pin_memory().numpy()
        b = torch.from_numpy(b).pin_memory().numpy()
    else:
        qs = torch.from_numpy(qs).pin_memory().numpy()
        db = torch.from_numpy(db).pin_memory().numpy()
    times, dev_ms = [], []
    for k in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if cfg == "cfg1":
            exact, cells = g.pairwise(a, b, g.Band.cells(w), None, ctx=ctx)
            out, cells2 = g.pairwise(a, b, g.Band.cells(w), exact * 1.05, ctx=ctx)
            cells += cells2
            n_units = 2 * npairs
        else:
            arg, dist, cells = g.nn1(qs, db, ctx=ctx)
            n_units = units
        torch.cuda.synchronize()
        if k >= args.warmup:
            times.append(time.perf_counter() - t0)
    e2e = n_units / statistics.mean(times)
    # device-resident: inputs already in HBM, CUDA events around the kernels
    if cfg == "cfg1":
        da, dbb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        dout = torch.empty(npairs, dtype=torch.float64, device="cuda")
        ub = torch.from_numpy(exact * 1.05).cuda()
        ctx.set_stream(torch.cuda.current_stream().cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clk = ClockSampler(0, poll=False)  # a ~0.1 ms region: samples at its edges
        for k in range(args.warmup + args.steps):
            if k == args.warmup:
                clk.__enter__()
                e0.record()
            for ubp in (None, ub):
                _capi.check(_capi.lib.eapdtw_pairwise_dev(
                    ctx.handle, C.c_void_p(da.data_ptr()), C.c_void_p(dbb.data_ptr()), npairs, L, w,
                    C.c_void_p(ubp.data_ptr() if ubp is not None else 0), 1,
                    C.c_void_p(dout.data_ptr()), None))
        e1.record()
        torch.cuda.synchronize()
        clk.__exit__(None, None, None)
        ms = e0.elapsed_time(e1) / args.steps
    else:
        dq, ddb = torch.from_numpy(qs).cuda(), torch.from_numpy(db).cuda()
        arg2 = np.empty(nq, dtype=np.uint64)
        dist2 = np.empty(nq)
        ctx.set_stream(torch.cuda.current_stream().cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clk = ClockSampler(0)
        for k in range(args.warmup + args.steps):
            if k == args.warmup:
                clk.__enter__()
                e0.record()
            _capi.check(_capi.lib.eapdtw_nn1_dev(
                ctx.handle, C.c_void_p(dq.data_ptr()), nq, C.c_void_p(ddb.data_ptr()), nd, L,
                _capi.UNBOUNDED_WINDOW, arg2.ctypes.data_as(C.POINTER(C.c_uint64)),
                dist2.ctypes.data_as(C.POINTER(C.c_double)), None))
        e1.record()
        torch.cuda.synchronize()
        clk.__exit__(None, None, None)
        ms = e0.elapsed_time(e1) / args.steps
    value = n_units / (ms * 1e-3)
    cells32 = ctx.last_cells_f32 if cfg != "cfg1" else 0
    roof = mixed_roofline(cells - cells32, cells32, ms * 1e-3, ctx.fp64_peak(), ctx.fp32_peak(),
                          "pairwise_kernel" if cfg == "cfg1" else "nn1_kernel")
    roof["traffic"], roof["ncu"] = committed_ncu(cfg)
    line = {"metric": unit.replace("/s", " per second"), "value": value, "unit": unit,
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic z-normalised N(0,1) random walks",
            "config": {"workload": BATCH_CONFIGS[cfg]},
            "roofline": roof,
            "e2e": {"value": e2e, "unit": unit,
                    "h2d_bytes_per_step": int((a.nbytes + b.nbytes) * 2) if cfg == "cfg1"
                    else int(qs.nbytes + db.nbytes),
                    "d2h_bytes_per_step": int(npairs * 8 * 2) if cfg == "cfg1" else nq * 16},
            "dtw_gcups_counted": cells / (ms * 1e-3) / 1e9, "cells_per_step": cells,
            "clocks": clk.summary(),
            "gpu_launches": 2 * args.steps}  # cfg1: two pairwise launches; cfg5: init + nn1
    print(json.dumps(line), flush=True)
    return 0


def grid_reference_step(lib, ref, q, threads, sample):
    """One bounded sample of the grid on the reference: every grid point's first
    `sample` candidates (one stats segment), grid points spread over the host
    threads (ctypes releases the GIL), each an unmodified similarity_search."""
    from concurrent.futures import ThreadPoolExecutor
    points = [(L, r) for L in GRID["lengths"] for r in GRID["ratios"]]

    def one(pt):
        L, r = pt
        return lib.similarity_search_threads(ref[:sample + L - 1], q, r, 1, query_length=L)
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        res = list(ex.map(one, points))
    return time.perf_counter() - t0, len(points) * sample, res


def run_nn1_sharded(args, qs, db, rank, world):
    """cfg5 over N GPUs: each rank holds 1/N of the database rows
    and all queries; 4 batches per rank with an NCCL all-reduce (MIN) of the
    per-query cutoffs between them, then one all-gather and a lexicographic
    (distance, lowest global index) merge.  Time = max over ranks."""
    import torch
    import torch.distributed as dist

    import paper_2010_05371_b200 as g
    from paper_2010_05371_b200.sharded import GpuNN1Shard, ShardedNN1, db_shard_bounds
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    nq, nd = qs.shape[0], db.shape[0]
    d0, d1 = db_shard_bounds(nd, world, rank)
    ctx = g.Context(local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    dq = torch.from_numpy(qs).to(dev)
    ddb = torch.from_numpy(db[d0:d1]).to(dev)
    shard = GpuNN1Shard(dq, ddb, ctx=ctx)
    runner = ShardedNN1(shard, rank, world, d0, batches=4, device=dev)
    for _ in range(args.warmup):
        runner.search()
    shard.cells = 0
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = ctx.launches
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            arg, dd = runner.search()
        e1.record(stream)
        torch.cuda.synchronize()
    cells_timed = shard.cells / max(1, args.steps)
    dist.barrier()
    ms = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    launches = ctx.launches - launches0
    # e2e: pinned host shard -> HBM, then the sharded search, every step
    qp, dbp = torch.from_numpy(qs).pin_memory(), torch.from_numpy(db[d0:d1]).pin_memory()
    e2e_t = []
    for it in range(args.steps + 1):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dq.copy_(qp, non_blocking=True)
        ddb.copy_(dbp, non_blocking=True)
        runner.search()
        torch.cuda.synchronize()
        if it:
            e2e_t.append(time.perf_counter() - t0)
    te = torch.tensor([statistics.mean(e2e_t)], dtype=torch.float64, device=dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    if rank == 0:
        unit = "query-series pairs/s"
        print(json.dumps({
            "metric": "query-series pairs per second", "value": nq * nd / (ms * 1e-3),
            "unit": unit, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic z-normalised N(0,1) random walks",
            "config": {"workload": BATCH_CONFIGS["cfg5"], "parallelism": f"db{world}",
                       "batches_per_rank": runner.batches},
            "roofline": None,
            "e2e": {"value": nq * nd / float(te.item()), "unit": unit,
                    "h2d_bytes_per_step": int(qs.nbytes + db[d0:d1].nbytes),
                    "d2h_bytes_per_step": nq * 16 * runner.batches},
            "gpu_launches": launches, "clocks": clk.summary(),
            "cells_per_step_rank0": cells_timed}), flush=True)
    dist.destroy_process_group()
    return 0


def run_grid(args):
    """The paper's / reference CLI's query-length x window-ratio grid on one
    device-resident reference (DeviceSeries): subsequences searched per second
    summed over the 20 searches."""
    import oracle
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    n = GRID["n"]
    if args.impl == "reference":  # the reference's own random_walk (io.cpp:124-137)
        ref = oracle.Reference().random_walk(n, GRID["seed"])
        q = oracle.Reference().random_walk(max(GRID["lengths"]), GRID["seed"] + 1)
    else:
        import torch

        import paper_2010_05371_b200 as g
        ref = g.random_walk(n, GRID["seed"])
        q = g.random_walk(max(GRID["lengths"]), GRID["seed"] + 1)
    units = sum(n - L + 1 for L in GRID["lengths"]) * len(GRID["ratios"])
    threads = os.cpu_count() or 1
    sample = 100_000
    if args.impl == "reference":
        lib = oracle.Reference()
        times = []
        for k in range(args.warmup + args.steps):
            dt, nunits, _ = grid_reference_step(lib, ref, q, threads, sample)
            if k >= args.warmup:
                times.append(dt)
        v = nunits / statistics.mean(times)
        smp = (f"first {sample} candidates of each of the 20 grid points, grid points in "
               f"parallel on {threads} threads")
        print(json.dumps({
            "impl": "reference", "metric": "subsequences searched/sec", "value": v,
            "unit": "subsequences/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": statistics.mean(times) * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: the reference's seeded random_walk", "config": {"workload": GRID_DESC},
            "cpu_baseline": {"value": v, "unit": "subsequences/s", "cores": threads,
                             "kind": "reference", "sample": smp},
            "e2e": {"value": v, "unit": "subsequences/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}), flush=True)
        return 0
    ctx = g.Context(0)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    dref = g.DeviceSeries(ref, ctx=ctx)

    def grid_once(reference):
        return [r for _, _, _, r in g.search_grid(reference, q, GRID["lengths"], GRID["ratios"],
                                                  ctx=ctx, concurrency=GRID["concurrency"])]
    for _ in range(args.warmup):
        grid_once(dref)
    torch.cuda.synchronize()
    launches0 = g.api.total_launches()  # the worker contexts' launches included
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            results = grid_once(dref)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    launches = g.api.total_launches() - launches0
    # e2e: search_grid on host memory (one pinned H2D of the reference per grid)
    pinned = torch.from_numpy(ref).pin_memory().numpy()
    e2e_t = []
    for it in range(args.steps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res_h = grid_once(pinned)
        torch.cuda.synchronize()
        if it:
            e2e_t.append(time.perf_counter() - t0)
    for a, b in zip(results, res_h):
        assert (a.best.location, a.best.distance_sq) == (b.best.location, b.best.distance_sq)
    cpu = None
    if not args.no_cpu_baseline:
        dt, nunits, _ = grid_reference_step(oracle.Reference(), ref, q, threads, sample)
        cpu = {"value": nunits / dt, "unit": "subsequences/s", "cores": threads,
               "kind": "reference",
               "sample": f"first {sample} candidates of each grid point, {threads} threads, "
                         f"{dt:.2f} s"}
    dref.close()
    print(json.dumps({
        "metric": "subsequences searched/sec", "value": units / (ms * 1e-3),
        "unit": "subsequences/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic: the reference's seeded random_walk",
        "config": {"workload": GRID_DESC, "searches_per_step": len(results),
                   "concurrency": f"{GRID['concurrency']} contexts (streams), one per query length",
                   "timing": "CUDA events on the caller's stream around the grid; every search "
                             "returns synchronously (its worker stream drained), so the span "
                             "covers all worker streams",
                   "l2": "8 MB reference resident in HBM (fits L2; each search streams its "
                         "own stats/envelope buffers)"},
        "roofline": None, "cpu_baseline": cpu,
        "e2e": {"value": units / statistics.mean(e2e_t), "unit": "subsequences/s",
                "h2d_bytes_per_step": int(ref.nbytes + 20 * 8 * 1024),
                "d2h_bytes_per_step": 20 * 88},
        "gpu_launches": launches // max(1, args.steps) * args.steps,
        "clocks": clk.summary(),
        "per_search_ms": {f"len{L}_r{r}": res.report.elapsed_seconds * 1e3
                          for (L, r), res in zip([(L, r) for L in GRID["lengths"]
                                                  for r in GRID["ratios"]], results)},
        "cells_per_step": sum(r.report.dp_cells_evaluated for r in results)}), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg4", choices=sorted(CONFIGS) + sorted(BATCH_CONFIGS) + ["grid"])
    ap.add_argument("--batches", type=int, default=8, help="best-so-far exchanges per search (N>1)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--opt", action="append", default=[], metavar="NAME=VALUE",
                    help="engine option of the context (eapdtw_ctx_set_option), for experiments")
    ap.add_argument("--shard-nn1", action="store_true",
                    help="cfg5: the sharded driver (batches + cutoff all-reduce) even at N=1")
    args = ap.parse_args()
    if args.config == "grid":
        return run_grid(args)
    if args.config in BATCH_CONFIGS:
        return run_batch(args)
    if args.impl == "reference":
        return run_reference_arm(args, args.config)

    import torch
    import torch.distributed as dist

    import paper_2010_05371_b200 as g
    from paper_2010_05371_b200.sharded import GpuShard, ShardedSearch, shard_bounds

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    n, m, ratio, desc = CONFIGS[args.config]
    use_lb = args.config != "cfg3-nolb"
    cfg = g.SearchConfig(window_ratio=ratio, use_lower_bounds=use_lb, tighten_ub=use_lb)
    w = g.window_cells_for(ratio, m)

    t_gen = time.perf_counter()
    ref, q = make_inputs(n, m)
    t_gen = time.perf_counter() - t_gen
    ncand = n - m + 1
    s0, s1 = shard_bounds(ncand, world, rank)
    npts = (s1 - s0) + m - 1

    ctx = g.Context(local)
    apply_opts(ctx, args)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    fp64_peak = ctx.fp64_peak()  # measured DADD issue rate (ops/s) on this GPU
    fp32_peak = ctx.fp32_peak()  # measured FADD issue rate (ops/s)

    dref = torch.from_numpy(ref[s0:s0 + npts]).to(f"cuda:{local}")
    key = torch.full((1,), 0, dtype=torch.int64, device=f"cuda:{local}")
    shard = GpuShard(dref.data_ptr(), npts, q, cfg, s0, key, ctx=ctx)
    runner = ShardedSearch(shard, rank, world, batches=args.batches if world > 1 else 1)

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- warm-up
    for _ in range(args.warmup):
        best, res = runner.search()
    torch.cuda.synchronize()

    # ---- the preparation kernels timed apart (the searches below run the
    #      envelope beside the stats chain on a side stream): achieved HBM GB/s
    #      against the measured peak, algorithmic bytes = 8 B read per point +
    #      16 B written per candidate (stats) / per point (envelope)
    prep_kernels = None
    if world == 1:
        user = dict(kv.split("=") for kv in args.opt)
        hbm = hbm_peak_gbs()
        prep_kernels = {}

        def prep_phases(spec):
            ctx.set_option("prep_overlap", 0)
            ctx.set_option("spec_stats", spec)
            pp = []
            for _ in range(3):
                runner.search()
                pp.append(shard.plan.timings())
            torch.cuda.synchronize()
            return pp

        def add(name, pp, key_, nbytes):
            ms_k = statistics.median(p_[key_] for p_ in pp)
            if ms_k > 1e-3:
                gbs = nbytes / (ms_k * 1e-3) / 1e9
                prep_kernels[name] = {"ms": ms_k, "algorithmic_bytes": nbytes, "achieved_gbs": gbs,
                                      "hbm_peak_gbs": hbm["value"], "peak_source": hbm["source"],
                                      "frac": gbs / hbm["value"]}

        pp = prep_phases(0)
        add("stats_chain_kernel", pp, "stats", 8 * npts + 16 * ncand)
        add("envelope_gw_kernel", pp, "envelope", 24 * npts)
        # the speculative search's prefix-sum statistics (the chain runs beside them)
        add("fast_stats_kernel", prep_phases(1), "stats", 8 * npts + 16 * ncand)
        ctx.set_option("prep_overlap", int(user.get("prep_overlap", 1)))
        ctx.set_option("spec_stats", int(user.get("spec_stats", -1)))

    # ---- timed region: K device-resident searches
    launches0 = ctx.launches
    phases = []
    cells = []
    sweep_cnt = []
    results = []
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            best, res = runner.search()
            phases.append(shard.plan.timings())
            cells.append(res.report.dp_cells_evaluated)
            sweep_cnt.append(shard.plan.counters())
            results.append(best)
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    launches = ctx.launches - launches0
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = ncand / (ms_max * 1e-3)

    # ---- roofline of the dominant kernel (the sweep: LB tiers + pruned DTW)
    sweep_ms = statistics.mean(p["sweep"] for p in phases)
    cells_mean = statistics.mean(cells)
    c64 = statistics.mean(c["cells"] for c in sweep_cnt)
    c32 = statistics.mean(c["cells_f32"] for c in sweep_cnt)
    roof = mixed_roofline(c64, c32, sweep_ms * 1e-3, fp64_peak, fp32_peak, "search_kernel (sweep)")
    phase_ms = {k: statistics.mean(p[k] for p in phases) for k in phases[0]}

    # ---- e2e: the public API with host buffers (pinned), H2D + search + D2H every step
    pinned = torch.from_numpy(ref[s0:s0 + npts]).pin_memory()
    e2e_times = []
    for it in range(args.steps + 1):
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if world == 1:
            r = g.similarity_search(pinned.numpy(), q, cfg, ctx=ctx)
            loc_e2e = r.best.location
        else:
            dref.copy_(pinned, non_blocking=True)
            best_e2e, _ = runner.search()
            loc_e2e = best_e2e[2]
        torch.cuda.synchronize()
        barrier()
        if it > 0:
            e2e_times.append(time.perf_counter() - t0)
    e2e_s = statistics.mean(e2e_times)
    te = torch.tensor([e2e_s], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = ncand / float(te.item())

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # one step of the reference arm's sample (oracle/_ref on the host cores)
        import oracle
        threads = os.cpu_count() or 1
        shards = reference_shards(ncand, threads, 0)
        dt, c, _ = reference_step(oracle.Reference(), ref, q, m, ratio, use_lb, shards, threads)
        cpu = {"value": c / dt, "unit": "subsequences/s", "cores": threads, "kind": "reference",
               "sample": f"{len(shards)} shards ({c} candidates) of the same reference, one "
                         f"unmodified similarity_search per shard on {threads} threads, "
                         f"{dt:.2f} s"}

    # DRAM traffic and issue-slot / pipe utilisation of the sweep (committed ncu capture)
    traffic, ncu_summary = committed_ncu(args.config)

    if rank == 0:
        best = results[-1]
        line = {
            "metric": "subsequences searched/sec",
            "value": value,
            "unit": "subsequences/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_max,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic: seeded N(0,1) random walks (mt19937_64 + Box-Muller), "
                    "no public dataset",
            "config": search_config(args.config, world, args.batches),
            "roofline": dict(roof, traffic=traffic, ncu=ncu_summary),
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "subsequences/s",
                    "h2d_bytes_per_step": npts * 8 + m * 8, "d2h_bytes_per_step": 88},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "dtw_gcups_counted": cells_mean / (ms_max * 1e-3) / 1e9,
            "full_band_equiv_gcups": ncand * band_cells(m, w) / (ms_max * 1e-3) / 1e9,
            "phase_ms": phase_ms,
            "prep_kernels": prep_kernels,
            "speculative_stats": ctx.spec_info(),
            "counted_cells_per_search": cells_mean,
            "sweep_counters": shard.plan.counters(),
            "result": {"location": best[2], "distance_sq": best[1]},
            "data_gen_s": t_gen,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
