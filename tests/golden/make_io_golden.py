"""Generate tests/golden/io_golden.json from the UNMODIFIED reference's file
formats (proj/src/io.cpp), compiled in place into oracle/_ref/libeapdtw_ref.so
by ``make -C oracle ref`` (ref_format_double / ref_emit_stats /
ref_load_series / ref_save_series in oracle/ref_capi.cpp forward to
io.cpp:50-55, :57-74, :17-42 and :44-48).

Run in the build container (the reference is not on the GPU box):

    python tests/golden/make_io_golden.py

The fixture pins paper_2010_05371_b200/seriesio.py (the GPU path's file
front end) without needing the reference at test time.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import struct
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

PATH_TOKEN = "@PATH@"


def bits(x: float) -> str:
    return "0x%016x" % struct.unpack("<Q", struct.pack("<d", float(x)))[0]


def format_cases() -> list[float]:
    vals = [0.0, -0.0, 1.0, -1.0, 2.0, 10.0, 100.0, 1e3, 1e4, 1e5, 1e6, 1e7, 123456.0,
            1234567.0, 0.5, 0.1, 0.25, 0.001, 0.0001, 0.00012, 1e-5, 1.5e-7, 1e-10,
            3.748871965313156, 6.256540673986855, 1.79e-24, 1e15, 1e16, 1e17, 1e21, 1e22,
            1e23, 12345678901234567890.0, 2.0 ** 53, 2.0 ** 53 + 2, 1.7976931348623157e308,
            5e-324, 2.2250738585072014e-308, 0.1 + 0.2, 1.0 / 3.0, 2.0 / 3.0, 100.5,
            99999.99, 1e-4 * 3, 4.35, 123.456, -7.25e-3, float("inf")]
    rng = np.random.default_rng(2010_05371)
    for e in range(-30, 31):
        vals.extend((rng.random(3) * 10.0 ** e).tolist())
        vals.append(float(round(rng.random() * 10 ** 6)) * 10.0 ** e)
    vals.extend((rng.standard_normal(40) * 1e3).tolist())
    return vals


def load_cases() -> list[str]:
    return ["1 2 3\n", "  -0.5\t1e3\n\n2.5e-3  \r\n", "-0 0 .5 5. 1E5 1e+05 1e-05\n",
            "3.748871965313156\n-1.7976931348623157e308\n", "5e-324 4e-320\n",
            "1e-400\n", "1e400\n", "+1\n", "abc\n", "1 2 x3\n", "1.0x\n", "inf\n",
            "nan\n", "-inf\n", "", "   \n\t\n", "0x1p3\n", "1,2\n", "1 2,\n", "1e\n",
            "--1\n", ".\n", "1..2\n", "007\n", "1_000\n", "infinity\n", "1e5.5\n"]


def trace_inputs():
    """(a, b, window, ub) cases: the worked example at the reference tests'
    thresholds (test_dtw.cpp:53-131, cli_tests.cpp:176-204) and seeded small
    pairs (equal and unequal lengths, banded and unbounded)."""
    S, T = [3.0, 1.0, 4.0, 4.0, 1.0, 1.0], [1.0, 3.0, 2.0, 1.0, 2.0, 2.0]
    cases = [(S, T, -1, ub) for ub in (float("inf"), 22.0, 9.0, 8.0, 6.0, 0.0)]
    cases += [(S, T, 1, 23.0), (S, T, 0, 22.0), ([0.0, 5.0, 0.0], [0.0, 1.0], -1, 17.0),
              ([0.0, 0.0], [0.0, 5.0], -1, 10.0), ([2.0], [5.0], -1, 9.0)]
    rng = np.random.default_rng(5371)
    for k in range(24):
        la = int(rng.integers(4, 24))
        lb = la if k % 3 else int(rng.integers(3, la + 1))
        a = np.cumsum(rng.standard_normal(la)).tolist()
        b = np.cumsum(rng.standard_normal(lb)).tolist()
        w = -1 if k % 4 == 0 else int(rng.integers(0, la))
        ub = float(rng.choice([np.inf, 1.0, 5.0, 20.0, 80.0]))
        cases.append((a, b, w, ub))
    return cases


def trace_cases(L):
    L.ref_trace_csv.argtypes = [C.c_int, C.POINTER(C.c_double), C.c_size_t,
                                C.POINTER(C.c_double), C.c_size_t, C.c_size_t, C.c_double,
                                C.c_char_p, C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
    res = []
    with tempfile.TemporaryDirectory() as tmp:
        p = os.path.join(tmp, "trace.csv")
        for a, b, w, ub in trace_inputs():
            for algo in (0, 1, 2):
                pa = (C.c_double * len(a))(*a)
                pb = (C.c_double * len(b))(*b)
                out, cells = C.c_double(0), C.c_uint64(0)
                window = oracle.UNBOUNDED if w < 0 else w
                if os.path.exists(p):
                    os.remove(p)
                rc = L.ref_trace_csv(algo, pa, len(a), pb, len(b), window, ub, p.encode(),
                                     C.byref(out), C.byref(cells))
                assert rc == 0
                text = open(p).read() if os.path.exists(p) else None
                res.append({"a": [bits(x) for x in a], "b": [bits(x) for x in b], "window": w,
                            "ub": bits(ub), "algo": algo, "result": bits(out.value),
                            "cells": cells.value, "csv": text})
    return res


def main():
    ref = oracle.Reference()
    L = ref.lib
    L.ref_format_double.argtypes = [C.c_double, C.c_char_p, C.c_size_t]
    L.ref_emit_stats.argtypes = [C.POINTER(oracle.SearchResult), C.c_char_p]
    L.ref_load_series.argtypes = [C.c_char_p, C.POINTER(C.c_double), C.c_size_t,
                                  C.POINTER(C.c_size_t), C.c_char_p, C.c_size_t]
    L.ref_save_series.argtypes = [C.POINTER(C.c_double), C.c_size_t, C.c_char_p]
    out = {"_source": "proj/src/io.cpp via oracle/_ref/libeapdtw_ref.so (make_io_golden.py)"}

    buf = C.create_string_buffer(128)
    fmt = []
    for v in format_cases():
        assert L.ref_format_double(v, buf, 128) == 0
        fmt.append([bits(v), buf.value.decode()])
    out["format_double"] = fmt

    stats = []
    reports = [
        dict(location=93139403, distance_sq=3.748871965313156, found=1, candidates_total=99998977,
             pruned_kim=91427321, pruned_keogh_eq=7053986, pruned_keogh_ec=180263,
             dtw_calls=1337407, dtw_abandoned=1337404, dp_cells_evaluated=21938966113,
             elapsed_seconds=0.05196326192220052),
        dict(location=0, distance_sq=float("inf"), found=0, candidates_total=0, pruned_kim=0,
             pruned_keogh_eq=0, pruned_keogh_ec=0, dtw_calls=0, dtw_abandoned=0,
             dp_cells_evaluated=0, elapsed_seconds=0.0),
        dict(location=42, distance_sq=0.0, found=1, candidates_total=1, pruned_kim=0,
             pruned_keogh_eq=0, pruned_keogh_ec=0, dtw_calls=1, dtw_abandoned=0,
             dp_cells_evaluated=16384, elapsed_seconds=1e-5),
        dict(location=2 ** 63 + 5, distance_sq=1.79e-24, found=1, candidates_total=2 ** 40,
             pruned_kim=12, pruned_keogh_eq=3, pruned_keogh_ec=4, dtw_calls=5,
             dtw_abandoned=6, dp_cells_evaluated=10 ** 15, elapsed_seconds=1234567.5),
        dict(location=7, distance_sq=1e16, found=1, candidates_total=8, pruned_kim=1,
             pruned_keogh_eq=1, pruned_keogh_ec=1, dtw_calls=5, dtw_abandoned=4,
             dp_cells_evaluated=99, elapsed_seconds=123.0),
        dict(location=3, distance_sq=0.0001, found=1, candidates_total=8, pruned_kim=1,
             pruned_keogh_eq=1, pruned_keogh_ec=1, dtw_calls=5, dtw_abandoned=4,
             dp_cells_evaluated=99, elapsed_seconds=1e15),
        dict(location=3, distance_sq=0.00012345, found=1, candidates_total=8, pruned_kim=1,
             pruned_keogh_eq=1, pruned_keogh_ec=1, dtw_calls=5, dtw_abandoned=4,
             dp_cells_evaluated=99, elapsed_seconds=123456789012345.6),
        dict(location=3, distance_sq=1e14, found=1, candidates_total=8, pruned_kim=1,
             pruned_keogh_eq=1, pruned_keogh_ec=1, dtw_calls=5, dtw_abandoned=4,
             dp_cells_evaluated=99, elapsed_seconds=2.5e-300),
    ]
    with tempfile.TemporaryDirectory() as tmp:
        p = os.path.join(tmp, "stats.json")
        for rep in reports:
            r = oracle.SearchResult()
            for k, v in rep.items():
                setattr(r, k, v)
            assert L.ref_emit_stats(C.byref(r), p.encode()) == 0
            with open(p) as f:
                stats.append({"report": {k: (bits(v) if isinstance(v, float) else v)
                                         for k, v in rep.items()}, "text": f.read()})
        out["emit_stats"] = stats

        loads = []
        cap = 64
        vals = (C.c_double * cap)()
        n = C.c_size_t(0)
        err = C.create_string_buffer(512)
        p = os.path.join(tmp, "series.txt")
        for content in load_cases():
            with open(p, "w") as f:
                f.write(content)
            rc = L.ref_load_series(p.encode(), vals, cap, C.byref(n), err, 512)
            if rc == 0:
                loads.append({"content": content, "values": [bits(vals[i]) for i in range(n.value)]})
            else:
                loads.append({"content": content,
                              "error": err.value.decode().replace(p, PATH_TOKEN)})
        out["load_series"] = loads
        missing = os.path.join(tmp, "missing.txt")
        rc = L.ref_load_series(missing.encode(), vals, cap, C.byref(n), err, 512)
        assert rc != 0
        out["load_missing_error"] = err.value.decode().replace(missing, PATH_TOKEN)

        saves = []
        for series in ([0.0, -0.0, 1.0, 1e-5, 3.748871965313156, 1e16, 100.0],
                       np.random.default_rng(7).standard_normal(16).tolist()):
            arr = (C.c_double * len(series))(*series)
            assert L.ref_save_series(arr, len(series), p.encode()) == 0
            with open(p) as f:
                saves.append({"values": [bits(v) for v in series], "text": f.read()})
        out["save_series"] = saves

    out["trace"] = trace_cases(L)

    with open(os.path.join(HERE, "io_golden.json"), "w") as f:
        json.dump(out, f, indent=1)
        f.write("\n")
    print(f"wrote {len(fmt)} format_double, {len(stats)} emit_stats, {len(loads)} load_series cases")


if __name__ == "__main__":
    main()
