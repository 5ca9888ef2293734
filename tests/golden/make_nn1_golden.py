"""Full-size golden of the UNMODIFIED reference for cfg5 (batched NN1, SURVEY
3.3): all 1000 queries x the 20000-series database, length 512, unbounded
band, each query's running cutoff (d = ea_pruned_dtw(db[k], q, bsf), strict <
so the lowest index wins ties), computed with oracle/_ref (the reference's
dtw.cpp compiled in place), queries spread over the host threads.

    python tests/golden/make_nn1_golden.py

Inputs are bench.py's cfg5 arrays (numpy default_rng(20261019) random walks,
z-normalised with the reference's RunningStats::over + znormalize_into), so
tests/test_gpu_parity.py can regenerate them on the GPU box and compare every
(argmin, distance bits) pair without the reference.
"""
from __future__ import annotations

import json
import os
import struct
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

SEED = 20261019  # bench.py SEED_REF (cfg5 data)
NQ, ND, L = 1000, 20000, 512


def cfg5_inputs(znormalize):
    """bench.py's cfg5 queries and database (queries drawn first)."""
    rng = np.random.default_rng(SEED)
    qs = np.stack([znormalize(np.cumsum(rng.standard_normal(L))) for _ in range(NQ)])
    db = np.stack([znormalize(np.cumsum(rng.standard_normal(L))) for _ in range(ND)])
    return qs, db


def bits(x: float) -> str:
    return "0x%016x" % struct.unpack("<Q", struct.pack("<d", float(x)))[0]


def main():
    ref = oracle.Reference()
    qs, db = cfg5_inputs(ref.znormalize)
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    arg, dist, cells = ref.nn1_threads(qs, db, oracle.UNBOUNDED, threads=threads)
    dt = time.perf_counter() - t0
    out = {"nq": NQ, "nd": ND, "len": L, "seed": SEED, "window": "unbounded",
           "reference_seconds": round(dt, 1), "threads": threads, "cells": int(cells),
           "argmin": [int(a) for a in arg], "distance_sq": [bits(d) for d in dist]}
    with open(os.path.join(HERE, "nn1_cfg5_golden.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))
        f.write("\n")
    print(f"cfg5 golden: {NQ} queries in {dt:.1f} s on {threads} threads, {cells} cells")


if __name__ == "__main__":
    main()
