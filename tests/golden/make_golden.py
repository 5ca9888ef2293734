"""Generate the committed golden fixtures from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref/libeapdtw_ref.so, which
``make -C oracle`` compiles from /root/reference/proj/src):

    python tests/golden/make_golden.py

Inputs are regenerated from seeds by ``paper_2010_05371_b200.random_walk``
(the reference's io.cpp:124-137 generator, pinned against
``ref_random_walk`` in tests/test_oracle.py) or by numpy's PCG64, so the
fixtures hold seeds + expected outputs (as IEEE bit patterns), not data.
"""
from __future__ import annotations

import json
import os
import struct
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

UNB = oracle.UNBOUNDED


def bits(x: float) -> str:
    return "0x%016x" % struct.unpack("<Q", struct.pack("<d", float(x)))[0]


def main():
    ref = oracle.Reference()
    out = {}

    # 1. worked example of the reference tests (test_dtw.cpp:15-16, :53-131)
    kS = [3, 1, 4, 4, 1, 1]
    kT = [1, 3, 2, 1, 2, 2]
    we = {"S": kS, "T": kT, "cases": []}
    for algo, w, ub in [(0, UNB, np.inf), (0, 0, np.inf), (0, 6, np.inf), (2, UNB, 9.0),
                        (2, UNB, 6.0), (2, 0, 22.0), (2, 0, 23.0), (2, 6, 9.0), (1, UNB, 6.0),
                        (1, UNB, 9.0)]:
        v, cells = ref.dtw(algo, kS, kT, w, ub)
        we["cases"].append({"algo": algo, "window": w if w != UNB else -1, "ub": ub,
                            "value": bits(v), "cells": cells})
    out["worked_example"] = we

    # 2. random pairs: contract sweep with ties, ub below/above, windows, cb
    rng = np.random.default_rng(20261019)
    pairs = []
    for it in range(400):
        la, lb = (int(x) for x in rng.integers(1, 40, 2))
        a = rng.uniform(-3, 3, la)
        b = rng.uniform(-3, 3, lb)
        w = int(rng.integers(0, 45)) if it % 5 else UNB
        full, _ = ref.dtw(0, a, b, w, np.inf)
        kind = it % 4
        if kind == 0:
            ub = full
        elif kind == 1:
            ub = full * rng.uniform(0.0, 1.0)
        elif kind == 2:
            ub = full * rng.uniform(1.0, 2.0) + 0.5
        else:
            ub = np.inf
        if not np.isfinite(full) and kind != 3:
            ub = rng.uniform(0, 40)
        rec = {"la": la, "lb": lb, "window": w if w != UNB else -1, "ub": bits(ub),
               "full": bits(full)}
        for algo in (1, 2):
            v, c = ref.dtw(algo, a, b, w, ub)
            rec[f"algo{algo}"] = bits(v)
            rec[f"cells{algo}"] = c
        pairs.append(rec)
    out["pairs"] = {"seed": 20261019, "generator": "numpy PCG64: la,lb=integers(1,40,2); "
                    "a,b=uniform(-3,3); w=integers(0,45) unless it%5==0 (unbounded); ub by it%4",
                    "cases": pairs}

    # 3. searches on the reference's own random_walk data
    searches = []
    for (n, sr, m, sq, ratio) in [(4000, 11, 64, 12, 0.1), (4000, 11, 64, 12, 0.3),
                                  (3000, 21, 96, 22, 0.2), (20000, 5, 128, 6, 0.05),
                                  (20000, 7, 200, 8, 0.5), (600, 3, 32, 4, 0.2),
                                  (50, 41, 1, 42, 0.1), (500, 31, 64, 32, 0.1)]:
        r = ref.random_walk(n, sr)
        q = ref.random_walk(m, sq)
        for algo in (0, 1, 2):
            for lb in (True, False):
                res = ref.similarity_search(r, q, ratio, query_length=m, algo=algo, use_lb=lb,
                                            tighten=lb)
                searches.append({"n": n, "seed_ref": sr, "m": m, "seed_query": sq,
                                 "ratio": ratio, "algo": algo, "use_lb": lb,
                                 "location": res.location, "distance_sq": bits(res.distance_sq),
                                 "report": {k: v for k, v in res.as_dict().items()
                                            if k not in ("location", "distance_sq",
                                                         "elapsed_seconds")}})
    out["searches"] = searches

    # 4. the acceptance grid data (acceptance.cpp:256-298): random_walk(100000,
    #    20260809) vs prefixes of random_walk(1024, 414243), EAP + LB + tighten.
    grid = []
    r = ref.random_walk(100000, 20260809)
    q = ref.random_walk(1024, 414243)
    for m in (128, 512, 1024):
        for ratio in (0.1, 0.2, 0.3, 0.4, 0.5):
            res = ref.similarity_search_threads(r, q, ratio, threads=os.cpu_count() or 1,
                                                query_length=m)
            grid.append({"m": m, "ratio": ratio, "location": res.location,
                         "distance_sq": bits(res.distance_sq)})
            print("grid", m, ratio, res.location, res.distance_sq, flush=True)
    out["acceptance_grid"] = {"n": 100000, "seed_ref": 20260809, "qlen": 1024,
                              "seed_query": 414243, "ref_checksum": bits(float(np.sum(r))),
                              "cases": grid}

    # 5. NN1 and pairwise batches (cfg5 / cfg1 shapes, scaled down)
    nn = []
    for (nq, nd, L, w, seed) in [(6, 300, 64, UNB, 101), (5, 200, 48, 5, 102),
                                 (4, 150, 128, 12, 103)]:
        g = np.random.default_rng(seed)
        qs = np.stack([ref.znormalize(np.cumsum(g.standard_normal(L))) for _ in range(nq)])
        db = np.stack([ref.znormalize(np.cumsum(g.standard_normal(L))) for _ in range(nd)])
        arg, dist, cells = ref.nn1_threads(qs, db, w, threads=4)
        nn.append({"nq": nq, "nd": nd, "len": L, "window": w if w != UNB else -1, "seed": seed,
                   "argmin": [int(x) for x in arg], "dist": [bits(x) for x in dist]})
    out["nn1"] = {"generator": "numpy PCG64(seed): each series = znormalize(cumsum("
                  "standard_normal(len))), queries first then db", "cases": nn}

    pw = []
    for (npairs, L, w, seed) in [(64, 256, 25, 201), (40, 100, 10, 202)]:
        g = np.random.default_rng(seed)
        a = np.stack([ref.znormalize(np.cumsum(g.standard_normal(L))) for _ in range(npairs)])
        b = np.stack([ref.znormalize(np.cumsum(g.standard_normal(L))) for _ in range(npairs)])
        exact, _ = ref.pairwise_threads(a, b, w, None, threads=4)
        o1, c1 = ref.pairwise_threads(a, b, w, None, threads=4)
        o2, c2 = ref.pairwise_threads(a, b, w, exact * 1.05, threads=4)
        o3, c3 = ref.pairwise_threads(a, b, w, exact * 0.9, threads=4)
        pw.append({"npairs": npairs, "len": L, "window": w, "seed": seed,
                   "inf": [bits(x) for x in o1], "x105": [bits(x) for x in o2],
                   "x090": [bits(x) for x in o3]})
    out["pairwise"] = {"generator": "numpy PCG64(seed): a rows then b rows, each "
                       "znormalize(cumsum(standard_normal(len)))", "cases": pw}

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
