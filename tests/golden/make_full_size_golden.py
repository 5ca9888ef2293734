"""Full-size golden results of the UNMODIFIED reference for the BASELINE search
configs cfg2-cfg4, generated in the build container with
oracle/_ref (the reference compiled in place), sharded over host threads at
100000-candidate segments (bit-identical to the unsharded search: each shard
reproduces the stats chain).

    python tests/golden/make_full_size_golden.py

Inputs are the bench's own seeded walks (bench.py SEED_REF / SEED_QUERY via
eapdtw_random_walk_normal), so tests/test_gpu_parity.py can regenerate them
on the GPU box and compare (location, distance bits) without the reference.
"""
from __future__ import annotations

import json
import os
import struct
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2010_05371_b200 as g  # noqa: E402

SEED_REF, SEED_QUERY = 20261019, 20261020  # bench.py
CONFIGS = {  # name: (n, m, ratio, use_lb)
    "cfg2": (1_000_000, 128, 0.05, True),
    "cfg3": (10_000_000, 512, 0.1, True),
    "cfg3-nolb": (10_000_000, 512, 0.1, False),
    "cfg4": (100_000_000, 1024, 205 / 1024, True),
}


def bits(x: float) -> str:
    return "0x%016x" % struct.unpack("<Q", struct.pack("<d", float(x)))[0]


def main():
    ref_lib = oracle.Reference()
    threads = os.cpu_count() or 1
    out = {}
    names = sys.argv[1:] or list(CONFIGS)
    path = os.path.join(HERE, "full_size_golden.json")
    if os.path.exists(path):
        out = json.load(open(path))
    for name in names:
        n, m, ratio, lb = CONFIGS[name]
        ref = g.random_walk_normal(n, SEED_REF)
        q = g.random_walk_normal(m, SEED_QUERY)
        t0 = time.perf_counter()
        r = ref_lib.similarity_search_threads(ref, q, ratio, threads, query_length=m,
                                              use_lb=lb, tighten=lb)
        dt = time.perf_counter() - t0
        out[name] = {"n": n, "m": m, "ratio": ratio, "use_lb": lb, "seed_ref": SEED_REF,
                     "seed_query": SEED_QUERY, "location": int(r.location),
                     "distance_sq": bits(r.distance_sq), "found": bool(r.found),
                     "reference_seconds": round(dt, 1), "threads": threads}
        print(name, out[name], flush=True)
        with open(path, "w") as f:
            json.dump(out, f, indent=1)
            f.write("\n")


if __name__ == "__main__":
    main()
