"""CPU: pin the C restatement (oracle/eapdtw_oracle.c) against the reference.

Two anchors: the committed golden fixtures (produced by the unmodified
reference, tests/golden/make_golden.py) and, when oracle/_ref is built, the
reference library itself on fresh random inputs.
"""
import json
import os
import struct

import numpy as np
import pytest

import oracle

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
UNB = oracle.UNBOUNDED


def fbits(h: str) -> float:
    return struct.unpack("<d", struct.pack("<Q", int(h, 16)))[0]


def w_of(x):
    return UNB if x == -1 else x


def test_worked_example(oracle_lib):
    we = GOLDEN["worked_example"]
    for c in we["cases"]:
        v, cells = oracle_lib.dtw(c["algo"], we["S"], we["T"], w_of(c["window"]), c["ub"])
        assert v == fbits(c["value"]), c
        assert cells == c["cells"], c
    # the headline constants of test_dtw.cpp:53-131
    assert oracle_lib.dtw_windowed(we["S"], we["T"]) == 9.0
    assert oracle_lib.dtw_windowed(we["S"], we["T"], 0) == 23.0
    assert oracle_lib.ea_pruned_dtw_windowed(we["S"], we["T"], UNB, 6.0) == np.inf


def test_random_pairs_golden(oracle_lib):
    g = GOLDEN["pairs"]
    rng = np.random.default_rng(g["seed"])
    for it, c in enumerate(g["cases"]):
        la, lb = (int(x) for x in rng.integers(1, 40, 2))
        a = rng.uniform(-3, 3, la)
        b = rng.uniform(-3, 3, lb)
        w = int(rng.integers(0, 45)) if it % 5 else UNB
        full, _ = oracle_lib.dtw(0, a, b, w)
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
        assert (la, lb) == (c["la"], c["lb"])
        assert full == fbits(c["full"])
        assert ub == fbits(c["ub"])
        for algo in (1, 2):
            v, cells = oracle_lib.dtw(algo, a, b, w, ub)
            assert v == fbits(c[f"algo{algo}"]), (it, algo)
            assert cells == c[f"cells{algo}"], (it, algo)


def test_searches_golden(oracle_lib, reference_lib):
    for c in GOLDEN["searches"]:
        r = reference_lib.random_walk(c["n"], c["seed_ref"])
        q = reference_lib.random_walk(c["m"], c["seed_query"])
        res = oracle_lib.similarity_search(r, q, c["ratio"], query_length=c["m"], algo=c["algo"],
                                           use_lb=c["use_lb"], tighten=c["use_lb"])
        assert res.location == c["location"], c
        assert res.distance_sq == fbits(c["distance_sq"]), c
        got = res.as_dict()
        for k, v in c["report"].items():
            if k == "found":
                assert bool(got[k]) == bool(v)
            else:
                assert got[k] == v, (k, c)


def test_random_walk_generator_pinned(reference_lib):
    """The product's host generator equals the reference's io.cpp random_walk."""
    from paper_2010_05371_b200 import random_walk
    for n, seed in [(1, 0), (1000, 11), (100000, 20260809)]:
        assert np.array_equal(random_walk(n, seed), reference_lib.random_walk(n, seed))
    g = GOLDEN["acceptance_grid"]
    r = random_walk(g["n"], g["seed_ref"])
    assert float(np.sum(r)) == fbits(g["ref_checksum"])


def test_znormalize_bit_identical(reference_lib, oracle_lib):
    from paper_2010_05371_b200 import znormalize
    rng = np.random.default_rng(7)
    for n in (1, 2, 17, 512):
        x = np.cumsum(rng.standard_normal(n)) * 37.0 + 1e3
        assert np.array_equal(znormalize(x), reference_lib.znormalize(x))
        assert np.array_equal(znormalize(x), oracle_lib.znormalize(x))
    assert np.array_equal(znormalize(np.full(8, 5.0)), np.zeros(8))


def test_oracle_vs_reference_random(oracle_lib, reference_lib):
    rng = np.random.default_rng(99)
    for it in range(600):
        la, lb = (int(x) for x in rng.integers(1, 30, 2))
        a = rng.uniform(-3, 3, la)
        b = rng.uniform(-3, 3, lb)
        w = int(rng.integers(0, 32)) if it % 3 else UNB
        ub = rng.uniform(0, 40) if it % 2 else np.inf
        for algo in (0, 1, 2):
            assert oracle_lib.dtw(algo, a, b, w, ub) == reference_lib.dtw(algo, a, b, w, ub)
        # genuine cumulative bounds (test_dtw.cpp:326-359)
        if la == lb:
            up, lo = reference_lib.compute_envelope(a, w)
            _, contrib, _ = oracle_lib.lb_keogh(up, lo, b)
            cb = oracle_lib.cumulative_bound(contrib)
            assert oracle_lib.dtw(2, a, b, w, ub, cb) == reference_lib.dtw(2, a, b, w, ub, cb)


def test_oracle_envelope_and_errors(oracle_lib, reference_lib):
    rng = np.random.default_rng(3)
    for it in range(100):
        n = int(rng.integers(1, 64))
        s = rng.uniform(-3, 3, n)
        w = int(rng.integers(0, 70))
        u1, l1 = oracle_lib.compute_envelope(s, w)
        u2, l2 = reference_lib.compute_envelope(s, w)
        assert np.array_equal(u1, u2) and np.array_equal(l1, l2)
    with pytest.raises(ValueError):
        oracle_lib.dtw(2, [], [1.0])
    with pytest.raises(ValueError):  # cb length mismatch (dtw.cpp:66-68)
        oracle_lib.dtw(2, [1.0, 2.0, 3.0], [1.0, 2.0, 4.0], UNB, 10.0, [1.0, 0.0])
    with pytest.raises(ValueError):  # increasing cb
        oracle_lib.dtw(2, [1.0, 2.0, 3.0], [1.0, 2.0, 4.0], UNB, 10.0, [0.0, 1.0, 0.0])
    with pytest.raises(ValueError):  # bad query length (search.cpp:122-127)
        oracle_lib.similarity_search(np.arange(10.0), np.arange(5.0), 0.1, query_length=6)


def test_sliding_stats_chain(oracle_lib):
    """The oracle's stats chain reproduces the search's (incl. the 100000 reset)."""
    rng = np.random.default_rng(5)
    ref = np.cumsum(rng.standard_normal(250_000))
    mean, sd = oracle_lib.sliding_stats(ref, 64)
    # batch stats at a reset point are exact restarts
    for s in (0, 100_000, 200_000):
        w = ref[s:s + 64]
        sm = 0.0
        sq = 0.0
        for x in w:
            sm += x
            sq += x * x
        mu = sm / 64
        assert mean[s] == mu
    assert np.allclose(mean, np.convolve(ref, np.ones(64) / 64, "valid"), rtol=1e-9, atol=1e-6)


def test_oracle_generator_equals_product_generator():
    """bench.py's reference arm generates its inputs with the oracle's copy of
    the benchmark generator (it must not load the product library): same bits
    as eapdtw_random_walk_normal (host code, no GPU needed)."""
    import numpy as np

    import oracle
    from paper_2010_05371_b200 import random_walk_normal
    o = oracle.Oracle()
    for n, seed in [(1, 3), (2, 5), (1001, 20261019), (1_000_003, 20261020)]:
        a = o.random_walk_normal(n, seed)
        b = random_walk_normal(n, seed)
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), (n, seed)
