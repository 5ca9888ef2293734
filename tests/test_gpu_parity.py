"""GPU parity: the CUDA path (through the C ABI) against the oracle and the
reference's golden fixtures.  Bar: bit-exact indices and distance bits."""
import json
import os
import struct

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
UNB = oracle.UNBOUNDED


def fbits(h: str) -> float:
    return struct.unpack("<d", struct.pack("<Q", int(h, 16)))[0]


def w_of(x):
    return UNB if x == -1 else x


@pytest.fixture(scope="module")
def gpu():
    import paper_2010_05371_b200 as g
    return g


def test_worked_example(gpu):
    we = GOLDEN["worked_example"]
    S, T = we["S"], we["T"]
    assert gpu.dtw_windowed(S, T, gpu.Band.unbounded()) == 9.0
    assert gpu.dtw_windowed(S, T, gpu.Band.cells(0)) == 23.0
    assert gpu.dtw_windowed(S, T, gpu.Band.cells(6)) == 9.0
    assert gpu.ea_pruned_dtw(S, T, 9.0) == 9.0
    assert gpu.is_pruned(gpu.ea_pruned_dtw(S, T, 6.0))
    assert gpu.is_pruned(gpu.ea_pruned_dtw_windowed(S, T, gpu.Band.cells(0), 22.0))
    assert gpu.ea_pruned_dtw_windowed(S, T, gpu.Band.cells(0), 23.0) == 23.0
    # length gap beyond the band: no alignment (test_dtw.cpp:77-79)
    assert gpu.is_pruned(gpu.dtw_windowed(np.ones(5), np.ones(9), gpu.Band.cells(2)))
    # single samples (test_dtw.cpp:133-141)
    assert gpu.dtw_full([2.0], [5.0]) == 9.0
    assert gpu.ea_pruned_dtw([2.0], [5.0], 9.0) == 9.0
    assert gpu.is_pruned(gpu.ea_pruned_dtw([2.0], [5.0], 8.9))
    # ub = 0 (test_dtw.cpp:143-149)
    assert gpu.ea_pruned_dtw([1.0, 2.0], [1.0, 2.0], 0.0) == 0.0
    assert gpu.is_pruned(gpu.ea_pruned_dtw([1.0, 2.0], [1.0, 2.5], 0.0))
    # discard run ending on the last column (test_dtw.cpp:307-316)
    assert gpu.ea_pruned_dtw([0.0, 5.0, 0.0], [0.0, 1.0], 17.0) == 17.0
    assert gpu.is_pruned(gpu.ea_pruned_dtw([0.0, 0.0], [0.0, 5.0], 10.0))


def test_errors(gpu):
    with pytest.raises(ValueError):
        gpu.ea_pruned_dtw([], [1.0], 1.0)
    with pytest.raises(ValueError):
        gpu.ea_pruned_dtw_windowed([1.0, 2.0, 3.0], [1.0, 2.0, 4.0], gpu.Band.unbounded(), 10.0,
                                   [1.0, 0.0])
    with pytest.raises(ValueError):
        gpu.ea_pruned_dtw_windowed([1.0, 2.0, 3.0], [1.0, 2.0, 4.0], gpu.Band.unbounded(), 10.0,
                                   [0.0, 1.0, 0.0])
    with pytest.raises(ValueError):
        gpu.ea_pruned_dtw_windowed([1.0, 2.0, 3.0], [1.0, 2.0, 4.0], gpu.Band.unbounded(), 10.0,
                                   [3.0, 2.0, 1.0])
    ref = gpu.random_walk(500, 31)
    q = gpu.random_walk(64, 32)
    with pytest.raises(ValueError):
        gpu.similarity_search(ref, q, gpu.SearchConfig(query_length=600))
    with pytest.raises(ValueError):
        gpu.similarity_search(q, ref, gpu.SearchConfig(query_length=0))


def test_random_pairs_golden(gpu):
    g = GOLDEN["pairs"]
    rng = np.random.default_rng(g["seed"])
    for it, c in enumerate(g["cases"]):
        la, lb = (int(x) for x in rng.integers(1, 40, 2))
        a = rng.uniform(-3, 3, la)
        b = rng.uniform(-3, 3, lb)
        w = int(rng.integers(0, 45)) if it % 5 else UNB
        if it % 4 in (1, 2):  # keep the generator stream aligned with make_golden.py
            rng.uniform(0.0, 1.0)
        if not np.isfinite(fbits(c["full"])) and it % 4 != 3:
            rng.uniform(0, 40)
        ub = fbits(c["ub"])
        band = gpu.Band(w)
        assert gpu.dtw_windowed(a, b, band) == fbits(c["full"]), it
        assert gpu.ea_pruned_dtw_windowed(a, b, band, ub) == fbits(c["algo2"]), it
        # symmetry under argument swap (test_dtw.cpp:291-305)
        assert gpu.ea_pruned_dtw_windowed(b, a, band, ub) == fbits(c["algo2"]), it


def test_contract_sweep_vs_oracle(gpu, oracle_lib):
    """Early-abandon contract incl. exact ties (test_dtw.cpp:183-201, acceptance crit. 4)."""
    rng = np.random.default_rng(12345)
    for it in range(300):
        la, lb = (int(x) for x in rng.integers(1, 70, 2))
        a = rng.uniform(-3, 3, la)
        b = rng.uniform(-3, 3, lb)
        w = int(rng.integers(0, 80)) if it % 3 else UNB
        d = oracle_lib.dtw_windowed(a, b, w)
        for ub in (d, d * 0.75, d * 1.25 + 1.0, np.inf,
                   rng.uniform(0, 2 * d + 1 if np.isfinite(d) else 50.0)):
            want = oracle_lib.ea_pruned_dtw_windowed(a, b, w, ub)
            got = gpu.ea_pruned_dtw_windowed(a, b, gpu.Band(w), ub)
            assert got == want, (it, ub)
            if np.isfinite(d) and d <= ub:
                assert got == d


def test_genuine_cumulative_bound(gpu, oracle_lib):
    """cb tightening never loses a qualifying result (test_dtw.cpp:326-359)."""
    rng = np.random.default_rng(777)
    for it in range(200):
        n = int(rng.integers(2, 60))
        s = rng.uniform(-3, 3, n)
        t = rng.uniform(-3, 3, n)
        w = int(rng.integers(0, n))
        want = oracle_lib.dtw_windowed(s, t, w)
        ub = want * rng.uniform(0.6, 1.4)
        up, lo = oracle_lib.compute_envelope(s, w)
        _, contrib, _ = oracle_lib.lb_keogh(up, lo, t)
        cb = oracle_lib.cumulative_bound(contrib)
        got = gpu.ea_pruned_dtw_windowed(s, t, gpu.Band(w), ub, cb)
        if want <= ub:
            assert got == want, it
        else:
            assert gpu.is_pruned(got), it
        assert got == oracle_lib.ea_pruned_dtw_windowed(s, t, w, ub, cb), it
        assert gpu.ea_pruned_dtw_windowed(s, t, gpu.Band(w), ub, np.zeros(n)) == \
            gpu.ea_pruned_dtw_windowed(s, t, gpu.Band(w), ub)


def _pw_data(case):
    g = np.random.default_rng(case["seed"])
    from paper_2010_05371_b200 import znormalize
    L = case["len"]
    a = np.stack([znormalize(np.cumsum(g.standard_normal(L))) for _ in range(case["npairs"])])
    b = np.stack([znormalize(np.cumsum(g.standard_normal(L))) for _ in range(case["npairs"])])
    return a, b


def test_pairwise_golden(gpu):
    for case in GOLDEN["pairwise"]["cases"]:
        a, b = _pw_data(case)
        w = gpu.Band.cells(case["window"])
        exact, _ = gpu.pairwise(a, b, w, None, prune=False)
        for key, ub in (("inf", None), ("x105", exact * 1.05), ("x090", exact * 0.9)):
            out, cells = gpu.pairwise(a, b, w, ub)
            want = np.array([fbits(h) for h in case[key]])
            assert np.array_equal(out, want), key
            assert cells > 0


def test_pairwise_cfg1_full_size(gpu, oracle_lib):
    """cfg1: 1024 pairs, L=256, w=25, cutoff +inf and 1.05x exact; bit-exact."""
    from paper_2010_05371_b200 import random_walk_normal, znormalize
    a = np.stack([znormalize(random_walk_normal(256, 1000 + p)) for p in range(1024)])
    b = np.stack([znormalize(random_walk_normal(256, 5000 + p)) for p in range(1024)])
    band = gpu.Band.cells(25)
    exact, _ = oracle_lib.pairwise(a, b, 25, None)
    got, _ = gpu.pairwise(a, b, band, None)
    assert np.array_equal(got, exact)
    ub = exact * 1.05
    want, _ = oracle_lib.pairwise(a, b, 25, ub)
    got, _ = gpu.pairwise(a, b, band, ub)
    assert np.array_equal(got, want)
    assert np.isfinite(got).all()


@pytest.mark.parametrize("idx", range(len(GOLDEN["searches"])))
def test_search_golden(gpu, idx):
    c = GOLDEN["searches"][idx]
    r = gpu.random_walk(c["n"], c["seed_ref"])
    q = gpu.random_walk(c["m"], c["seed_query"])
    cfg = gpu.SearchConfig(query_length=c["m"], window_ratio=c["ratio"],
                           algorithm=gpu.Algo(c["algo"]), use_lower_bounds=c["use_lb"],
                           tighten_ub=c["use_lb"])
    res = gpu.similarity_search(r, q, cfg)
    assert res.best.found
    assert res.best.location == c["location"]
    assert res.best.distance_sq == fbits(c["distance_sq"])
    rep = res.report
    assert rep.candidates_total == c["n"] - c["m"] + 1
    assert rep.candidates_total == (rep.pruned_kim + rep.pruned_keogh_eq + rep.pruned_keogh_ec
                                    + rep.dtw_calls)
    assert rep.dtw_abandoned <= rep.dtw_calls
    if not c["use_lb"]:
        assert rep.dtw_calls == rep.candidates_total


@pytest.mark.parametrize("idx", range(15))
def test_acceptance_grid_golden(gpu, idx):
    g = GOLDEN["acceptance_grid"]
    c = g["cases"][idx]
    r = gpu.random_walk(g["n"], g["seed_ref"])
    q = gpu.random_walk(g["qlen"], g["seed_query"])
    res = gpu.similarity_search(r, q, gpu.SearchConfig(query_length=c["m"],
                                                       window_ratio=c["ratio"]))
    assert res.best.location == c["location"]
    assert res.best.distance_sq == fbits(c["distance_sq"])


def test_ties_and_exact_copy(gpu):
    """Ties go to the earliest location (test_search.cpp:209-237); an exact
    normalised copy is found at distance 0 (test_search.cpp:143-158)."""
    rng = np.random.default_rng(0x5ca40007)
    m = 40
    ref = (rng.integers(0, 13, 1500) - 6).astype(np.float64)
    motif = (rng.integers(0, 13, m) - 6).astype(np.float64)
    ref[200:200 + m] = motif
    ref[900:900 + m] = motif
    for algo in gpu.Algo:
        for lb in (True, False):
            cfg = gpu.SearchConfig(window_ratio=0.1, algorithm=algo, use_lower_bounds=lb,
                                   tighten_ub=lb)
            res = gpu.similarity_search(ref, motif, cfg)
            assert res.best.location == 200 and res.best.distance_sq == 0.0, (algo, lb)
            rep = res.report  # counter conservation (search.hpp:68-77), incl. a full queue
            assert rep.candidates_total == (rep.pruned_kim + rep.pruned_keogh_eq +
                                            rep.pruned_keogh_ec + rep.dtw_calls)
    ref2 = (rng.integers(0, 13, 2000) - 6).astype(np.float64)
    q2 = (rng.integers(0, 13, 48) - 6).astype(np.float64)
    ref2[700:748] = q2
    res = gpu.similarity_search(ref2, q2, gpu.SearchConfig(window_ratio=0.1))
    assert res.best.location == 700 and res.best.distance_sq == 0.0
    # rough integer data: the cascade prunes little, every survivor goes through
    # the queue exactly once
    for n, m in ((4000, 64), (2000, 48)):
        r = (rng.integers(0, 13, n) - 6).astype(np.float64)
        q = (rng.integers(0, 13, m) - 6).astype(np.float64)
        rep = gpu.similarity_search(r, q, gpu.SearchConfig(window_ratio=0.1)).report
        assert rep.candidates_total == n - m + 1
        assert rep.candidates_total == (rep.pruned_kim + rep.pruned_keogh_eq +
                                        rep.pruned_keogh_ec + rep.dtw_calls)


def test_degenerate_queries(gpu, oracle_lib):
    ref = gpu.random_walk(50, 41)
    q = gpu.random_walk(1, 42)
    res = gpu.similarity_search(ref, q, gpu.SearchConfig(window_ratio=0.1))
    assert res.best.location == 0 and res.best.distance_sq == 0.0
    assert res.report.candidates_total == 50
    # constant stretches normalise to zeros (search.cpp:41-44)
    ref = np.concatenate([gpu.random_walk(300, 1), np.full(200, 3.0), gpu.random_walk(300, 2)])
    q = gpu.random_walk(32, 3)
    for ratio in (0.0, 0.1, 1.0):
        want = oracle_lib.similarity_search(ref, q, ratio)
        got = gpu.similarity_search(ref, q, gpu.SearchConfig(window_ratio=ratio))
        assert (got.best.location, got.best.distance_sq) == (want.location, want.distance_sq)
    # query as long as the reference: one candidate
    r = gpu.random_walk(64, 9)
    q = gpu.random_walk(64, 10)
    want = oracle_lib.similarity_search(r, q, 0.2)
    got = gpu.similarity_search(r, q, gpu.SearchConfig(window_ratio=0.2))
    assert (got.best.location, got.best.distance_sq) == (want.location, want.distance_sq)


def test_nn1_golden(gpu):
    for c in GOLDEN["nn1"]["cases"]:
        g = np.random.default_rng(c["seed"])
        from paper_2010_05371_b200 import znormalize
        L = c["len"]
        qs = np.stack([znormalize(np.cumsum(g.standard_normal(L))) for _ in range(c["nq"])])
        db = np.stack([znormalize(np.cumsum(g.standard_normal(L))) for _ in range(c["nd"])])
        band = gpu.Band(w_of(c["window"]))
        arg, dist, cells = gpu.nn1(qs, db, band)
        assert [int(x) for x in arg] == c["argmin"]
        assert [float(x) for x in dist] == [fbits(h) for h in c["dist"]]
        assert cells > 0


def test_nn1_ties_lowest_index(gpu):
    from paper_2010_05371_b200 import znormalize
    rng = np.random.default_rng(4)
    db = np.stack([znormalize(np.cumsum(rng.standard_normal(32))) for _ in range(200)])
    db[150] = db[17]
    db[190] = db[17]
    qs = db[[17, 3]].copy()
    arg, dist, _ = gpu.nn1(qs, db)
    assert int(arg[0]) == 17 and dist[0] == 0.0
    assert int(arg[1]) == 3 and dist[1] == 0.0


def test_cfg2_full_size(gpu, oracle_lib):
    """cfg2 at its BASELINE size: N=1e6, m=128, ratio 0.05 (w=6), full cascade."""
    ref = gpu.random_walk_normal(1_000_000, 7)
    q = gpu.random_walk_normal(128, 8)
    want = oracle_lib.similarity_search(ref, q, 0.05)
    got = gpu.similarity_search(ref, q, gpu.SearchConfig(window_ratio=0.05))
    assert got.best.location == want.location
    assert got.best.distance_sq == want.distance_sq
    # cascade disabled: EAPrunedDTW alone gives the same answer
    got2 = gpu.similarity_search(ref, q, gpu.SearchConfig(window_ratio=0.05,
                                                          use_lower_bounds=False))
    assert (got2.best.location, got2.best.distance_sq) == (want.location, want.distance_sq)


def test_sharded_plan_equals_unsharded(gpu, oracle_lib):
    """Shards at multiples of 100000 with an (m-1) halo reproduce the chain."""
    import torch
    ref = gpu.random_walk_normal(350_000, 17)
    q = gpu.random_walk_normal(96, 18)
    cfg = gpu.SearchConfig(window_ratio=0.1)
    want = oracle_lib.similarity_search(ref, q, 0.1)
    dref = torch.from_numpy(ref).cuda()
    m = 96
    ncand = ref.size - m + 1
    best = None
    for s0 in range(0, ncand, 100_000):
        s1 = min(ncand, s0 + 100_000)
        plan = gpu.SearchPlan(dref.data_ptr() + 8 * s0, (s1 - s0) + m - 1, q, cfg, s0)
        plan.prepare()
        mid = plan.candidates // 2
        plan.run(0, mid)
        plan.run(mid, plan.candidates)
        r = plan.result()
        plan.close()
        cand = (r.best.distance_sq, r.best.location)
        best = cand if best is None or cand < best else best
    assert best == (want.distance_sq, want.location)


def test_engines_long_series_vs_oracle(gpu, oracle_lib):
    """Long random-walk pairs: anti-diagonal window shifts, overflow fallback
    to the strip engine, unequal lengths, all band widths; bit-exact."""
    from paper_2010_05371_b200 import znormalize
    rng = np.random.default_rng(2026)
    for it in range(120):
        la = int(rng.integers(150, 700))
        lb = la if it % 3 else int(rng.integers(100, la + 1))
        a = znormalize(np.cumsum(rng.standard_normal(la)))
        b = znormalize(np.cumsum(rng.standard_normal(lb)))
        w = [5, 30, 70, 150, 300, UNB][it % 6]
        if w != UNB and abs(la - lb) > w:
            w = UNB
        d = oracle_lib.dtw_windowed(a, b, w)
        for ub in (np.inf, d, d * 1.05, d * 0.9, d * 3.0):
            want = oracle_lib.ea_pruned_dtw_windowed(a, b, w, ub)
            got = gpu.ea_pruned_dtw_windowed(a, b, gpu.Band(w), ub)
            assert got == want, (it, la, lb, w, ub, got, want)
    # batched: every pair in one launch, mixed cutoffs
    a = np.stack([znormalize(np.cumsum(rng.standard_normal(400))) for _ in range(64)])
    b = np.stack([znormalize(np.cumsum(rng.standard_normal(400))) for _ in range(64)])
    for w in (20, 100, 250, UNB):
        exact, _ = oracle_lib.pairwise(a, b, w, None)
        ub = exact * rng.uniform(0.8, 1.3, 64)
        want, _ = oracle_lib.pairwise(a, b, w, ub)
        got, _ = gpu.pairwise(a, b, gpu.Band(w), ub)
        assert np.array_equal(got, want), w


@pytest.mark.parametrize("ad_k,screen", [(0, 0), (1, 8), (3, 16), (5, 32), (0, 64), (3, 48),
                                          (0, 16)])
def test_engine_and_screen_variants(gpu, oracle_lib, ad_k, screen):
    """Every exact DTW engine (strip, anti-diagonal K=1/3/5) and phase-A screen
    depth gives the oracle's exact answer, with and without the cascade."""
    ctx = gpu.default_context()
    for n, m, ratio, seed in [(60_000, 96, 0.1, 1), (40_000, 200, 0.3, 2), (30_000, 64, 1.0, 3),
                              (50_000, 128, 0.05, 4)]:
        ref = gpu.random_walk_normal(n, 100 + seed)
        q = gpu.random_walk_normal(m, 200 + seed)
        want = oracle_lib.similarity_search(ref, q, ratio)
        for lb in (True, False):
            with ctx.options(ad_k=ad_k, screen_rows=screen):
                got = gpu.similarity_search(ref, q, gpu.SearchConfig(window_ratio=ratio,
                                                                     use_lower_bounds=lb))
            assert (got.best.location, got.best.distance_sq) == (want.location,
                                                                 want.distance_sq), (n, m, lb)
            rep = got.report
            assert rep.candidates_total == (rep.pruned_kim + rep.pruned_keogh_eq +
                                            rep.pruned_keogh_ec + rep.dtw_calls)


def test_nn1_cfg5_database_scale(gpu, reference_lib_optional):
    """cfg5 shape: the full 20000 x 512 database, unbounded band, a subset of
    queries checked against the reference loop (running cutoff, lowest index)."""
    from paper_2010_05371_b200 import znormalize
    rng = np.random.default_rng(55)
    db = np.stack([znormalize(np.cumsum(rng.standard_normal(512))) for _ in range(20000)])
    qs = np.stack([znormalize(np.cumsum(rng.standard_normal(512))) for _ in range(6)])
    arg, dist, _ = gpu.nn1(qs, db)
    warg, wdist, _ = reference_lib_optional.nn1(qs, db, UNB)
    assert [int(x) for x in arg] == [int(x) for x in warg]
    assert np.array_equal(dist, wdist)


@pytest.mark.gpu
@pytest.mark.parametrize("m,ratio", [(64, 0.05), (300, 0.2), (700, 1.0), (1100, 0.15)])
def test_tighten_ub_never_changes_the_result(gpu, oracle_lib, m, ratio):
    """tighten_ub (lazy cumulative-bound row thresholds, search.cpp:101-113)
    against the untightened search and the oracle: identical (location, d)."""
    # (the unbounded-window case is slow on the CPU oracle: a shorter reference)
    ref = gpu.random_walk_normal(200_000 if ratio < 1.0 else 40_000, 40 + m)
    q = gpu.random_walk_normal(m, 41 + m)
    want = oracle_lib.similarity_search(ref, q, ratio)
    got = gpu.similarity_search(ref, q, gpu.SearchConfig(window_ratio=ratio, tighten_ub=True))
    off = gpu.similarity_search(ref, q, gpu.SearchConfig(window_ratio=ratio, tighten_ub=False))
    assert (got.best.location, got.best.distance_sq) == (want.location, want.distance_sq)
    assert (off.best.location, off.best.distance_sq) == (want.location, want.distance_sq)
    # a planted near-copy of the query: the threshold collapses onto it
    ref2 = ref.copy()
    at = ref.size // 2 + 1234
    ref2[at:at + m] = q * 1.5 + 0.25 + 1e-9 * np.arange(m)
    want2 = oracle_lib.similarity_search(ref2, q, ratio)
    got2 = gpu.similarity_search(ref2, q, gpu.SearchConfig(window_ratio=ratio))
    assert (got2.best.location, got2.best.distance_sq) == (want2.location, want2.distance_sq)


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,ratio,lb", [(450_000, 128, 0.1, True), (1_234_567, 300, 0.2, True),
                                          (700_001, 64, 0.05, False), (1_500_000, 256, 0.2, True)])
def test_streamed_host_search_equals_device_search(gpu, oracle_lib, n, m, ratio, lb):
    """The host-pointer search streams long references in two parts (the second
    part's copy under the first part's sweep): same answer as the oracle and as
    the unstreamed path, including a best match planted in each part."""
    ref = gpu.random_walk_normal(n, 90 + m)
    q = gpu.random_walk_normal(m, 91 + m)
    cfg = gpu.SearchConfig(window_ratio=ratio, use_lower_bounds=lb, tighten_ub=lb)
    for plant in (None, n // 5, n - m - 3):
        r = ref.copy()
        if plant is not None:
            r[plant:plant + m] = q * 2.0 - 1.0
        want = oracle_lib.similarity_search(r, q, ratio, use_lb=lb, tighten=lb)
        ctx = gpu.default_context()
        with ctx.options(streamed=1):
            got = gpu.similarity_search(r, q, cfg)
        with ctx.options(streamed=0):
            plain = gpu.similarity_search(r, q, cfg)
        assert (got.best.location, got.best.distance_sq) == (want.location, want.distance_sq)
        assert (plain.best.location, plain.best.distance_sq) == (want.location, want.distance_sq)
        assert got.report.candidates_total == n - m + 1


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,ratio,lb", [(300_000, 128, 0.05, True), (200_000, 512, 0.1, False),
                                          (150_000, 1024, 0.2, True), (60_000, 257, 1.0, True)])
def test_fp32_screen_never_changes_the_result(gpu, oracle_lib, n, m, ratio, lb):
    """The FP32 screening engine (dtw_f32.cuh) only abandons with an
    error-inflated threshold: with it (default) and without it (option f32=0)
    the search returns the oracle's (location, d) bit for bit, including
    planted near-ties whose DTW differs from the best by far less than the
    FP32 guard."""
    ref = gpu.random_walk_normal(n, 70 + m)
    q = gpu.random_walk_normal(m, 71 + m)
    r = ref.copy()
    a, b = n // 3, (2 * n) // 3
    r[a:a + m] = q * 3.0 + 7.0
    r[b:b + m] = q * 3.0 + 7.0
    r[b + m // 2] += 1e-7  # second copy: d2 a hair above the first (0)
    for arr in (ref, r):
        want = oracle_lib.similarity_search(arr, q, ratio, use_lb=lb, tighten=lb)
        cfg = gpu.SearchConfig(window_ratio=ratio, use_lower_bounds=lb, tighten_ub=lb)
        ctx = gpu.default_context()
        with ctx.options(f32=1):
            on = gpu.similarity_search(arr, q, cfg)
        with ctx.options(f32=0):
            off = gpu.similarity_search(arr, q, cfg)
        assert (on.best.location, on.best.distance_sq) == (want.location, want.distance_sq)
        assert (off.best.location, off.best.distance_sq) == (want.location, want.distance_sq)


@pytest.mark.gpu
def test_fp32_screen_falls_back_on_large_values(gpu, reference_lib_optional):
    """Series that are not z-normalised (|x| above the FP32 screen's value
    bound sqrt(len)+1) make the screen undecided: the exact engine answers.
    Mixed database: some rows within the bound, some far outside."""
    rng = np.random.default_rng(77)
    L = 128
    db = np.cumsum(rng.standard_normal((3000, L)), axis=1)
    db[::3] *= 40.0                    # every third row far outside the bound
    qs = np.cumsum(rng.standard_normal((5, L)), axis=1)
    qs[1] *= 40.0                      # one query outside too
    for band in (UNB, 12):
        arg, dist, _ = gpu.nn1(qs, db, gpu.Band(band))
        warg, wdist, _ = reference_lib_optional.nn1(qs, db, band)
        assert [int(x) for x in arg] == [int(x) for x in warg]
        assert np.array_equal(dist, wdist)


@pytest.mark.gpu
@pytest.mark.parametrize("rank", [(0, 16384, 1), (16, 16384, 1), (4, 512, 1), (8, 64, 3)])
def test_warm_start_never_changes_the_result(gpu, oracle_lib, rank):
    """The warm start (probe, rank pass with its list mode and waves, coarse
    pass) only changes the order in which candidates are tried: the answer is
    the oracle's, with the best match planted where the rank pass does not
    look (not a multiple of the rank stride) and a tie planted later."""
    n, m, ratio = 400_000, 200, 0.1
    ref = gpu.random_walk_normal(n, 501)
    q = gpu.random_walk_normal(m, 502)
    r = ref.copy()
    r[123_457:123_457 + m] = q * 0.5 + 3.0   # exact z-normalised copy (d = 0)
    r[300_001:300_001 + m] = q * 2.0 - 1.0   # a second copy: tie, higher index
    want = oracle_lib.similarity_search(r, q, ratio)
    ctx = gpu.default_context()
    for coarse in (0, 64):
        with ctx.options(rank_stride=rank[0], rank_k=rank[1], rank_waves=rank[2],
                         coarse_stride=coarse, rank_min=0):
            got = gpu.similarity_search(r, q, gpu.SearchConfig(window_ratio=ratio))
        assert (got.best.location, got.best.distance_sq) == (want.location, want.distance_sq)
        rep = got.report
        assert rep.candidates_total == n - m + 1


FULL = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "full_size_golden.json")))


@pytest.mark.parametrize("name", sorted(FULL))
def test_baseline_configs_full_size_vs_reference(gpu, name):
    """cfg2-cfg4 at their BASELINE sizes against the unmodified reference's
    answer (tests/golden/full_size_golden.json, make_full_size_golden.py):
    bit-exact location and distance through the host-pointer API (streamed
    for cfg4) and through a device-resident series."""
    c = FULL[name]
    ref = gpu.random_walk_normal(c["n"], c["seed_ref"])
    q = gpu.random_walk_normal(c["m"], c["seed_query"])
    cfg = gpu.SearchConfig(window_ratio=c["ratio"], use_lower_bounds=c["use_lb"],
                           tighten_ub=c["use_lb"])
    want = (c["location"], fbits(c["distance_sq"]))
    got = gpu.similarity_search(ref, q, cfg)
    assert (got.best.location, got.best.distance_sq) == want
    assert got.report.candidates_total == c["n"] - c["m"] + 1
    with gpu.DeviceSeries(ref) as dref:
        got2 = dref.search(q, cfg)
    assert (got2.best.location, got2.best.distance_sq) == want


NN1_GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "nn1_cfg5_golden.json")


@pytest.mark.skipif(not os.path.exists(NN1_GOLDEN), reason="cfg5 golden not generated")
def test_nn1_cfg5_full_size_vs_reference(gpu):
    """cfg5 at its BASELINE size: all 1000 queries x 20000 series x 512,
    unbounded band, against the unmodified reference's running-cutoff loop
    (tests/golden/make_nn1_golden.py): every argmin and distance bit, through
    the host API and through device-resident inputs."""
    import importlib.util
    import torch
    spec = importlib.util.spec_from_file_location(
        "make_nn1_golden", os.path.join(os.path.dirname(__file__), "golden", "make_nn1_golden.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    gold = json.load(open(NN1_GOLDEN))
    qs, db = mod.cfg5_inputs(gpu.znormalize)
    want_arg = np.array(gold["argmin"], dtype=np.uint64)
    want_d = np.array([fbits(h) for h in gold["distance_sq"]])
    arg, dist, _ = gpu.nn1(qs, db)
    assert np.array_equal(np.asarray(arg, dtype=np.uint64), want_arg)
    assert np.array_equal(dist.view(np.uint64), want_d.view(np.uint64))
    # the same through the sharded batch path on one GPU (cutoffs carried
    # between database batches, lexicographic merge)
    from paper_2010_05371_b200.sharded import GpuNN1Shard, ShardedNN1
    dq, ddb = torch.from_numpy(qs).cuda(), torch.from_numpy(db).cuda()
    sh = ShardedNN1(GpuNN1Shard(dq, ddb), 0, 1, 0, batches=3, device=dq.device)
    ai, ad = sh.search()
    assert np.array_equal(np.asarray(ai, dtype=np.uint64), want_arg)
    assert np.array_equal(ad.view(np.uint64), want_d.view(np.uint64))


@pytest.mark.parametrize("n,m,ratio,lb", [(300_000, 256, 0.2, True), (200_000, 512, 0.1, False),
                                          (150_000, 1024, 0.2, True), (60_000, 300, 1.0, True),
                                          (100_000, 40, 0.5, True), (80_000, 200, 0.15, False)])
def test_fp32_screen_probe_directions_agree(gpu, oracle_lib, n, m, ratio, lb):
    """The FP32 screen's two-direction probe (probe_strips strips forward and
    on the reversed pair, then the likelier direction to its end) and the
    forward-only pass (probe_strips 0) both return the oracle's (location, d)
    bit for bit, on plain walks and with planted exact and near-exact copies
    (one time-warped by a quarter of the band, near a band edge)."""
    ref = gpu.random_walk_normal(n, 80 + m)
    q = gpu.random_walk_normal(m, 81 + m)
    r = ref.copy()
    a, b = n // 4, (3 * n) // 5
    r[a:a + m] = q * 2.5 - 1.0
    r[b + m // 2] += 1e-7
    w = max(1, int(ratio * m) // 4)
    warped = np.concatenate([np.repeat(q[:1], w), q[:m - w]])  # q delayed by w samples
    r[b:b + m] = warped * 0.7 + 2.0
    ctx = gpu.default_context()
    cfg = gpu.SearchConfig(window_ratio=ratio, use_lower_bounds=lb, tighten_ub=lb)
    for arr in (ref, r):
        want = oracle_lib.similarity_search(arr, q, ratio, use_lb=lb, tighten=lb)
        for k in (0, 1, 2, 4):
            with ctx.options(probe_strips=k):
                got = gpu.similarity_search(arr, q, cfg)
            assert (got.best.location, got.best.distance_sq) == (want.location, want.distance_sq), k


def test_nn1_probe_directions_agree(gpu, reference_lib_optional):
    """NN1 with the two-direction FP32 probe and without it: the reference
    loop's argmin and distance bits (unbounded and banded)."""
    from paper_2010_05371_b200 import znormalize
    rng = np.random.default_rng(606)
    L = 300
    db = np.stack([znormalize(np.cumsum(rng.standard_normal(L))) for _ in range(3000)])
    qs = np.stack([znormalize(np.cumsum(rng.standard_normal(L))) for _ in range(24)])
    db[1234] = qs[5]
    ctx = gpu.default_context()
    for band in (UNB, 40):
        warg, wdist, _ = reference_lib_optional.nn1(qs, db, band)
        for k in (0, 1, 3):
            with ctx.options(probe_strips=k):
                arg, dist, _ = gpu.nn1(qs, db, gpu.Band(band))
            assert [int(x) for x in arg] == [int(x) for x in warg], k
            assert np.array_equal(dist, wdist), k


@pytest.mark.timeout(900)
def test_long_series_beyond_shared_memory(gpu, oracle_lib, reference_lib_optional):
    """Lengths whose buffers exceed shared memory run with the per-warp
    buffers in global memory (pairwise, search) or fewer warps per block
    (NN1): pairwise L = 20000, search m = 12000, NN1 L = 4096, all equal to
    the oracle / the reference loop."""
    from paper_2010_05371_b200 import znormalize
    rng = np.random.default_rng(4242)
    # pairwise, L = 20000 (and an unequal pair), band and unbounded
    a = znormalize(np.cumsum(rng.standard_normal(20_000)))
    b = znormalize(np.cumsum(rng.standard_normal(20_000)))
    c = znormalize(np.cumsum(rng.standard_normal(19_000)))
    for x, y, w in ((a, b, 2000), (a, c, 1500), (b, c, UNB)):
        d = oracle_lib.dtw_windowed(x, y, w)
        assert gpu.dtw_windowed(x, y, gpu.Band(w)) == d
        for ub in (d, d * 0.999, d * 1.5):
            assert gpu.ea_pruned_dtw_windowed(x, y, gpu.Band(w), ub) == \
                oracle_lib.ea_pruned_dtw_windowed(x, y, w, ub)
    # search, m = 12000
    ref = gpu.random_walk_normal(40_000, 4243)
    q = gpu.random_walk_normal(12_000, 4244)
    ref[21_000:33_000] = q * 0.8 + 1.0
    ref[25_000] += 1e-3
    for ratio, lb in ((0.02, True), (0.01, False)):
        want = oracle_lib.similarity_search(ref, q, ratio, use_lb=lb, tighten=lb)
        got = gpu.similarity_search(ref, q, gpu.SearchConfig(window_ratio=ratio,
                                                             use_lower_bounds=lb, tighten_ub=lb))
        assert (got.best.location, got.best.distance_sq) == (want.location, want.distance_sq)
    # NN1, L = 4096
    L = 4096
    qs = np.stack([znormalize(np.cumsum(rng.standard_normal(L))) for _ in range(3)])
    db = np.stack([znormalize(np.cumsum(rng.standard_normal(L))) for _ in range(24)])
    db[17] = qs[1]
    for band in (UNB, 300):
        warg, wdist, _ = reference_lib_optional.nn1(qs, db, band)
        arg, dist, _ = gpu.nn1(qs, db, gpu.Band(band))
        assert [int(x) for x in arg] == [int(x) for x in warg]
        assert np.array_equal(dist, wdist)


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,ratio,lb", [(300_000, 128, 0.05, True), (250_000, 512, 0.1, True),
                                          (250_000, 512, 0.1, False), (120_000, 1024, 0.2, True),
                                          (60_000, 257, 1.0, True)])
def test_speculative_statistics_never_change_the_result(gpu, oracle_lib, n, m, ratio, lb):
    """Speculative prefix-sum statistics (option spec_stats; fast_stats_kernel
    beside the exact chain of search.cpp:156-168): the search prunes on them
    with widened guards, re-evaluates the completed candidates on the chain's
    statistics, and returns the oracle's (location, d) bit for bit -- with
    planted exact ties (lowest index wins) and a near-tie 1e-7 above."""
    ref = gpu.random_walk_normal(n, 170 + m)
    q = gpu.random_walk_normal(m, 171 + m)
    r = ref.copy()
    a, b = n // 3, (2 * n) // 3
    r[a:a + m] = q * 3.0 + 7.0
    r[b:b + m] = q * 3.0 + 7.0
    r[b + m // 2] += 1e-7
    ctx = gpu.default_context()
    for arr in (ref, r):
        want = oracle_lib.similarity_search(arr, q, ratio, use_lb=lb, tighten=lb)
        cfg = gpu.SearchConfig(window_ratio=ratio, use_lower_bounds=lb, tighten_ub=lb)
        with ctx.options(spec_stats=1, streamed=0, rank_min=0 if m == 512 else 32_000_000):
            on = gpu.similarity_search(arr, q, cfg)
            info = ctx.spec_info()
        with ctx.options(spec_stats=0, streamed=0):
            off = gpu.similarity_search(arr, q, cfg)
        assert (on.best.location, on.best.distance_sq) == (want.location, want.distance_sq)
        assert (off.best.location, off.best.distance_sq) == (want.location, want.distance_sq)
        assert 0.0 <= info["deviation"] <= 8e-6 and info["listed"] >= 1
        rep = on.report
        assert rep.candidates_total == n - m + 1
        assert rep.candidates_total == (rep.pruned_kim + rep.pruned_keogh_eq + rep.pruned_keogh_ec
                                        + rep.dtw_calls)


@pytest.mark.gpu
def test_speculative_statistics_fall_back_to_the_chain(gpu, oracle_lib):
    """When the prefix-sum statistics are further from the chain's than
    assumed (here: an assumed deviation of 1e-9, below what a random walk
    shows), or disagree on a constant window (sd below 1e-12, search.cpp:13),
    nothing of the speculative pass is kept: the search is redone on the
    exact statistics and still equals the oracle."""
    n, m, ratio = 200_000, 256, 0.1
    ref = gpu.random_walk_normal(n, 991) * 50.0 + 4.0e5  # a large offset: a noisy chain
    q = gpu.random_walk_normal(m, 992)
    flat = ref.copy()
    flat[50_000:50_000 + 3 * m] = 1234.5  # constant windows
    ctx = gpu.default_context()
    for arr, opts in ((ref, dict(spec_stats=1, spec_eps=1, streamed=0)),
                      (flat, dict(spec_stats=1, streamed=0))):
        want = oracle_lib.similarity_search(arr, q, ratio)
        before = ctx.spec_info()["fallbacks"]
        with ctx.options(**opts):
            got = gpu.similarity_search(arr, q, gpu.SearchConfig(window_ratio=ratio))
            after = ctx.spec_info()
        assert (got.best.location, got.best.distance_sq) == (want.location, want.distance_sq)
        if arr is ref:
            assert after["fallbacks"] == before + 1


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,ratio", [(200_000, 300, 0.1), (150_000, 1024, 0.2), (120_000, 257, 0.05)])
def test_keogh_visiting_order_never_changes_the_result(gpu, oracle_lib, n, m, ratio):
    """The LB_Keogh tiers visit the positions by descending |q| like the
    reference (search.cpp:143-149, option lb_blocks=0) or by parts (the first
    256 positions, then the rest: lb_blocks=1, the default): any order gives
    the same sums, so both return the oracle's (location, d) bit for bit, and
    the counter invariant holds."""
    ref = gpu.random_walk_normal(n, 270 + m)
    q = gpu.random_walk_normal(m, 271 + m)
    want = oracle_lib.similarity_search(ref, q, ratio)
    ctx = gpu.default_context()
    for blocks in (0, 1):
        with ctx.options(lb_blocks=blocks):
            got = gpu.similarity_search(ref, q, gpu.SearchConfig(window_ratio=ratio))
        assert (got.best.location, got.best.distance_sq) == (want.location, want.distance_sq)
        rep = got.report
        assert rep.candidates_total == (rep.pruned_kim + rep.pruned_keogh_eq + rep.pruned_keogh_ec
                                        + rep.dtw_calls)
