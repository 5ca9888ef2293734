"""GPU parity of the search's preparation kernels, element by element:
the sliding statistics (stats_chain_kernel, the RunningStats chain of
search.cpp:156-168 with its 100000-slide reset) and the raw sliding envelope
(envelope_kernel, compute_envelope's window of lower_bounds.cpp:9-49) against
the oracle's restatements.  Bar: every element bit-identical."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    import paper_2010_05371_b200 as g
    return g


@pytest.mark.parametrize("m", [1, 2, 7, 128, 1024])
def test_sliding_stats_bit_identical_across_resets(gpu, oracle_lib, m):
    """1.2e6 points: 12 stats segments, so the chain crosses 11 resets (and
    the last segment is short)."""
    ref = gpu.random_walk_normal(1_200_003, 300 + m)
    mean, sd = gpu.sliding_stats(ref, m)
    wmean, wsd = oracle_lib.sliding_stats(ref, m)
    assert mean.shape == wmean.shape
    assert np.array_equal(mean.view(np.uint64), wmean.view(np.uint64))
    assert np.array_equal(sd.view(np.uint64), wsd.view(np.uint64))


def test_sliding_stats_edge_cases(gpu, oracle_lib):
    """m = n (one window), a constant stretch (variance floored at 0), and a
    reference whose candidate count is an exact multiple of the reset
    interval."""
    for ref, m in [(gpu.random_walk_normal(500, 1), 500),
                   (np.concatenate([np.full(3000, 2.5), gpu.random_walk_normal(5000, 2)]), 64),
                   (gpu.random_walk_normal(200_000 + 31, 3), 32)]:
        mean, sd = gpu.sliding_stats(ref, m)
        wmean, wsd = oracle_lib.sliding_stats(ref, m)
        assert np.array_equal(mean.view(np.uint64), wmean.view(np.uint64))
        assert np.array_equal(sd.view(np.uint64), wsd.view(np.uint64))
    with pytest.raises(ValueError):
        gpu.sliding_stats(np.ones(10), 11)


@pytest.mark.parametrize("r", [0, 1, 6, 51, 205, 1024])
def test_sliding_envelope_equals_compute_envelope(gpu, oracle_lib, r):
    """The global envelope of radius r equals compute_envelope(series, r) of
    the whole series (the clamp to [0, n) at both ends included)."""
    ref = gpu.random_walk_normal(1_200_000, 400 + r)
    up, lo = gpu.sliding_envelope(ref, r)
    wup, wlo = oracle_lib.compute_envelope(ref, r)
    assert np.array_equal(up, wup)
    assert np.array_equal(lo, wlo)


def test_sliding_envelope_short_series(gpu, oracle_lib):
    """Series shorter than the radius and than one tile."""
    for n, r in [(1, 0), (1, 5), (17, 40), (300, 299), (9000, 1500)]:
        x = gpu.random_walk_normal(n, n + r)
        up, lo = gpu.sliding_envelope(x, r)
        wup, wlo = oracle_lib.compute_envelope(x, r)
        assert np.array_equal(up, wup), (n, r)
        assert np.array_equal(lo, wlo), (n, r)


# --- the reference's lower-bound API (lower_bounds.hpp:12-63) on the device --

@pytest.mark.parametrize("n,w", [(1, 0), (7, 3), (100, 0), (300, 25), (1024, 205), (500, 499),
                                 (2000, 1999), (40_000, 3000), (9000, -1)])
def test_compute_envelope_vs_reference(gpu, oracle_lib, n, w):
    """compute_envelope(series, Band) bit for bit, including radii beyond the
    tiled kernel's window (the global-memory doubling path) and unbounded."""
    x = gpu.random_walk_normal(n, 10 + n)
    band = gpu.Band.unbounded() if w < 0 else gpu.Band.cells(w)
    env = gpu.compute_envelope(x, band)
    wu, wl = oracle_lib.compute_envelope(x, oracle_lib_window(w))
    assert np.array_equal(env.upper, wu) and np.array_equal(env.lower, wl)
    assert env.window == (n if w < 0 else min(w, n))
    with pytest.raises(ValueError):
        gpu.compute_envelope([], gpu.Band.cells(3))


def oracle_lib_window(w):
    import oracle
    return oracle.UNBOUNDED if w < 0 else w


def test_lb_kim_keogh_cumulative_vs_reference(gpu, oracle_lib):
    """lb_kim_fl, lb_keogh (natural and |q|-descending order, with and without
    abandoning, contributions of the visited positions) and cumulative_bound:
    the reference's bits; invalid arguments raise like the reference."""
    rng = np.random.default_rng(123)
    for it in range(40):
        n = int(rng.integers(2, 400))
        q = gpu.znormalize(np.cumsum(rng.standard_normal(n)))
        c = gpu.znormalize(np.cumsum(rng.standard_normal(n)))
        assert gpu.lb_kim_fl(q, c) == (q[0] - c[0]) ** 2 + (q[-1] - c[-1]) ** 2
        w = int(rng.integers(0, n))
        env = gpu.compute_envelope(q, gpu.Band.cells(w))
        order = np.argsort(-np.abs(q), kind="stable")
        for ab_at in (np.inf, 0.5, 5.0):
            for o in (None, order):
                got = gpu.lb_keogh(env, c, ab_at, o)
                total, contrib, abandoned = oracle_lib.lb_keogh(env.upper, env.lower, c, ab_at, o)
                assert got.total == total and got.abandoned == abandoned
                if not abandoned:
                    assert np.array_equal(got.contributions, contrib)
                    cb = gpu.cumulative_bound(got.contributions)
                    assert np.array_equal(cb, oracle_lib.cumulative_bound(contrib))
    with pytest.raises(ValueError):
        gpu.lb_kim_fl([1.0], [2.0])
    with pytest.raises(ValueError):
        gpu.cumulative_bound([1.0, -0.5, 0.0])
    env = gpu.compute_envelope(np.arange(5.0), gpu.Band.cells(1))
    with pytest.raises(ValueError):
        gpu.lb_keogh(env, np.arange(4.0))


def test_running_stats_and_znormalize_into(gpu, oracle_lib):
    x = gpu.random_walk_normal(777, 5)
    st = gpu.RunningStats.over(x)
    out = gpu.znormalize_into(x, st)
    assert np.array_equal(out, oracle_lib.znormalize(x))
    assert np.array_equal(gpu.znormalize_into(np.full(10, 3.0), gpu.RunningStats.over(np.full(10, 3.0))),
                          np.zeros(10))


def test_left_prune_is_its_own_schedule(gpu, oracle_lib):
    """dtw_left_prune_windowed (left_prune_scan, dtw.cpp:130-182): the
    reference's value on random pairs and thresholds, and a cell count
    between EAPrunedDTW's and the full DP's (criterion 5's dominance)."""
    rng = np.random.default_rng(9)
    UNB = gpu.UNBOUNDED_WINDOW
    for it in range(300):
        la = int(rng.integers(1, 120))
        lb = la if it % 2 else int(rng.integers(1, 120))
        a = np.cumsum(rng.standard_normal(la))
        b = np.cumsum(rng.standard_normal(lb))
        w = [UNB, 3, 20, 60][it % 4]
        if w != UNB and abs(la - lb) > w:
            w = UNB
        d = oracle_lib.dtw_windowed(a, b, w)
        for ub in (np.inf, d, d * 0.7, d * 1.3):
            want = oracle_lib.dtw(1, a, b, w, ub)[0]
            got, cl = gpu.dtw_left_prune_windowed(a, b, gpu.Band(w), ub, return_cells=True)
            assert got == want, (it, la, lb, w, ub)
            with gpu.default_context().options(ad_k=0):  # the strip engine for all three
                _, ce = gpu.ea_pruned_dtw_windowed(a, b, gpu.Band(w), ub, return_cells=True)
                _, cl = gpu.dtw_left_prune_windowed(a, b, gpu.Band(w), ub, return_cells=True)
                _, cf = gpu.dtw_windowed(a, b, gpu.Band(w), return_cells=True)
            assert ce <= cl <= cf, (it, ce, cl, cf)


@pytest.mark.parametrize("lb", [True, False])
def test_left_prune_search(gpu, oracle_lib, lb):
    """Algo::left_prune searches run the left-pruning kernel: the oracle's
    answer (full and EAPrunedDTW agree), and the exact-DP cells of a
    left-pruning search lie between EAPrunedDTW's and the full DP's."""
    ref = gpu.random_walk_normal(120_000, 77)
    q = gpu.random_walk_normal(96, 78)
    want = oracle_lib.similarity_search(ref, q, 0.1, use_lb=lb, tighten=lb)
    res = {}
    for algo in (gpu.Algo.full, gpu.Algo.left_prune, gpu.Algo.ea_pruned):
        with gpu.default_context().options(f32=0, screen_rows=0):
            r = gpu.similarity_search(ref, q, gpu.SearchConfig(window_ratio=0.1, algorithm=algo,
                                                               use_lower_bounds=lb, tighten_ub=lb))
        assert (r.best.location, r.best.distance_sq) == (want.location, want.distance_sq), algo
        res[algo] = r.report.dp_cells_evaluated
    assert res[gpu.Algo.left_prune] <= res[gpu.Algo.full]
