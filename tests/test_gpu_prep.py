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
