"""The multi-device C ABI (eapdtw_multi_*: one host thread, a context per
device, an NCCL communicator) on the one GPU this run has: the reference's
answers through the sharded search and the row-split NN1, batches and cutoff
all-reduces included.  (N > 1 shares this host logic; the gloo tests in
test_sharded.py cover the same sharding with several ranks.)"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    import paper_2010_05371_b200 as g
    return g


@pytest.fixture(scope="module")
def mg(gpu):
    m = gpu.MultiDevice([0])
    yield m
    m.close()


@pytest.mark.parametrize("n,m,ratio,lb,batches", [(450_000, 128, 0.05, True, 1),
                                                  (450_000, 300, 0.2, True, 4),
                                                  (250_001, 96, 0.1, False, 3)])
def test_multi_similarity_search_equals_oracle(gpu, oracle_lib, mg, n, m, ratio, lb, batches):
    ref = gpu.random_walk_normal(n, 600 + m)
    q = gpu.random_walk_normal(m, 601 + m)
    r = ref.copy()
    r[n // 3:n // 3 + m] = q * 1.5 - 0.5
    want = oracle_lib.similarity_search(r, q, ratio, use_lb=lb, tighten=lb)
    got = mg.similarity_search(r, q, gpu.SearchConfig(window_ratio=ratio, use_lower_bounds=lb,
                                                      tighten_ub=lb), batches=batches)
    assert (got.best.location, got.best.distance_sq) == (want.location, want.distance_sq)
    rep = got.report
    assert rep.candidates_total == n - m + 1
    assert rep.candidates_total == rep.pruned_kim + rep.pruned_keogh_eq + rep.pruned_keogh_ec + rep.dtw_calls


def test_multi_errors(gpu, mg):
    with pytest.raises(ValueError):
        mg.similarity_search(np.ones(10), np.ones(20))
    with pytest.raises(ValueError):
        gpu.MultiDevice([0, 0])


def test_multi_nn1_equals_reference(gpu, reference_lib_optional, mg):
    from paper_2010_05371_b200 import znormalize
    rng = np.random.default_rng(31)
    L = 200
    qs = np.stack([znormalize(np.cumsum(rng.standard_normal(L))) for _ in range(20)])
    db = np.stack([znormalize(np.cumsum(rng.standard_normal(L))) for _ in range(2500)])
    db[1700] = qs[4]
    db[60] = qs[4]
    for band, batches in ((None, 3), (30, 1)):
        warg, wdist, _ = reference_lib_optional.nn1(qs, db, gpu.UNBOUNDED_WINDOW if band is None
                                                    else band)
        arg, dist, cells = mg.nn1(qs, db, band, batches=batches)
        assert [int(x) for x in arg] == [int(x) for x in warg]
        assert np.array_equal(dist, wdist)
        assert cells > 0
    assert int(mg.nn1(qs, db)[0][4]) == 60
