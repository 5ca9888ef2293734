"""CPU (gloo, world_size 2): the multi-GPU host logic of paper_2010_05371_b200.sharded.

The product backend is the C-ABI search plan on each GPU; here every rank
plugs the C oracle in as its shard backend, so the sharding (100000-aligned
shard starts with an (m-1)-point halo), the best-so-far all-reduce between
batches and the final lexicographic (distance, lowest global index) merge are
exercised exactly as bench.py drives them under torchrun."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2010_05371_b200.sharded import (INF_KEY, STATS_RESET, ShardedSearch, double_of,
                                           key_of, lexicographic_min, shard_bounds)


def test_shard_bounds_cover_and_align():
    for ncand in (1, 99_999, 100_000, 100_001, 999_873, 99_998_977):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_bounds(ncand, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == ncand
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0
            for s0, s1 in spans:
                assert s0 % STATS_RESET == 0 or s0 == ncand
                assert s1 >= s0


def test_keys_and_lexicographic_min():
    for d in (0.0, 1e-300, 1.5, 3.75, 1e300, float("inf")):
        assert double_of(key_of(d)) == d
    ds = [0.0, 1e-300, 1.5, 3.75, 1e300, float("inf")]
    assert [key_of(d) for d in ds] == sorted(key_of(d) for d in ds)
    assert key_of(float("inf")) == INF_KEY
    assert lexicographic_min([(True, 2.0, 9), (True, 2.0, 4), (True, 3.0, 1), (False, 0, 0)]) \
        == (True, 2.0, 4)
    assert lexicographic_min([(False, 0.0, 0)]) == (False, float("inf"), 0)


class OracleShard:
    """CPU stand-in for GpuShard: the oracle's similarity_search on the shard."""

    def __init__(self, ref, q, m, ratio, s0, s1, key):
        import oracle
        self.o = oracle.Oracle()
        self.slice = ref[s0:s1 + m - 1]
        self.q, self.m, self.ratio, self.s0 = q, m, ratio, s0
        self.key = key
        self.candidates = s1 - s0
        self.res = None
        self.runs = []

    def reset(self):
        self.key.fill_(INF_KEY)
        self.res = None

    def prepare(self):
        pass

    def run(self, begin, end):
        self.runs.append((begin, end))
        if self.res is None:
            self.res = self.o.similarity_search(self.slice, self.q, self.ratio,
                                                query_length=self.m)
        if self.res.found:
            self.key.fill_(min(int(self.key.item()), key_of(self.res.distance_sq)))

    def result(self):
        from paper_2010_05371_b200.api import BestSoFar, SearchReport, SearchResult
        r = self.res
        return SearchResult(BestSoFar(int(r.location) + self.s0, float(r.distance_sq),
                                      bool(r.found)), SearchReport())


def _worker(rank, world, port, ref, q, m, ratio, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ncand = ref.size - m + 1
        s0, s1 = shard_bounds(ncand, world, rank)
        key = torch.full((1,), 0, dtype=torch.int64)
        shard = OracleShard(ref, q, m, ratio, s0, s1, key)
        runner = ShardedSearch(shard, rank, world, batches=3)
        best, _ = runner.search()
        # every rank ends with the global minimum key after the exchanges
        out[rank] = (best, int(key.item()), len(shard.runs))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(ref, q, m, ratio, world=2):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), ref, q, m, ratio, out), nprocs=world, join=True)
    return dict(out)


@pytest.mark.timeout(300)
def test_two_rank_search_equals_unsharded(oracle_lib):
    from paper_2010_05371_b200 import random_walk_normal
    ref = random_walk_normal(260_000, 31)
    q = random_walk_normal(48, 32)
    want = oracle_lib.similarity_search(ref, q, 0.1)
    res = _run(ref, q, 48, 0.1)
    for rank in (0, 1):
        best, key, nruns = res[rank]
        assert best == (True, want.distance_sq, want.location)
        assert key == key_of(want.distance_sq)
        assert nruns == 3


@pytest.mark.timeout(300)
def test_two_rank_tie_goes_to_lowest_global_index(oracle_lib):
    """Equal minima in both shards: the final merge keeps the lower index."""
    rng = np.random.default_rng(11)
    m = 40
    ref = (rng.integers(0, 13, 250_000) - 6).astype(np.float64)
    motif = (rng.integers(0, 13, m) - 6).astype(np.float64)
    ref[150_000:150_000 + m] = motif  # rank 0 holds [0, 200000), rank 1 the rest
    ref[230_000:230_000 + m] = motif
    ref[120_000:120_000 + m] = motif
    want = oracle_lib.similarity_search(ref, motif, 0.1)
    assert want.distance_sq == 0.0 and want.location == 120_000
    res = _run(ref, motif, m, 0.1)
    for rank in (0, 1):
        assert res[rank][0] == (True, 0.0, 120_000)


# --- sharded NN1 (cfg5) ------------------------------------------------

class OracleNN1Shard:
    """CPU stand-in for GpuNN1Shard: the oracle's NN1 over rows [b0, b1) of the
    shard, with eapdtw_nn1_dev_cutoff's contract (a row counts iff its distance
    is <= the query's cutoff; none -> argmin 0, +inf)."""

    def __init__(self, queries, db_shard):
        import oracle
        self.o = oracle.Oracle()
        self.qs, self.db = queries, db_shard
        self.nq, self.rows = queries.shape[0], db_shard.shape[0]
        self.cutoffs = []

    def run(self, b0, b1, cutoff):
        c = cutoff.numpy().copy()
        self.cutoffs.append(c)
        arg, d, _ = self.o.nn1(self.qs, self.db[b0:b1])
        arg = np.asarray(arg, dtype=np.int64)
        d = np.asarray(d, dtype=np.float64)
        out = d > c
        arg[out] = 0
        d[out] = np.inf
        return arg, d


def _nn1_worker(rank, world, port, qs, db, batches, out):
    from paper_2010_05371_b200.sharded import ShardedNN1, db_shard_bounds
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d0, d1 = db_shard_bounds(db.shape[0], world, rank)
        shard = OracleNN1Shard(qs, db[d0:d1])
        arg, d = ShardedNN1(shard, rank, world, d0, batches=batches).search()
        out[rank] = (arg.tolist(), d.tolist(), [c.tolist() for c in shard.cutoffs])
    finally:
        dist.destroy_process_group()


def test_db_shard_bounds():
    from paper_2010_05371_b200.sharded import db_shard_bounds
    for nd in (1, 7, 20000, 20001):
        for world in (1, 2, 3, 8):
            spans = [db_shard_bounds(nd, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == nd
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


@pytest.mark.timeout(300)
def test_two_rank_nn1_equals_unsharded(oracle_lib):
    """Database split over 2 ranks x 3 batches with the cutoff all-reduce:
    per query the unsharded argmin and distance, ties to the lowest global
    index (exact copies planted in both ranks' halves)."""
    from paper_2010_05371_b200 import znormalize
    rng = np.random.default_rng(77)
    L, nq, nd = 32, 6, 60
    qs = np.stack([znormalize(np.cumsum(rng.standard_normal(L))) for _ in range(nq)])
    db = np.stack([znormalize(np.cumsum(rng.standard_normal(L))) for _ in range(nd)])
    db[40] = qs[0]  # rank 1 holds rows 30..59: an exact copy there ...
    db[12] = qs[0]  # ... and a lower-index one in rank 0
    db[55] = qs[1]  # only in rank 1
    want_arg, want_d, _ = oracle_lib.nn1(qs, db)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_nn1_worker, args=(2, _free_port(), qs, db, 3, out), nprocs=2, join=True)
    for rank in (0, 1):
        arg, d, cutoffs = out[rank]
        assert arg == [int(x) for x in want_arg]
        assert d == [float(x) for x in want_d]
        assert arg[0] == 12 and d[0] == 0.0 and arg[1] == 55
        # the second batch already starts from the global best of the first
        assert all(np.isinf(cutoffs[0]))
        assert not np.isinf(cutoffs[1]).any()


@pytest.mark.gpu
def test_gpu_nn1_shard_batches_and_cutoffs(oracle_lib):
    """eapdtw_nn1_dev_cutoff through GpuNN1Shard: 3 batches with the cutoff
    carried (world 1) equal the oracle; a cutoff at the exact distance keeps
    the match (ties kept); just below it finds nothing."""
    from paper_2010_05371_b200 import Context, znormalize
    from paper_2010_05371_b200.sharded import GpuNN1Shard, ShardedNN1
    rng = np.random.default_rng(5)
    L, nq, nd = 128, 40, 3000
    qs = np.stack([znormalize(np.cumsum(rng.standard_normal(L))) for _ in range(nq)])
    db = np.stack([znormalize(np.cumsum(rng.standard_normal(L))) for _ in range(nd)])
    db[2500] = qs[3]
    db[100] = qs[3]
    want_arg, want_d, _ = oracle_lib.nn1(qs, db)
    ctx = Context(0)
    shard = GpuNN1Shard(torch.from_numpy(qs).cuda(), torch.from_numpy(db).cuda(), ctx=ctx)
    arg, d = ShardedNN1(shard, 0, 1, 0, batches=3, device="cuda").search()
    assert arg.tolist() == [int(x) for x in want_arg]
    assert d.tolist() == [float(x) for x in want_d]
    assert arg[3] == 100 and d[3] == 0.0
    exact = torch.from_numpy(np.asarray(want_d)).cuda()
    a2, d2 = shard.run(0, nd, exact)
    assert a2.tolist() == [int(x) for x in want_arg] and d2.tolist() == d.tolist()
    below = torch.from_numpy(np.nextafter(np.asarray(want_d), 0.0)).cuda()
    a3, d3 = shard.run(0, nd, below)
    assert np.isinf(d3[np.asarray(want_d) > 0]).all()
    ctx.close()


# --- the same host logic on real kernels: 2 gloo ranks sharing cuda:0 -----------
# The ranks' kernels never wait on one another (the exchange happens on the
# host between launches), so two processes on one GPU are safe here.

def _gpu_worker(rank, world, port, ref, q, m, ratio, qs, db, out):
    import paper_2010_05371_b200 as g
    from paper_2010_05371_b200.sharded import (GpuNN1Shard, GpuShard, ShardedNN1,
                                               db_shard_bounds)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        ncand = ref.size - m + 1
        s0, s1 = shard_bounds(ncand, world, rank)
        dref = torch.from_numpy(ref[s0:s1 + m - 1].copy()).cuda()
        key = torch.full((1,), INF_KEY, dtype=torch.int64, device="cuda")
        shard = GpuShard(dref.data_ptr(), dref.numel(), q, g.SearchConfig(window_ratio=ratio),
                         s0, key)
        best, _ = ShardedSearch(shard, rank, world, batches=4).search()
        shard.close()
        d0, d1 = db_shard_bounds(db.shape[0], world, rank)
        nshard = GpuNN1Shard(torch.from_numpy(qs).cuda(), torch.from_numpy(db[d0:d1].copy()).cuda())
        arg, d = ShardedNN1(nshard, rank, world, d0, batches=3, device="cuda").search()
        out[rank] = (best, int(key.item()), arg.tolist(), d.tolist())
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_two_rank_gpu_shards_equal_oracle(oracle_lib):
    """cfg2-size search (N=1e6, m=128, w=6%) split over 2 ranks on cuda:0,
    GpuShard + ShardedSearch with the key all-reduced between 4 batches, and a
    2-rank GpuNN1Shard + ShardedNN1 with cutoffs carried between batches: both
    equal the oracle (ties across ranks to the lowest global index)."""
    from paper_2010_05371_b200 import random_walk_normal, znormalize
    ref = random_walk_normal(1_000_000, 7)
    q = random_walk_normal(128, 8)
    m, ratio = 128, 0.05
    ref[850_001:850_001 + m] = q * 1.7 - 0.2   # near-exact copies in rank 1's shard ...
    ref[250_003:250_003 + m] = q * 0.3 + 4.0   # ... and in rank 0's
    want = oracle_lib.similarity_search(ref, q, ratio)
    assert want.location in (250_003, 850_001) and want.distance_sq < 1e-12
    rng = np.random.default_rng(9)
    L = 96
    qs = np.stack([znormalize(np.cumsum(rng.standard_normal(L))) for _ in range(12)])
    db = np.stack([znormalize(np.cumsum(rng.standard_normal(L))) for _ in range(2000)])
    db[1500] = qs[2]
    db[300] = qs[2]
    want_arg, want_d, _ = oracle_lib.nn1(qs, db)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_gpu_worker, args=(2, _free_port(), ref, q, m, ratio, qs, db, out), nprocs=2,
             join=True)
    for rank in (0, 1):
        best, key, arg, d = out[rank]
        assert best == (True, want.distance_sq, want.location)
        assert key == key_of(want.distance_sq)
        assert arg == [int(x) for x in want_arg]
        assert d == [float(x) for x in want_d]
        assert arg[2] == 300
