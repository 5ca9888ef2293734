"""Multi-GPU subsequence search: one process per GPU, torch.distributed (NCCL).

The reference series is split into contiguous candidate ranges, one per rank.
Shard starts are multiples of 100000 candidates -- the stats reset interval of
similarity_search (search.cpp:16, :164-167) -- and every shard carries the
(m-1)-point halo its last candidates need, so each rank's stats chain is
bit-identical to the unsharded one.  The only exchange is the
best-so-far: between candidate batches the ranks all-reduce (MIN) the 8-byte
order-preserving threshold key, so every rank prunes with the global best.  The
final answer is the lexicographic (distance, lowest global index) minimum,
gathered once at the end.

The compute backend is pluggable so the host logic can be exercised on CPU
with gloo (tests/test_sharded.py): ``GpuShard`` is the product backend (the
C-ABI search plan); a test may pass any object with the same four methods.
"""
from __future__ import annotations

import math
import struct

import numpy as np

STATS_RESET = 100_000  # search.cpp:16


def shard_bounds(ncand: int, world: int, rank: int) -> tuple[int, int]:
    """Candidate range [s0, s1) of ``rank``: whole 100000-candidate segments,
    split as evenly as possible (earlier ranks take the remainder)."""
    nseg = (ncand + STATS_RESET - 1) // STATS_RESET
    base, extra = divmod(nseg, world)
    seg0 = rank * base + min(rank, extra)
    seg1 = seg0 + base + (1 if rank < extra else 0)
    return min(ncand, seg0 * STATS_RESET), min(ncand, seg1 * STATS_RESET)


def key_of(d: float) -> int:
    """Order-preserving int64 key of a non-negative double (its bit pattern)."""
    return struct.unpack("<q", struct.pack("<d", float(d)))[0]


def double_of(k: int) -> float:
    return struct.unpack("<d", struct.pack("<q", int(k)))[0]


INF_KEY = key_of(math.inf)


def all_reduce_min(t, group=None):
    """In-place MIN all-reduce.  Under gloo a CUDA tensor goes through a host
    copy (ordered on torch's current stream); NCCL reduces it in place."""
    import torch.distributed as dist
    if t.is_cuda and dist.get_backend(group) == "gloo":
        c = t.cpu()
        dist.all_reduce(c, op=dist.ReduceOp.MIN, group=group)
        t.copy_(c)
    else:
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)


def all_gather(t, world, group=None):
    """all_gather of one tensor per rank (host copies under gloo)."""
    import torch
    import torch.distributed as dist
    if t.is_cuda and dist.get_backend(group) == "gloo":
        t = t.cpu()
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return out


def lexicographic_min(records):
    """records: iterable of (found, distance, global_location)."""
    best = (False, math.inf, 0)
    for found, d, loc in records:
        if not found:
            continue
        if not best[0] or (d, loc) < (best[1], best[2]):
            best = (True, float(d), int(loc))
    return best


class GpuShard:
    """Backend over the C-ABI search plan for one shard (device-resident).

    The plan's context runs on torch's current stream of the key's device, so
    the kernels, the key's fill, the collectives on the key (NCCL waits on
    that stream) and any host copy of it are ordered with one another."""

    def __init__(self, ref_shard_dev_ptr: int, n_points: int, query, cfg, global_offset: int,
                 key_tensor, ctx=None):
        import torch

        from .api import Context, SearchPlan
        self.own_ctx = ctx is None
        self.ctx = ctx or Context(key_tensor.device.index or 0)
        self.ctx.set_stream(torch.cuda.current_stream(key_tensor.device).cuda_stream)
        self.plan = SearchPlan(ref_shard_dev_ptr, n_points, query, cfg, global_offset,
                               ctx=self.ctx)
        self.key = key_tensor
        self.plan.set_ub_key(key_tensor.data_ptr())

    @property
    def candidates(self) -> int:
        return self.plan.candidates

    def reset(self):
        self.key.fill_(INF_KEY)
        self.plan.reset()

    def prepare(self):
        self.plan.prepare()

    def run(self, begin: int, end: int):
        self.plan.run(begin, end)

    def result(self):
        return self.plan.result()

    def close(self):
        self.plan.close()
        if self.own_ctx:
            self.ctx.close()


class ShardedSearch:
    """Drive one rank's shard with best-so-far exchange between batches."""

    def __init__(self, backend, rank: int, world: int, batches: int = 8, group=None):
        self.backend = backend
        self.rank = rank
        self.world = world
        self.batches = max(1, int(batches))
        self.group = group

    def search(self):
        import torch.distributed as dist
        b = self.backend
        b.reset()
        b.prepare()
        nc = b.candidates
        edges = np.linspace(0, nc, self.batches + 1).astype(np.int64)
        if self.world > 1:
            # share the probe phase's best before the sweep starts
            all_reduce_min(b.key, self.group)
        for k in range(self.batches):
            b.run(int(edges[k]), int(edges[k + 1]))
            if self.world > 1:
                all_reduce_min(b.key, self.group)
        res = b.result()
        if self.world > 1:
            # a speculative search (csrc/capi.cu) only learns its exact best in
            # result(): every rank's key ends at the global exact minimum
            all_reduce_min(b.key, self.group)
        return self.finalize(res)

    def finalize(self, res):
        """Lexicographic (distance, lowest global index) across ranks."""
        import torch
        mine = (bool(res.best.found), float(res.best.distance_sq), int(res.best.location))
        if self.world == 1:
            return mine, res
        dev = self.backend.key.device
        t = torch.tensor([key_of(mine[1]) if mine[0] else INF_KEY, mine[2], int(mine[0])],
                         dtype=torch.int64, device=dev)
        out = all_gather(t, self.world, self.group)
        recs = [(bool(o[2].item()), double_of(o[0].item()), int(o[1].item())) for o in out]
        return lexicographic_min(recs), res


# --- batched NN1 (cfg5) over a database sharded across ranks -----

def db_shard_bounds(nd: int, world: int, rank: int) -> tuple[int, int]:
    """Database rows [d0, d1) of ``rank``: contiguous, as even as possible
    (earlier ranks take the remainder), so global index order = rank order."""
    base, extra = divmod(nd, world)
    d0 = rank * base + min(rank, extra)
    return d0, d0 + base + (1 if rank < extra else 0)


def merge_nn1(best_d, best_i, d, i):
    """Per-query lexicographic (distance, lowest global index) merge, in place.
    Entries with d = +inf carry no match."""
    take = np.isfinite(d) & ((d < best_d) | ((d == best_d) & (i < best_i)))
    best_d[take] = d[take]
    best_i[take] = i[take]


class GpuNN1Shard:
    """Backend over eapdtw_nn1_dev_cutoff: the queries and this rank's database
    rows resident on its GPU (torch float64 tensors, row-major)."""

    def __init__(self, queries_dev, db_shard_dev, window=None, ctx=None):
        from .api import default_context
        self.ctx = ctx or default_context()
        self.q = queries_dev
        self.db = db_shard_dev
        self.window = window
        self.nq, self.len = int(queries_dev.shape[0]), int(queries_dev.shape[1])
        self.rows = int(db_shard_dev.shape[0])
        self.cells = 0

    def run(self, b0: int, b1: int, cutoff):
        """(argmin local to [b0, b1), dist) of every query over rows [b0, b1),
        starting from the per-query cutoff tensor (device float64)."""
        import ctypes as C

        from . import _capi
        from .api import _window
        arg = np.empty(self.nq, dtype=np.uint64)
        dist = np.empty(self.nq)
        cells = C.c_uint64(0)
        import torch
        # the cutoff was written (H2D copy / all-reduce) on torch's stream
        torch.cuda.current_stream(self.q.device).synchronize()
        ptr = self.db.data_ptr() + b0 * self.len * 8
        _capi.check(_capi.lib.eapdtw_nn1_dev_cutoff(
            self.ctx.handle, C.c_void_p(self.q.data_ptr()), self.nq, C.c_void_p(ptr), b1 - b0,
            self.len, _window(self.window), C.c_void_p(cutoff.data_ptr()),
            arg.ctypes.data_as(C.POINTER(C.c_uint64)), dist.ctypes.data_as(C.POINTER(C.c_double)),
            C.byref(cells)))
        self.cells += cells.value
        return arg.astype(np.int64), dist


class ShardedNN1:
    """One rank's part of a sharded NN1: its database rows [offset, offset +
    rows) in ``batches`` batches; between batches the ranks all-reduce (MIN)
    the per-query best distance, which is the next batch's cutoff everywhere.
    The final answer per query is the lexicographic (distance, lowest global
    index) minimum over the ranks (one all-gather)."""

    def __init__(self, backend, rank: int, world: int, offset: int, batches: int = 4,
                 device=None, group=None):
        self.backend = backend
        self.rank, self.world = rank, world
        self.offset = int(offset)
        self.batches = max(1, int(batches))
        self.device = device
        self.group = group

    def search(self):
        import torch
        b = self.backend
        nq = b.nq
        best_d = np.full(nq, math.inf)
        best_i = np.zeros(nq, dtype=np.int64)
        cutoff = torch.full((nq,), math.inf, dtype=torch.float64, device=self.device)
        edges = np.linspace(0, b.rows, self.batches + 1).astype(np.int64)
        for k in range(self.batches):
            b0, b1 = int(edges[k]), int(edges[k + 1])
            if b1 > b0:
                arg, d = b.run(b0, b1, cutoff)
                merge_nn1(best_d, best_i, d, arg + self.offset + b0)
            cutoff = torch.from_numpy(best_d.copy()).to(cutoff.device)
            if self.world > 1:
                all_reduce_min(cutoff, self.group)
        if self.world == 1:
            return best_i, best_d
        mine = torch.stack([torch.from_numpy(best_d).view(torch.int64),
                            torch.from_numpy(best_i)]).to(cutoff.device)
        parts = all_gather(mine, self.world, self.group)
        out_d = np.full(nq, math.inf)
        out_i = np.zeros(nq, dtype=np.int64)
        for p in parts:  # rank order = global index order
            p = p.cpu()
            merge_nn1(out_d, out_i, p[0].view(torch.float64).numpy(), p[1].numpy())
        return out_i, out_d
