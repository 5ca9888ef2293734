"""ctypes loaders for the parity oracles.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline / reference legs may import this package, and only
as the checker or the timed CPU baseline -- never as the product path.

Two oracles live here:

* ``liboracle.so`` -- ``eapdtw_oracle.c``, a plain-C restatement of the
  reference algorithms (each function cites the reference file:line it follows).
* ``_ref/libeapdtw_ref.so`` -- the reference's own ``proj/src`` hot path,
  compiled unmodified (``oracle/Makefile``) behind ``ref_capi.cpp``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
UNBOUNDED = (1 << 64) - 1
_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)
_szp = C.POINTER(C.c_size_t)


class SearchResult(C.Structure):
    """Mirror of SearchResult/SearchReport (search.hpp:68-82), flattened."""

    _fields_ = [
        ("location", C.c_uint64),
        ("distance_sq", C.c_double),
        ("found", C.c_int32),
        ("pad_", C.c_int32),
        ("candidates_total", C.c_uint64),
        ("pruned_kim", C.c_uint64),
        ("pruned_keogh_eq", C.c_uint64),
        ("pruned_keogh_ec", C.c_uint64),
        ("dtw_calls", C.c_uint64),
        ("dtw_abandoned", C.c_uint64),
        ("dp_cells_evaluated", C.c_uint64),
        ("elapsed_seconds", C.c_double),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "pad_"}


def _arr(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    return x, x.ctypes.data_as(_dp)


def build(force: bool = False, ref: bool | None = None) -> None:
    """Compile liboracle.so (and _ref when /root/reference is present)."""
    targets = [os.path.join(HERE, "liboracle.so")]
    if ref is None:
        ref = os.path.isdir("/root/reference/proj/src")
    if ref:
        targets.append("ref")
    cmd = ["make", "-s", "-C", HERE] + (["-B"] if force else []) + targets
    subprocess.run(cmd, check=True)


class _Lib:
    def __init__(self, path, prefix):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        self.lib = C.CDLL(path)
        self.p = prefix
        L = self.lib
        f = getattr(L, prefix + "dtw")
        f.argtypes = [C.c_int, _dp, C.c_size_t, _dp, C.c_size_t, C.c_size_t, C.c_double, _dp,
                      C.c_size_t, _dp, _u64p]
        f.restype = C.c_int
        f = getattr(L, prefix + "similarity_search")
        f.argtypes = [_dp, C.c_size_t, _dp, C.c_size_t, C.c_size_t, C.c_double, C.c_int, C.c_int,
                      C.c_int, C.POINTER(SearchResult)]
        f.restype = C.c_int
        f = getattr(L, prefix + "compute_envelope")
        f.argtypes = [_dp, C.c_size_t, C.c_size_t, _dp, _dp]
        f.restype = C.c_int

    def dtw(self, algo, a, b, window=UNBOUNDED, ub=np.inf, cb=None):
        """algo: 0 dtw_windowed, 1 dtw_left_prune_windowed, 2 ea_pruned_dtw_windowed.

        Returns (value, cells).  Raises ValueError on the reference's
        std::invalid_argument conditions."""
        a, pa = _arr(a)
        b, pb = _arr(b)
        if cb is None:
            cb_arr, pcb, ncb = None, None, 0
        else:
            cb_arr, pcb = _arr(cb)
            ncb = len(cb_arr)
        out = C.c_double()
        cells = C.c_uint64(0)
        rc = getattr(self.lib, self.p + "dtw")(algo, pa, len(a), pb, len(b), window, ub, pcb, ncb,
                                               C.byref(out), C.byref(cells))
        if rc == 1:
            raise ValueError("invalid argument")
        if rc:
            raise RuntimeError(f"oracle rc={rc}")
        return out.value, cells.value

    def ea_pruned_dtw_windowed(self, a, b, window, ub=np.inf, cb=None):
        return self.dtw(2, a, b, window, ub, cb)[0]

    def dtw_windowed(self, a, b, window=UNBOUNDED):
        return self.dtw(0, a, b, window)[0]

    def similarity_search(self, ref, query, ratio, query_length=0, algo=2, use_lb=True,
                          tighten=True):
        ref, pr = _arr(ref)
        q, pq = _arr(query)
        res = SearchResult()
        rc = getattr(self.lib, self.p + "similarity_search")(
            pr, len(ref), pq, len(q), query_length, ratio, algo, int(use_lb), int(tighten),
            C.byref(res))
        if rc == 1:
            raise ValueError("invalid argument")
        if rc:
            raise RuntimeError(f"oracle rc={rc}")
        return res

    def compute_envelope(self, s, window):
        s, ps = _arr(s)
        up = np.empty_like(s)
        lo = np.empty_like(s)
        rc = getattr(self.lib, self.p + "compute_envelope")(ps, len(s), window,
                                                            up.ctypes.data_as(_dp),
                                                            lo.ctypes.data_as(_dp))
        if rc:
            raise ValueError("invalid argument")
        return up, lo


class Oracle(_Lib):
    """The C restatement (liboracle.so)."""

    def __init__(self):
        super().__init__(os.path.join(HERE, "liboracle.so"), "orc_")
        L = self.lib
        L.orc_sliding_stats.argtypes = [_dp, C.c_size_t, C.c_size_t, _dp, _dp]
        L.orc_pairwise.argtypes = [_dp, _dp, C.c_size_t, C.c_size_t, C.c_size_t, _dp, _dp, _u64p]
        L.orc_nn1.argtypes = [_dp, C.c_size_t, _dp, C.c_size_t, C.c_size_t, C.c_size_t, _u64p, _dp,
                              _u64p]
        L.orc_znormalize.argtypes = [_dp, C.c_size_t, _dp]
        L.orc_lb_keogh.argtypes = [_dp, _dp, _dp, C.c_size_t, C.c_double, _szp, _dp,
                                   C.POINTER(C.c_int)]
        L.orc_lb_keogh.restype = C.c_double
        L.orc_cumulative_bound.argtypes = [_dp, C.c_size_t, _dp]
        L.orc_random_walk_normal.argtypes = [C.c_size_t, C.c_uint64, _dp]

    def random_walk_normal(self, n, seed):
        """Benchmark data: x0 = 0, x[i+1] = x[i] + N(0,1) (mt19937_64 +
        Box-Muller), identical to the product's eapdtw_random_walk_normal."""
        out = np.empty(n)
        if self.lib.orc_random_walk_normal(n, seed, out.ctypes.data_as(_dp)):
            raise ValueError("invalid argument")
        return out

    def sliding_stats(self, ref, m):
        ref, pr = _arr(ref)
        n = len(ref) - m + 1
        mean = np.empty(n)
        sd = np.empty(n)
        rc = self.lib.orc_sliding_stats(pr, len(ref), m, mean.ctypes.data_as(_dp),
                                        sd.ctypes.data_as(_dp))
        if rc:
            raise ValueError("invalid argument")
        return mean, sd

    def znormalize(self, x):
        x, px = _arr(x)
        out = np.empty_like(x)
        if self.lib.orc_znormalize(px, len(x), out.ctypes.data_as(_dp)):
            raise ValueError("invalid argument")
        return out

    def pairwise(self, a, b, window, ub=None):
        a, pa = _arr(a)
        b, pb = _arr(b)
        n, L = a.shape
        out = np.empty(n)
        cells = C.c_uint64(0)
        if ub is not None:
            ub, pu = _arr(ub)
        else:
            pu = None
        rc = self.lib.orc_pairwise(pa, pb, n, L, window, pu, out.ctypes.data_as(_dp),
                                   C.byref(cells))
        if rc:
            raise ValueError("invalid argument")
        return out, cells.value

    def nn1(self, queries, db, window=UNBOUNDED):
        q, pq = _arr(queries)
        d, pd = _arr(db)
        nq, L = q.shape
        nd = d.shape[0]
        arg = np.empty(nq, dtype=np.uint64)
        dist = np.empty(nq)
        cells = C.c_uint64(0)
        rc = self.lib.orc_nn1(pq, nq, pd, nd, L, window, arg.ctypes.data_as(_u64p),
                              dist.ctypes.data_as(_dp), C.byref(cells))
        if rc:
            raise ValueError("invalid argument")
        return arg, dist, cells.value

    def lb_keogh(self, upper, lower, x, abandon_above=np.inf, order=None):
        upper, pu = _arr(upper)
        lower, pl = _arr(lower)
        x, px = _arr(x)
        contrib = np.empty_like(x)
        ab = C.c_int(0)
        po = None
        if order is not None:
            order = np.ascontiguousarray(order, dtype=np.uint64)
            po = order.ctypes.data_as(_szp)
        total = self.lib.orc_lb_keogh(pu, pl, px, len(x), abandon_above, po,
                                      contrib.ctypes.data_as(_dp), C.byref(ab))
        return total, contrib, bool(ab.value)

    def cumulative_bound(self, c):
        c, pc = _arr(c)
        cb = np.empty_like(c)
        if self.lib.orc_cumulative_bound(pc, len(c), cb.ctypes.data_as(_dp)):
            raise ValueError("invalid argument")
        return cb


class Reference(_Lib):
    """The unmodified reference library (oracle/_ref/libeapdtw_ref.so)."""

    PATH = os.path.join(HERE, "_ref", "libeapdtw_ref.so")

    def __init__(self):
        super().__init__(self.PATH, "ref_")
        L = self.lib
        L.ref_random_walk.argtypes = [C.c_size_t, C.c_uint64, _dp]
        L.ref_similarity_search_threads.argtypes = [_dp, C.c_size_t, _dp, C.c_size_t, C.c_size_t,
                                                    C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                                                    C.POINTER(SearchResult)]
        L.ref_pairwise_threads.argtypes = [_dp, _dp, C.c_size_t, C.c_size_t, C.c_size_t, _dp,
                                           C.c_int, _dp, _u64p]
        L.ref_nn1_threads.argtypes = [_dp, C.c_size_t, _dp, C.c_size_t, C.c_size_t, C.c_size_t,
                                      C.c_int, _u64p, _dp, _u64p]
        L.ref_znormalize.argtypes = [_dp, C.c_size_t, _dp]

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(cls.PATH)

    def random_walk(self, n, seed):
        out = np.empty(n)
        if self.lib.ref_random_walk(n, seed, out.ctypes.data_as(_dp)):
            raise ValueError("invalid argument")
        return out

    def znormalize(self, x):
        x, px = _arr(x)
        out = np.empty_like(x)
        if self.lib.ref_znormalize(px, len(x), out.ctypes.data_as(_dp)):
            raise ValueError("invalid argument")
        return out

    def similarity_search_threads(self, ref, query, ratio, threads, query_length=0, algo=2,
                                  use_lb=True, tighten=True):
        ref, pr = _arr(ref)
        q, pq = _arr(query)
        res = SearchResult()
        rc = self.lib.ref_similarity_search_threads(pr, len(ref), pq, len(q), query_length, ratio,
                                                    algo, int(use_lb), int(tighten), threads,
                                                    C.byref(res))
        if rc:
            raise ValueError(f"rc={rc}")
        return res

    def pairwise_threads(self, a, b, window, ub=None, threads=1):
        a, pa = _arr(a)
        b, pb = _arr(b)
        n, L = a.shape
        out = np.empty(n)
        cells = C.c_uint64(0)
        pu = None
        if ub is not None:
            ub, pu = _arr(ub)
        rc = self.lib.ref_pairwise_threads(pa, pb, n, L, window, pu, threads,
                                           out.ctypes.data_as(_dp), C.byref(cells))
        if rc:
            raise ValueError(f"rc={rc}")
        return out, cells.value

    def nn1_threads(self, queries, db, window=UNBOUNDED, threads=1):
        q, pq = _arr(queries)
        d, pd = _arr(db)
        nq, L = q.shape
        arg = np.empty(nq, dtype=np.uint64)
        dist = np.empty(nq)
        cells = C.c_uint64(0)
        rc = self.lib.ref_nn1_threads(pq, nq, pd, d.shape[0], L, window, threads,
                                      arg.ctypes.data_as(_u64p), dist.ctypes.data_as(_dp),
                                      C.byref(cells))
        if rc:
            raise ValueError(f"rc={rc}")
        return arg, dist, cells.value
