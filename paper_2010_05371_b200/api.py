"""Python mirror of the reference's public C++ API, executed on the B200.

Names, argument meaning and error behaviour follow the reference headers
(paths relative to /root/reference/proj):

* ``PRUNED``, ``is_pruned``, ``Series``          include/eapdtw/series.hpp:16-50
* ``Band``                                        include/eapdtw/dtw.hpp:16-23
* ``ea_pruned_dtw_windowed``, ``ea_pruned_dtw``,
  ``dtw_windowed``                                include/eapdtw/dtw.hpp:69-99
* ``Algo``, ``SearchConfig``, ``BestSoFar``,
  ``SearchReport``, ``SearchResult``,
  ``similarity_search``                           include/eapdtw/search.hpp:50-119

``std::invalid_argument`` maps to ``ValueError``.  Every compute call goes
through the C ABI of ``libeapdtw_b200.so`` (include/eapdtw_b200.h); there is
no CPU path.  Batched entry points with no reference counterpart (``pairwise``
for cfg1, ``nn1`` for cfg5, ``ShardedSearch`` for multi-GPU) sit beside them.
"""
from __future__ import annotations

import ctypes as C
import contextlib
import enum
import math
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from ._capi import check, lib

PRUNED = math.inf
UNBOUNDED_WINDOW = _capi.UNBOUNDED_WINDOW
_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)


def is_pruned(v: float) -> bool:
    """series.hpp:18"""
    return v == PRUNED


class Series:
    """Validated, non-empty, finite float64 samples (series.hpp:22-50)."""

    __slots__ = ("_x",)

    def __init__(self, samples):
        x = np.ascontiguousarray(np.asarray(samples, dtype=np.float64).reshape(-1))
        if x.size == 0:
            raise ValueError("Series: empty input")
        bad = ~np.isfinite(x)
        if bad.any():
            raise ValueError(f"Series: non-finite sample at index {int(np.argmax(bad))}")
        self._x = x

    def __len__(self):
        return self._x.size

    def length(self) -> int:
        return self._x.size

    def __getitem__(self, i):
        return self._x[i]

    def view(self) -> np.ndarray:
        return self._x

    def prefix(self, n: int) -> "Series":
        if n == 0 or n > self._x.size:
            raise ValueError("Series::prefix: bad length")
        return Series(self._x[:n].copy())


@dataclass(frozen=True)
class Band:
    """Sakoe-Chiba band (dtw.hpp:16-23)."""

    window: int = UNBOUNDED_WINDOW

    @staticmethod
    def unbounded() -> "Band":
        return Band(UNBOUNDED_WINDOW)

    @staticmethod
    def cells(w: int) -> "Band":
        return Band(int(w))

    def is_unbounded(self) -> bool:
        return self.window == UNBOUNDED_WINDOW


class Algo(enum.IntEnum):
    """search.hpp:56"""

    full = _capi.ALGO_FULL
    left_prune = _capi.ALGO_LEFT_PRUNE
    ea_pruned = _capi.ALGO_EA_PRUNED


@dataclass
class SearchConfig:
    """search.hpp:60-66"""

    query_length: int = 0
    window_ratio: float = 0.1
    algorithm: Algo = Algo.ea_pruned
    use_lower_bounds: bool = True
    tighten_ub: bool = True

    def to_c(self) -> _capi.SearchConfigC:
        return _capi.SearchConfigC(int(self.query_length), float(self.window_ratio),
                                   int(self.algorithm), int(bool(self.use_lower_bounds)),
                                   int(bool(self.tighten_ub)), 0)


@dataclass
class BestSoFar:
    """search.hpp:50-54"""

    location: int = 0
    distance_sq: float = PRUNED
    found: bool = False


@dataclass
class SearchReport:
    """search.hpp:68-77 (GPU semantics: see DESIGN.md, 'Counters')."""

    candidates_total: int = 0
    pruned_kim: int = 0
    pruned_keogh_eq: int = 0
    pruned_keogh_ec: int = 0
    dtw_calls: int = 0
    dtw_abandoned: int = 0
    dp_cells_evaluated: int = 0  # DP cells evaluated by every engine (dtw.cpp:28-33)
    elapsed_seconds: float = 0.0
    screen_cells_evaluated: int = 0  # ... of which the FP32 screening pass (GPU only)


@dataclass
class SearchResult:
    """search.hpp:79-82"""

    best: BestSoFar = field(default_factory=BestSoFar)
    report: SearchReport = field(default_factory=SearchReport)

    @staticmethod
    def from_c(r: _capi.SearchResultC) -> "SearchResult":
        return SearchResult(
            BestSoFar(int(r.location), float(r.distance_sq), bool(r.found)),
            SearchReport(int(r.candidates_total), int(r.pruned_kim), int(r.pruned_keogh_eq),
                         int(r.pruned_keogh_ec), int(r.dtw_calls), int(r.dtw_abandoned),
                         int(r.dp_cells_evaluated), float(r.elapsed_seconds),
                         int(r.screen_cells_evaluated)))


class Context:
    """Owns one ``eapdtw_ctx`` (device, stream, scratch buffers)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib.eapdtw_ctx_create(C.byref(h), int(device)))
        self.handle = h
        self.device = int(device)

    def close(self):
        if self.handle and not getattr(self, "_borrowed", False):
            lib.eapdtw_ctx_destroy(self.handle)
        self.handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: int | None):
        """Run on a CUDA stream handle (e.g. ``torch.cuda.current_stream().cuda_stream``).
        Handle 0 is the legacy default stream (torch's default stream), passed
        on as cudaStreamLegacy; None restores the context's own stream."""
        if stream_ptr is None:
            h = None
        elif int(stream_ptr) == 0:
            h = 1  # EAPDTW_STREAM_LEGACY (cudaStreamLegacy)
        else:
            h = int(stream_ptr)
        check(lib.eapdtw_ctx_set_stream(self.handle, C.c_void_p(h)))

    def set_option(self, name: str, value: int):
        """Engine option (include/eapdtw_b200.h: eapdtw_ctx_set_option)."""
        check(lib.eapdtw_ctx_set_option(self.handle, name.encode(), int(value)))

    def get_option(self, name: str) -> int:
        v = C.c_int64()
        check(lib.eapdtw_ctx_get_option(self.handle, name.encode(), C.byref(v)))
        return int(v.value)

    @contextlib.contextmanager
    def options(self, **kw):
        """Set options for the duration of a ``with`` block."""
        old = {k: self.get_option(k) for k in kw}
        try:
            for k, v in kw.items():
                self.set_option(k, v)
            yield self
        finally:
            for k, v in old.items():
                self.set_option(k, v)

    def synchronize(self):
        check(lib.eapdtw_ctx_synchronize(self.handle))

    @property
    def launches(self) -> int:
        return int(lib.eapdtw_ctx_launches(self.handle))

    def fp64_peak(self) -> float:
        v = C.c_double()
        check(lib.eapdtw_fp64_peak(self.handle, C.byref(v)))
        return v.value

    def fp32_peak(self) -> float:
        v = C.c_double()
        check(lib.eapdtw_fp32_peak(self.handle, C.byref(v)))
        return v.value

    @property
    def last_cells_f32(self) -> int:
        """FP32-screen share of the last nn1 call's cells."""
        return int(lib.eapdtw_ctx_last_cells_f32(self.handle))

    def spec_info(self) -> dict:
        """Speculative statistics of the last search (eapdtw_ctx_spec_info):
        measured deviation (< 0: no speculation), candidates re-evaluated
        exactly, and the process-wide count of searches redone on the chain."""
        dev, listed, fb = C.c_double(), C.c_uint64(), C.c_uint64()
        check(lib.eapdtw_ctx_spec_info(self.handle, C.byref(dev), C.byref(listed), C.byref(fb)))
        return {"deviation": dev.value, "listed": int(listed.value), "fallbacks": int(fb.value)}


class MultiDevice:
    """One host thread driving several GPUs through the C ABI
    (eapdtw_multi_*): a context per device and an NCCL communicator over them.
    The reference's similarity_search and the NN1 loop over all devices, with
    the best-so-far / per-query cutoffs all-reduced between batches."""

    def __init__(self, devices):
        devs = (C.c_int * len(devices))(*[int(d) for d in devices])
        h = C.c_void_p()
        check(lib.eapdtw_multi_create(C.byref(h), devs, len(devices)))
        self.handle = h
        self.devices = [int(d) for d in devices]

    def context(self, i: int) -> "Context":
        """The i-th device's context (borrowed: options apply to its searches)."""
        ctx = Context.__new__(Context)
        ctx.handle = C.c_void_p(lib.eapdtw_multi_context(self.handle, int(i)))
        ctx.device = self.devices[i]
        ctx._borrowed = True
        return ctx

    def similarity_search(self, reference, query, cfg: "SearchConfig | None" = None,
                          batches: int = 8) -> "SearchResult":
        cfg = cfg or SearchConfig()
        r, q = _as_f64(reference), _as_f64(query)
        c = cfg.to_c()
        out = _capi.SearchResultC()
        check(lib.eapdtw_multi_similarity_search(self.handle, _ptr(r), r.size, _ptr(q), q.size,
                                                 C.byref(c), int(batches), C.byref(out)))
        return SearchResult.from_c(out)

    def nn1(self, queries, db, band=None, batches: int = 4):
        qs = np.ascontiguousarray(np.asarray(queries, dtype=np.float64))
        d = np.ascontiguousarray(np.asarray(db, dtype=np.float64))
        nq, L = qs.shape
        arg = np.empty(nq, dtype=np.uint64)
        dist = np.empty(nq)
        cells = C.c_uint64(0)
        check(lib.eapdtw_multi_nn1(self.handle, _ptr(qs.reshape(-1)), nq, _ptr(d.reshape(-1)),
                                   d.shape[0], L, _window(band), int(batches),
                                   arg.ctypes.data_as(C.POINTER(C.c_uint64)), _ptr(dist),
                                   C.byref(cells)))
        return arg, dist, cells.value

    def close(self):
        if self.handle:
            lib.eapdtw_multi_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def total_launches() -> int:
    """Kernels launched by every context of this process (eapdtw_total_launches)."""
    return int(lib.eapdtw_total_launches())


_tls = threading.local()


def default_context(device: int = 0) -> Context:
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]


def _as_f64(x) -> np.ndarray:
    if isinstance(x, Series):
        return x.view()
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(-1))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _window(band) -> int:
    if band is None:
        return UNBOUNDED_WINDOW
    if isinstance(band, Band):
        return band.window
    return int(band)


# --- DTW kernels (dtw.hpp:69-99) --------------------------------------------

def ea_pruned_dtw_windowed(a, b, band, ub: float, cumulative_bound=(), *, ctx=None,
                           return_cells: bool = False):
    """dtw.hpp:93-99.  Exact DTW if it is <= ub, else PRUNED."""
    ctx = ctx or default_context()
    a, b = _as_f64(a), _as_f64(b)
    cb = _as_f64(cumulative_bound) if len(cumulative_bound) else None
    out = C.c_double()
    cells = C.c_uint64(0)
    check(lib.eapdtw_ea_pruned_dtw_windowed(
        ctx.handle, _ptr(a), a.size, _ptr(b), b.size, _window(band), float(ub),
        _ptr(cb) if cb is not None else None, 0 if cb is None else cb.size, C.byref(out),
        C.byref(cells)))
    return (out.value, cells.value) if return_cells else out.value


def ea_pruned_dtw(a, b, ub: float, *, ctx=None, return_cells: bool = False):
    """dtw.hpp:85-87 (unbounded band)."""
    return ea_pruned_dtw_windowed(a, b, Band.unbounded(), ub, ctx=ctx, return_cells=return_cells)


def dtw_windowed(a, b, band, *, ctx=None, return_cells: bool = False):
    """dtw.hpp:72-74: the plain banded DP (no abandoning)."""
    ctx = ctx or default_context()
    a, b = _as_f64(a), _as_f64(b)
    out = C.c_double()
    cells = C.c_uint64(0)
    check(lib.eapdtw_dtw_windowed(ctx.handle, _ptr(a), a.size, _ptr(b), b.size, _window(band),
                                  C.byref(out), C.byref(cells)))
    return (out.value, cells.value) if return_cells else out.value


def dtw_left_prune_windowed(a, b, band, ub: float, *, ctx=None, return_cells: bool = False):
    """dtw.hpp:76-83: left_prune_scan (dtw.cpp:130-182) -- pruning from the
    left only; exact value iff <= ub, else PRUNED."""
    ctx = ctx or default_context()
    a, b = _as_f64(a), _as_f64(b)
    out = C.c_double()
    cells = C.c_uint64(0)
    check(lib.eapdtw_dtw_left_prune_windowed(ctx.handle, _ptr(a), a.size, _ptr(b), b.size,
                                             _window(band), float(ub), C.byref(out),
                                             C.byref(cells)))
    return (out.value, cells.value) if return_cells else out.value


def dtw_left_prune(a, b, ub: float, *, ctx=None, return_cells: bool = False):
    """dtw.hpp:76-79 (unbounded band)."""
    return dtw_left_prune_windowed(a, b, Band.unbounded(), ub, ctx=ctx, return_cells=return_cells)


# --- lower bounds (lower_bounds.hpp:12-63), computed on the device ----------

@dataclass
class Envelope:
    """lower_bounds.hpp:15-21"""

    upper: np.ndarray
    lower: np.ndarray
    window: int = 0

    def length(self) -> int:
        return int(self.upper.size)


@dataclass
class BoundResult:
    """lower_bounds.hpp:42-46"""

    total: float = 0.0
    contributions: np.ndarray = field(default_factory=lambda: np.zeros(0))
    abandoned: bool = False


def compute_envelope(series, band, *, ctx=None) -> Envelope:
    """lower_bounds.hpp:25 -- sliding max/min over [j-w, j+w] clamped to the
    series (an unbounded band: the whole series)."""
    ctx = ctx or default_context()
    x = _as_f64(series)
    up = np.empty(x.size)
    lo = np.empty(x.size)
    w = _window(band)
    check(lib.eapdtw_compute_envelope(ctx.handle, _ptr(x), x.size, w, _ptr(up), _ptr(lo)))
    return Envelope(up, lo, x.size if w == UNBOUNDED_WINDOW else min(w, x.size))


def lb_kim_fl(q, c, *, ctx=None) -> float:
    """lower_bounds.hpp:33 / lower_bounds.cpp:51-55"""
    ctx = ctx or default_context()
    q, c = _as_f64(q), _as_f64(c)
    if q.size != c.size:
        raise ValueError("lb_kim_fl: length mismatch")
    out = C.c_double()
    check(lib.eapdtw_lb_kim_fl(ctx.handle, _ptr(q), _ptr(c), q.size, C.byref(out)))
    return out.value


def lb_keogh(env: Envelope, series, abandon_above: float = PRUNED, order=None, *,
             ctx=None) -> BoundResult:
    """lower_bounds.hpp:52-54 / lower_bounds.cpp:57-88 (visiting order, strict
    abandon)."""
    ctx = ctx or default_context()
    x = _as_f64(series)
    up, lo = _as_f64(env.upper), _as_f64(env.lower)
    if up.size != lo.size:
        raise ValueError("lb_keogh: malformed envelope")
    po = None
    if order is not None and len(order) > 0:
        o = np.ascontiguousarray(np.asarray(order, dtype=np.uint64))
        po = o.ctypes.data_as(C.POINTER(C.c_size_t))
        n_order = o.size
    else:
        n_order = 0
    if n_order not in (0, x.size):
        raise ValueError("lb_keogh: order/series length mismatch")
    total = C.c_double()
    contrib = np.zeros(x.size)
    ab = C.c_int(0)
    if up.size != x.size:
        raise ValueError("lb_keogh: length mismatch")
    check(lib.eapdtw_lb_keogh(ctx.handle, _ptr(up), _ptr(lo), _ptr(x), x.size,
                              float(abandon_above), po, C.byref(total), _ptr(contrib),
                              C.byref(ab)))
    return BoundResult(total.value, contrib, bool(ab.value))


def cumulative_bound(contributions, *, ctx=None) -> np.ndarray:
    """lower_bounds.hpp:63 / lower_bounds.cpp:90-103: cb[i] = sum_{j>i} c[j]."""
    ctx = ctx or default_context()
    c = _as_f64(contributions)
    cb = np.zeros(c.size)
    if c.size:
        check(lib.eapdtw_cumulative_bound(ctx.handle, _ptr(c), c.size, _ptr(cb)))
    return cb


@dataclass
class RunningStats:
    """search.hpp:16-42"""

    sum: float = 0.0
    sum_of_squares: float = 0.0
    count: int = 0

    @staticmethod
    def over(window) -> "RunningStats":
        x = _as_f64(window)
        s, q = C.c_double(), C.c_double()
        check(lib.eapdtw_running_stats_over(_ptr(x), x.size, C.byref(s), C.byref(q)))
        return RunningStats(s.value, q.value, x.size)

    def mean(self) -> float:
        return self.sum / float(self.count)

    def variance(self) -> float:
        m = self.mean()
        v = self.sum_of_squares / float(self.count) - m * m
        return v if v > 0.0 else 0.0

    def stddev(self) -> float:
        return math.sqrt(self.variance())


def znormalize_into(src, stats: RunningStats) -> np.ndarray:
    """search.hpp:46 / search.cpp:37-46 with the given statistics."""
    x = _as_f64(src)
    out = np.empty(x.size)
    check(lib.eapdtw_znormalize_into(_ptr(x), x.size, float(stats.sum),
                                     float(stats.sum_of_squares), int(stats.count), _ptr(out)))
    return out


def dtw_full(a, b, *, ctx=None):
    """dtw.hpp:69-70"""
    return dtw_windowed(a, b, Band.unbounded(), ctx=ctx)


def pairwise(a, b, band, ub=None, *, prune: bool = True, ctx=None):
    """cfg1 batch: ``out[p] = ea_pruned_dtw_windowed(a[p], b[p], band, ub[p])``.

    a, b: (npairs, len) float64 host arrays.  Returns (out, cells)."""
    ctx = ctx or default_context()
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    if a.shape != b.shape or a.ndim != 2:
        raise ValueError("pairwise: a and b must be (npairs, len) of equal shape")
    n, L = a.shape
    out = np.empty(n)
    cells = C.c_uint64(0)
    ubp = None
    if ub is not None:
        ub = np.ascontiguousarray(ub, dtype=np.float64)
        ubp = _ptr(ub)
    check(lib.eapdtw_pairwise(ctx.handle, _ptr(a), _ptr(b), n, L, _window(band), ubp,
                              int(prune), out.ctypes.data_as(_dp), C.byref(cells)))
    return out, cells.value


def nn1(queries, db, band=None, *, ctx=None):
    """cfg5 batch: per query the lowest-index argmin of
    ``ea_pruned_dtw_windowed(db[k], q, band, bsf)`` with a running cutoff.
    Returns (argmin uint64[nq], dist float64[nq], cells)."""
    ctx = ctx or default_context()
    q = np.ascontiguousarray(queries, dtype=np.float64)
    d = np.ascontiguousarray(db, dtype=np.float64)
    if q.ndim != 2 or d.ndim != 2 or q.shape[1] != d.shape[1]:
        raise ValueError("nn1: queries (nq, len) and db (nd, len) must share len")
    arg = np.empty(q.shape[0], dtype=np.uint64)
    dist = np.empty(q.shape[0])
    cells = C.c_uint64(0)
    check(lib.eapdtw_nn1(ctx.handle, _ptr(q), q.shape[0], _ptr(d), d.shape[0], q.shape[1],
                         _window(band), arg.ctypes.data_as(_u64p), dist.ctypes.data_as(_dp),
                         C.byref(cells)))
    return arg, dist, cells.value


# --- search (search.hpp:118-119) ---------------------------------------------

def similarity_search(reference, query, cfg: SearchConfig | None = None, *, ctx=None
                      ) -> SearchResult:
    """Nearest z-normalised subsequence of ``reference`` under windowed DTW.

    ``reference`` may be a Series or any float64 array (pinned host memory
    gives the fastest copy); its Series validation (series.hpp:24-31) runs on
    the device after the copy, the query's on the host."""
    ctx = ctx or default_context()
    cfg = cfg or SearchConfig()
    ref = _as_f64(reference)
    q = query.view() if isinstance(query, Series) else Series(query).view()
    res = _capi.SearchResultC()
    c = cfg.to_c()
    check(lib.eapdtw_similarity_search(ctx.handle, _ptr(ref), ref.size, _ptr(q), q.size,
                                       C.byref(c), C.byref(res)))
    return SearchResult.from_c(res)


def similarity_search_dev(ref_dev_ptr: int, n: int, query, cfg: SearchConfig, *, ctx=None
                          ) -> SearchResult:
    """Same as similarity_search with the reference already resident in HBM."""
    ctx = ctx or default_context()
    q = _as_f64(query)
    res = _capi.SearchResultC()
    c = cfg.to_c()
    check(lib.eapdtw_similarity_search_dev(ctx.handle, C.c_void_p(ref_dev_ptr), int(n), _ptr(q),
                                           q.size, C.byref(c), C.byref(res)))
    return SearchResult.from_c(res)


# --- trace (KernelTrace, dtw.hpp:42-57) ------------------------------------------

class TraceEventC(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("pad_", C.c_uint32), ("row", C.c_uint64),
                ("col", C.c_uint64), ("value", C.c_double)]


@dataclass
class KernelTrace:
    """dtw.hpp:42-57 with capture_cells = true: the evaluated cells
    (row, col, value) in evaluation order, discard points, pruning points and
    the abandon cell (None unless the kernel abandoned).  ``result`` is the
    traced call's return value."""

    cells_evaluated: int = 0
    cells: list = field(default_factory=list)
    discard_points: list = field(default_factory=list)
    pruning_points: list = field(default_factory=list)
    abandon_cell: tuple | None = None
    result: float = PRUNED


_TRACE_ALGO = {Algo.full: 0, Algo.left_prune: 1, Algo.ea_pruned: 2}


def trace(a, b, algo=Algo.ea_pruned, ub: float = PRUNED, band=None, *, ctx=None) -> KernelTrace:
    """Per-cell trace of one DTW on the device (the CLI's ``trace``,
    eapdtw_cli.cpp:91-108): ``dtw_full``/``dtw_windowed`` (algo full; ub
    ignored), ``dtw_left_prune(_windowed)`` or ``ea_pruned_dtw(_windowed)``,
    rows/cols 1-based.  A debugging path: one device thread."""
    ctx = ctx or default_context()
    a, b = _as_f64(a), _as_f64(b)
    code = _TRACE_ALGO[Algo(algo)]
    cap = (max(a.size, b.size) + 2) * (min(a.size, b.size) + 2) * 2 + 8
    ev = (TraceEventC * cap)()
    n = C.c_size_t(0)
    cells = C.c_uint64(0)
    out = C.c_double(0.0)
    check(lib.eapdtw_trace(ctx.handle, code, _ptr(a), a.size, _ptr(b), b.size, _window(band),
                           float(ub), ev, cap, C.byref(n), C.byref(cells), C.byref(out)))
    if n.value > cap:  # cannot happen (at most 2 events per cell + rows + 2)
        raise RuntimeError(f"trace: {n.value} events exceed the buffer ({cap})")
    t = KernelTrace(cells_evaluated=int(cells.value), result=float(out.value))
    for k in range(n.value):
        e = ev[k]
        if e.kind == 0:
            t.cells.append((int(e.row), int(e.col), float(e.value)))
        elif e.kind == 1:
            t.discard_points.append((int(e.row), int(e.col)))
        elif e.kind == 2:
            t.pruning_points.append((int(e.row), int(e.col)))
        else:
            t.abandon_cell = (int(e.row), int(e.col))
    return t


class DeviceSeries:
    """A reference series resident in HBM (``eapdtw_series``): uploaded and
    validated once, then searched any number of times -- the reference CLI's
    bench grid (eapdtw_cli.cpp:110-142) and multi-query searches."""

    def __init__(self, samples, *, ctx=None):
        self.ctx = ctx or default_context()
        x = samples.view() if isinstance(samples, Series) else _as_f64(samples)
        h = C.c_void_p()
        check(lib.eapdtw_series_upload(self.ctx.handle, _ptr(x), x.size, C.byref(h)))
        self.handle = h

    def __len__(self) -> int:
        return int(lib.eapdtw_series_length(self.handle))

    @property
    def device_ptr(self) -> int:
        return int(lib.eapdtw_series_device_ptr(self.handle))

    def search(self, query, cfg: SearchConfig | None = None, *, ctx=None) -> SearchResult:
        """similarity_search (search.hpp:118-119) against this reference, on
        ``ctx`` (default: the context that uploaded it; any context on the
        same device may search it, one host thread per context)."""
        cfg = cfg or SearchConfig()
        ctx = ctx or self.ctx
        q = query.view() if isinstance(query, Series) else Series(query).view()
        res = _capi.SearchResultC()
        c = cfg.to_c()
        check(lib.eapdtw_similarity_search_series(ctx.handle, self.handle, _ptr(q), q.size,
                                                  C.byref(c), C.byref(res)))
        return SearchResult.from_c(res)

    def close(self):
        if getattr(self, "handle", None):
            lib.eapdtw_series_free(self.handle)
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


# Worker contexts of concurrent grids, kept between calls: a fresh context
# allocates its scratch on first use (cudaMalloc/cudaFree synchronise the
# device), which would cost more than the overlap gains.
_pool_lock = threading.Lock()
_pool: dict = {}


def _pool_get(device: int) -> Context:
    with _pool_lock:
        free = _pool.setdefault(device, [])
        if free:
            return free.pop()
    return Context(device)


def _pool_put(ctx: Context) -> None:
    with _pool_lock:
        _pool.setdefault(ctx.device, []).append(ctx)


def search_grid(reference, query, lengths, ratios, algos=(Algo.ea_pruned,), *,
                use_lower_bounds: bool = True, tighten_ub: bool = True, ctx=None,
                concurrency: int = 1):
    """The reference CLI's bench grid (run_bench, eapdtw_cli.cpp:110-142):
    for each algorithm, query length (a prefix of ``query``) and window
    ratio, one similarity_search of the same reference.  The reference is
    uploaded to HBM once.  Yields ``(algo, length, ratio, SearchResult)`` in
    the reference's loop order (algo, then length, then ratio).

    ``concurrency`` > 1 runs the query lengths on that many contexts (CUDA
    streams, one host thread each) against the same resident series: one
    length's searches share their stats chain, and different lengths' latency-
    bound phases overlap.  Results are identical; they are yielded once all
    workers finish."""
    own = not isinstance(reference, DeviceSeries)
    ref = DeviceSeries(reference, ctx=ctx) if own else reference

    def cfg_of(algo, length, ratio):
        return SearchConfig(query_length=int(length), window_ratio=float(ratio),
                            algorithm=Algo(algo), use_lower_bounds=use_lower_bounds,
                            tighten_ub=tighten_ub and use_lower_bounds)
    try:
        workers = max(1, min(int(concurrency), len(lengths)))
        if workers == 1:
            for algo in algos:
                for length in lengths:
                    for ratio in ratios:
                        yield (Algo(algo), int(length), float(ratio),
                               ref.search(query, cfg_of(algo, length, ratio)))
            return
        import threading
        results, errors = {}, []

        def work(my_lengths):
            wctx = _pool_get(ref.ctx.device)
            try:
                for length in my_lengths:  # same m consecutively: stats cache hits
                    for algo in algos:
                        for ratio in ratios:
                            results[(Algo(algo), int(length), float(ratio))] = ref.search(
                                query, cfg_of(algo, length, ratio), ctx=wctx)
            except Exception as e:  # noqa: BLE001 -- re-raised in the caller
                errors.append(e)
            finally:
                _pool_put(wctx)
        threads = [threading.Thread(target=work, args=(list(lengths)[w::workers],))
                   for w in range(workers)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            raise errors[0]
        for algo in algos:
            for length in lengths:
                for ratio in ratios:
                    key = (Algo(algo), int(length), float(ratio))
                    yield key + (results[key],)
    finally:
        if own:
            ref.close()


def search_many(reference, queries, cfg: SearchConfig | None = None, *, ctx=None,
                concurrency: int = 4) -> list:
    """similarity_search of every query in ``queries`` against one reference
    uploaded to HBM once; returns the SearchResults in input order.  Queries
    are spread over ``concurrency`` pooled contexts (streams / host threads);
    each context caches the sliding stats of its last query length, so
    queries of equal length after a worker's first reuse them."""
    cfg = cfg or SearchConfig()
    queries = list(queries)
    own = not isinstance(reference, DeviceSeries)
    ref = DeviceSeries(reference, ctx=ctx) if own else reference
    try:
        workers = max(1, min(int(concurrency), len(queries)))
        if workers == 1:
            return [ref.search(q, cfg) for q in queries]
        import threading
        out, errors = [None] * len(queries), []

        def work(idx):
            wctx = _pool_get(ref.ctx.device)
            try:
                for k in idx:
                    out[k] = ref.search(queries[k], cfg, ctx=wctx)
            except Exception as e:  # noqa: BLE001 -- re-raised in the caller
                errors.append(e)
            finally:
                _pool_put(wctx)
        # equal lengths stay together within a worker (stats cache hits)
        order = sorted(range(len(queries)),
                       key=lambda k: len(queries[k]) if cfg.query_length == 0 else 0)
        threads = [threading.Thread(target=work, args=(order[w::workers],))
                   for w in range(workers)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            raise errors[0]
        return out
    finally:
        if own:
            ref.close()


class SearchPlan:
    """One shard of a (possibly multi-GPU) search: stepped C-ABI plan."""

    def __init__(self, ref_dev_ptr: int, n: int, query, cfg: SearchConfig, global_offset: int = 0,
                 *, ctx=None):
        self.ctx = ctx or default_context()
        q = _as_f64(query)
        self._q = q
        c = cfg.to_c()
        h = C.c_void_p()
        check(lib.eapdtw_search_plan_create(self.ctx.handle, C.c_void_p(ref_dev_ptr), int(n),
                                            _ptr(q), q.size, C.byref(c), int(global_offset),
                                            C.byref(h)))
        self.handle = h

    @property
    def candidates(self) -> int:
        return int(lib.eapdtw_search_plan_candidates(self.handle))

    @property
    def ub_key_ptr(self) -> int:
        return int(lib.eapdtw_search_plan_ub_key(self.handle))

    def reset(self):
        check(lib.eapdtw_search_plan_reset(self.handle))

    def set_ub_key(self, dev_ptr: int | None):
        """Use a caller-owned int64 device key (all-reduced MIN across ranks)."""
        check(lib.eapdtw_search_plan_set_ub_key(self.handle, C.c_void_p(dev_ptr or 0)))

    def prepare(self):
        check(lib.eapdtw_search_plan_prepare(self.handle))

    def run(self, begin: int, end: int):
        check(lib.eapdtw_search_plan_run(self.handle, int(begin), int(end)))

    def result(self) -> SearchResult:
        res = _capi.SearchResultC()
        check(lib.eapdtw_search_plan_result(self.handle, C.byref(res)))
        return SearchResult.from_c(res)

    def counters(self):
        out = (C.c_uint64 * 10)()
        check(lib.eapdtw_search_plan_counters(self.handle, out))
        keys = ["kim", "keogh_eq", "keogh_ec", "dtw_calls", "dtw_abandoned", "cells",
                "candidates", "engine_overflows", "screened", "cells_f32"]
        return dict(zip(keys, (int(x) for x in out)))

    def timings(self):
        ms = (C.c_float * 4)()
        check(lib.eapdtw_search_plan_timings(self.handle, ms))
        return {"stats": ms[0], "envelope": ms[1], "probe": ms[2], "sweep": ms[3]}

    def close(self):
        if self.handle:
            lib.eapdtw_search_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


# --- host helpers ------------------------------------------------------------

def sliding_stats(reference, m: int, *, ctx=None):
    """(mean, sd) of every length-m window, by the search's stats kernel
    (the RunningStats chain of similarity_search, search.cpp:156-168)."""
    ctx = ctx or default_context()
    r = _as_f64(reference)
    nc = r.size - int(m) + 1
    mean = np.empty(max(nc, 0))
    sd = np.empty(max(nc, 0))
    check(lib.eapdtw_sliding_stats(ctx.handle, _ptr(r), r.size, int(m), _ptr(mean), _ptr(sd)))
    return mean, sd


def sliding_envelope(reference, r: int, *, ctx=None):
    """(upper, lower): the sliding max / min of radius r over the whole series
    (compute_envelope's window, lower_bounds.cpp:9-49), by the search's
    envelope kernel."""
    ctx = ctx or default_context()
    x = _as_f64(reference)
    up = np.empty(x.size)
    lo = np.empty(x.size)
    check(lib.eapdtw_sliding_envelope(ctx.handle, _ptr(x), x.size, int(r), _ptr(up), _ptr(lo)))
    return up, lo


def znormalize(x) -> np.ndarray:
    """RunningStats::over + znormalize_into (search.cpp:25-46), bit-identical."""
    x = _as_f64(x)
    out = np.empty_like(x)
    check(lib.eapdtw_znormalize(_ptr(x), x.size, _ptr(out)))
    return out


def random_walk(n: int, seed: int) -> np.ndarray:
    """The reference's random_walk (io.cpp:124-137): uniform steps in [-0.5, 0.5)."""
    out = np.empty(int(n))
    check(lib.eapdtw_random_walk_uniform(int(n), int(seed), _ptr(out)))
    return out


def random_walk_normal(n: int, seed: int) -> np.ndarray:
    """Benchmark data: x0 = 0, increments i.i.d. N(0,1) (mt19937_64 + Box-Muller)."""
    out = np.empty(int(n))
    check(lib.eapdtw_random_walk_normal(int(n), int(seed), _ptr(out)))
    return out


def window_cells_for(ratio: float, m: int) -> int:
    """search.cpp:18-21"""
    w = math.floor(ratio * float(m))
    return 0 if w <= 0.0 else int(w)
