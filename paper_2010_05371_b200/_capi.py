"""ctypes binding of libeapdtw_b200.so (the C ABI declared in include/eapdtw_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2010_05371_b200``).  There is no fallback: if the library is
missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libeapdtw_b200.so")

EAPDTW_OK = 0
EAPDTW_EINVAL = 1
EAPDTW_ECUDA = 2
EAPDTW_ENOMEM = 3
EAPDTW_ENCCL = 4
UNBOUNDED_WINDOW = (1 << 64) - 1

ALGO_FULL = 0
ALGO_LEFT_PRUNE = 1
ALGO_EA_PRUNED = 2

_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)
_vp = C.c_void_p


class SearchConfigC(C.Structure):
    _fields_ = [
        ("query_length", C.c_size_t),
        ("window_ratio", C.c_double),
        ("algorithm", C.c_int32),
        ("use_lower_bounds", C.c_int32),
        ("tighten_ub", C.c_int32),
        ("reserved_", C.c_int32),
    ]


class SearchResultC(C.Structure):
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
        ("screen_cells_evaluated", C.c_uint64),
    ]


# (name, restype, argtypes) for every symbol include/eapdtw_b200.h declares.
SIGNATURES = [
    ("eapdtw_last_error", C.c_char_p, []),
    ("eapdtw_version", C.c_int, []),
    ("eapdtw_device_count", C.c_int, []),
    ("eapdtw_ctx_create", C.c_int, [C.POINTER(_vp), C.c_int]),
    ("eapdtw_ctx_destroy", C.c_int, [_vp]),
    ("eapdtw_ctx_set_stream", C.c_int, [_vp, _vp]),
    ("eapdtw_ctx_set_option", C.c_int, [_vp, C.c_char_p, C.c_int64]),
    ("eapdtw_ctx_get_option", C.c_int, [_vp, C.c_char_p, C.POINTER(C.c_int64)]),
    ("eapdtw_ctx_synchronize", C.c_int, [_vp]),
    ("eapdtw_ctx_launches", C.c_uint64, [_vp]),
    ("eapdtw_total_launches", C.c_uint64, []),
    ("eapdtw_ctx_last_cells_f32", C.c_uint64, [_vp]),
    ("eapdtw_ctx_spec_info", C.c_int, [_vp, C.POINTER(C.c_double), C.POINTER(C.c_uint64),
                                       C.POINTER(C.c_uint64)]),
    ("eapdtw_ea_pruned_dtw_windowed", C.c_int,
     [_vp, _dp, C.c_size_t, _dp, C.c_size_t, C.c_size_t, C.c_double, _dp, C.c_size_t, _dp,
      _u64p]),
    ("eapdtw_dtw_windowed", C.c_int,
     [_vp, _dp, C.c_size_t, _dp, C.c_size_t, C.c_size_t, _dp, _u64p]),
    ("eapdtw_dtw_left_prune_windowed", C.c_int,
     [_vp, _dp, C.c_size_t, _dp, C.c_size_t, C.c_size_t, C.c_double, _dp, _u64p]),
    ("eapdtw_compute_envelope", C.c_int, [_vp, _dp, C.c_size_t, C.c_size_t, _dp, _dp]),
    ("eapdtw_lb_kim_fl", C.c_int, [_vp, _dp, _dp, C.c_size_t, _dp]),
    ("eapdtw_lb_keogh", C.c_int,
     [_vp, _dp, _dp, _dp, C.c_size_t, C.c_double, C.POINTER(C.c_size_t), _dp, _dp,
      C.POINTER(C.c_int)]),
    ("eapdtw_cumulative_bound", C.c_int, [_vp, _dp, C.c_size_t, _dp]),
    ("eapdtw_running_stats_over", C.c_int, [_dp, C.c_size_t, _dp, _dp]),
    ("eapdtw_znormalize_into", C.c_int,
     [_dp, C.c_size_t, C.c_double, C.c_double, C.c_uint64, _dp]),
    ("eapdtw_trace", C.c_int,
     [_vp, C.c_int, _dp, C.c_size_t, _dp, C.c_size_t, C.c_size_t, C.c_double, _vp, C.c_size_t,
      C.POINTER(C.c_size_t), _u64p, _dp]),
    ("eapdtw_pairwise", C.c_int,
     [_vp, _dp, _dp, C.c_size_t, C.c_size_t, C.c_size_t, _dp, C.c_int, _dp, _u64p]),
    ("eapdtw_pairwise_dev", C.c_int,
     [_vp, _vp, _vp, C.c_size_t, C.c_size_t, C.c_size_t, _vp, C.c_int, _vp, _u64p]),
    ("eapdtw_similarity_search", C.c_int,
     [_vp, _dp, C.c_size_t, _dp, C.c_size_t, C.POINTER(SearchConfigC),
      C.POINTER(SearchResultC)]),
    ("eapdtw_similarity_search_dev", C.c_int,
     [_vp, _vp, C.c_size_t, _dp, C.c_size_t, C.POINTER(SearchConfigC),
      C.POINTER(SearchResultC)]),
    ("eapdtw_series_upload", C.c_int, [_vp, _dp, C.c_size_t, C.POINTER(_vp)]),
    ("eapdtw_series_device_ptr", _vp, [_vp]),
    ("eapdtw_series_length", C.c_size_t, [_vp]),
    ("eapdtw_series_free", C.c_int, [_vp]),
    ("eapdtw_similarity_search_series", C.c_int,
     [_vp, _vp, _dp, C.c_size_t, C.POINTER(SearchConfigC), C.POINTER(SearchResultC)]),
    ("eapdtw_search_plan_create", C.c_int,
     [_vp, _vp, C.c_size_t, _dp, C.c_size_t, C.POINTER(SearchConfigC), C.c_uint64,
      C.POINTER(_vp)]),
    ("eapdtw_search_plan_reset", C.c_int, [_vp]),
    ("eapdtw_search_plan_set_ub_key", C.c_int, [_vp, _vp]),
    ("eapdtw_search_plan_prepare", C.c_int, [_vp]),
    ("eapdtw_search_plan_candidates", C.c_size_t, [_vp]),
    ("eapdtw_search_plan_run", C.c_int, [_vp, C.c_size_t, C.c_size_t]),
    ("eapdtw_search_plan_ub_key", _vp, [_vp]),
    ("eapdtw_search_plan_result", C.c_int, [_vp, C.POINTER(SearchResultC)]),
    ("eapdtw_search_plan_timings", C.c_int, [_vp, C.POINTER(C.c_float)]),
    ("eapdtw_search_plan_counters", C.c_int, [_vp, _u64p]),
    ("eapdtw_search_plan_destroy", C.c_int, [_vp]),
    ("eapdtw_nn1", C.c_int,
     [_vp, _dp, C.c_size_t, _dp, C.c_size_t, C.c_size_t, C.c_size_t, _u64p, _dp, _u64p]),
    ("eapdtw_nn1_dev", C.c_int,
     [_vp, _vp, C.c_size_t, _vp, C.c_size_t, C.c_size_t, C.c_size_t, _u64p, _dp, _u64p]),
    ("eapdtw_nn1_dev_cutoff", C.c_int,
     [_vp, _vp, C.c_size_t, _vp, C.c_size_t, C.c_size_t, C.c_size_t, _vp, _u64p, _dp, _u64p]),
    ("eapdtw_sliding_stats", C.c_int, [_vp, _dp, C.c_size_t, C.c_size_t, _dp, _dp]),
    ("eapdtw_sliding_envelope", C.c_int, [_vp, _dp, C.c_size_t, C.c_size_t, _dp, _dp]),
    ("eapdtw_multi_create", C.c_int, [C.POINTER(_vp), C.POINTER(C.c_int), C.c_int]),
    ("eapdtw_multi_destroy", C.c_int, [_vp]),
    ("eapdtw_multi_device_count", C.c_int, [_vp]),
    ("eapdtw_multi_context", _vp, [_vp, C.c_int]),
    ("eapdtw_multi_similarity_search", C.c_int,
     [_vp, _dp, C.c_size_t, _dp, C.c_size_t, C.POINTER(SearchConfigC), C.c_int,
      C.POINTER(SearchResultC)]),
    ("eapdtw_multi_nn1", C.c_int,
     [_vp, _dp, C.c_size_t, _dp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_int, _u64p, _dp,
      _u64p]),
    ("eapdtw_znormalize", C.c_int, [_dp, C.c_size_t, _dp]),
    ("eapdtw_random_walk_uniform", C.c_int, [C.c_size_t, C.c_uint64, _dp]),
    ("eapdtw_random_walk_normal", C.c_int, [C.c_size_t, C.c_uint64, _dp]),
    ("eapdtw_fp64_peak", C.c_int, [_vp, _dp]),
    ("eapdtw_fp32_peak", C.c_int, [_vp, _dp]),
]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built; run __graft_entry__.build() (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


class EapdtwError(RuntimeError):
    """A CUDA-side failure (EAPDTW_ECUDA / EAPDTW_ENOMEM)."""


def check(rc: int) -> None:
    """Map status codes to exceptions: EINVAL -> ValueError (the reference's
    std::invalid_argument), everything else -> EapdtwError."""
    if rc == EAPDTW_OK:
        return
    msg = (lib.eapdtw_last_error() or b"").decode(errors="replace")
    if rc == EAPDTW_EINVAL:
        raise ValueError(msg)
    raise EapdtwError(f"eapdtw rc={rc}: {msg}")
