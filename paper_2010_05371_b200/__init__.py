"""paper_2010_05371_b200 -- B200-native (sm_100a) EAPrunedDTW subsequence search.

The hot path of arXiv 2010.05371 (z-normalised NN1 subsequence search under
windowed DTW: sliding stats -> LB_Kim -> LB_Keogh EQ/EC -> EAPrunedDTW ->
best-so-far) as hand-written CUDA behind a C ABI (include/eapdtw_b200.h),
with a Python mirror of the reference's C++ API in :mod:`.api`.
"""
from .api import (  # noqa: F401
    PRUNED,
    UNBOUNDED_WINDOW,
    Algo,
    Band,
    BestSoFar,
    Context,
    DeviceSeries,
    KernelTrace,
    SearchConfig,
    SearchPlan,
    SearchReport,
    SearchResult,
    Series,
    default_context,
    dtw_full,
    dtw_windowed,
    ea_pruned_dtw,
    ea_pruned_dtw_windowed,
    is_pruned,
    nn1,
    pairwise,
    random_walk,
    random_walk_normal,
    similarity_search,
    similarity_search_dev,
    sliding_envelope,
    sliding_stats,
    search_grid,
    search_many,
    trace,
    window_cells_for,
    znormalize,
)
from ._capi import LIB_PATH, EapdtwError  # noqa: F401
