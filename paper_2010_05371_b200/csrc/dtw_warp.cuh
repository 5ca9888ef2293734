// dtw_warp.cuh -- warp-cooperative, exactly-rounded pruned DTW for sm_100a.
//
// One warp evaluates one (row series, column series) pair.  It replaces the
// reference's ea_pruned_scan (proj/src/dtw.cpp:197-296) for the GPU:
//
//   * Rows are swept in strips of 32, lane L owning row i0+L.  The strip walks
//     the columns as a skewed wavefront: at step t lane L is at column
//     jb + t - L, so the top neighbour (i-1, j) is the value lane L-1 produced
//     one step earlier (one __shfl_up_sync of a double) and the diagonal is
//     the top received one step before that.  The left neighbour is the
//     lane's own previous value.  The last row of a strip is written to a
//     per-warp shared-memory row buffer that feeds lane 0 of the next strip.
//   * Every kept cell is fl(fl(fl(a-b)^2) + min(left, top, diag)) with the
//     explicitly rounded __dsub_rn/__dmul_rn/__dadd_rn, i.e. the same bits as
//     the reference's squared_cost + min3 (dtw.hpp:60-63, dtw.cpp:115) built
//     without contraction.
//   * Pruning is SOUND in the sense of SURVEY.md A.4: a cell is "live" iff its
//     value is <= ub; the live range of each row is bracketed by a left border
//     (first live column, the role of EAPrunedDTW's next_start) and a right
//     border found with a per-lane "finished" flag propagated by __ballot_sync
//     (the role of the pruning point pp, dtw.cpp:278-285).  Dead cells are
//     never needed: every path through a value > ub ends > ub because costs
//     are non-negative and IEEE addition is monotone.  Hence the returned
//     value is bit-identical to the full DP whenever that value is <= ub, and
//     +inf (PRUNED, series.hpp:16) otherwise -- the contract pinned by
//     test_dtw.cpp:183-201 and :267-289.
//   * KILL=true additionally replaces dead cells by +inf; it is used with the
//     per-row thresholds of a cumulative bound (row_threshold, dtw.cpp:81-86),
//     whose thresholds grow with the row so a dead value must not come back.
#pragma once
#include <cstdint>
#include <cfloat>
#include <climits>
#include <cuda_runtime.h>

namespace eapdtw_b200 {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ double d_inf() { return __longlong_as_double(0x7ff0000000000000LL); }

// squared_cost (dtw.hpp:60-63) with explicit rounding: no FMA contraction.
__device__ __forceinline__ double sq_cost(double a, double b) {
  const double d = __dsub_rn(a, b);
  return __dmul_rn(d, d);
}
__device__ __forceinline__ double dmin2(double a, double b) { return b < a ? b : a; }

// Global best-so-far as an order-preserving 64-bit key: for d >= 0 (and +inf)
// the IEEE bit pattern orders like the value, so atomicMin on the bits is a
// valid running threshold.
__device__ __forceinline__ double key_to_double(unsigned long long k) {
  return __longlong_as_double(static_cast<long long>(k));
}

struct alignas(16) BestRecord {  // exact (distance, lowest index) record
  double d;
  unsigned long long idx;
};

// Lexicographic (d, idx) minimum, 16-byte CAS (ATOMG.E.CAS.128 on sm_100a).
__device__ __forceinline__ void best_record_update(BestRecord* rec, double d,
                                                   unsigned long long idx) {
  BestRecord cur;
  cur.d = *reinterpret_cast<volatile double*>(&rec->d);
  cur.idx = *reinterpret_cast<volatile unsigned long long*>(&rec->idx);
  while (d < cur.d || (d == cur.d && idx < cur.idx)) {
    BestRecord want{d, idx};
    BestRecord seen = atomicCAS(rec, cur, want);
    if (seen.d == cur.d && seen.idx == cur.idx) break;
    cur = seen;
  }
}

__device__ __forceinline__ double load_ub(const unsigned long long* key) {
  return key_to_double(*reinterpret_cast<const volatile unsigned long long*>(key));
}

// Evaluate one pruned DTW with a warp.
//   rowval(k)  : value of row k (0-based), evaluated once per lane per strip
//   lr         : number of rows (the longer series, reference orient dtw.cpp:48-52)
//   qs         : column series in shared/global memory, 1-based (qs[1..lc])
//   w          : effective half window (effective_window, dtw.cpp:57-62)
//   get_ub()   : current threshold, re-read at every strip (warp-uniform)
//   rowthr(i)  : per-row threshold given the strip ub (identity without a cb)
//   rowbuf     : per-warp scratch, lc+1 doubles
//   cells      : incremented (by lane 0) with the number of evaluated cells
template <bool KILL, class RowFn, class UbFn, class RowThrFn>
__device__ double warp_dtw(const RowFn& rowval, int lr, const double* __restrict__ qs, int lc,
                           int w, UbFn&& get_ub, RowThrFn&& rowthr, double* __restrict__ rowbuf,
                           unsigned long long& cells) {
  const int lane = threadIdx.x & 31;
  const double INF = d_inf();
  int lo = 0, hi = 0;  // live column range of the row held in rowbuf (row i0-1)
  if (lane == 0) rowbuf[0] = 0.0;
  __syncwarp();
  double result = INF;
  unsigned long long ncell = 0;

  for (int i0 = 1; i0 <= lr; i0 += 32) {
    const double ub_strip = get_ub();
    const int i = i0 + lane;
    const bool active = i <= lr;
    // Clamp to the largest finite double so an infinite threshold never
    // makes an unreachable (+inf) cell "live".
    const double ub = fmin(rowthr(ub_strip, i), DBL_MAX);
    const double c = active ? rowval(i - 1) : 0.0;
    const int last_lane = min(31, lr - i0);
    const int jb = max(lo, 1);
    const int bl = max(max(1, i - w), jb);       // first computable column of row i
    const int bh = active ? min(lc, i + w) : -1;  // last band column of row i
    double left = INF;
    double v = INF;
    double top_prev = (lane == 0 && jb - 1 >= lo && jb - 1 <= hi) ? rowbuf[jb - 1] : INF;
    bool fin = !active;
    unsigned finmask = __ballot_sync(kFull, fin);
    int newlo = INT_MAX, newhi = -1;
    int j = jb - lane;

    for (;;) {
      const double shfl = __shfl_up_sync(kFull, v, 1);
      const bool up_fin = lane == 0 ? (j > hi) : ((finmask >> (lane - 1)) & 1u);
      double top = shfl;
      if (lane == 0) top = (j >= lo && j <= hi) ? rowbuf[j] : INF;
      const double diag = top_prev;
      top_prev = top;
      const bool inb = !fin && j >= bl && j <= bh;
      double nv = INF;
      if (inb) nv = __dadd_rn(sq_cost(c, qs[j]), dmin2(left, dmin2(top, diag)));
      const bool live = nv <= ub;
      if (KILL && !live) nv = INF;
      if (live) {
        newlo = min(newlo, j);
        newhi = j;
      }
      if (lane == last_lane && j == lc && live && i == lr) result = nv;
      if (lane == 31 && inb) rowbuf[j] = nv;
      left = nv;
      v = nv;
      fin = fin || j > bh || (up_fin && !live);
      const unsigned inbmask = __ballot_sync(kFull, inb);
      ncell += __popc(inbmask);
      finmask = __ballot_sync(kFull, fin);
      if (finmask == kFull) break;
      ++j;
    }
    __syncwarp();
    const int lo_n = __shfl_sync(kFull, newlo, last_lane);
    const int hi_n = __shfl_sync(kFull, newhi, last_lane);
    if (hi_n < 0) {  // the last row of the strip has no live cell: borders collided
      result = INF;
      break;
    }
    lo = lo_n;
    hi = hi_n;
  }
  if (lane == 0) cells += ncell;
  // Only the lane that owns row lr holds a finite result; warp-wide min.
  for (int off = 16; off > 0; off >>= 1) result = dmin2(result, __shfl_xor_sync(kFull, result, off));
  return result;
}

}  // namespace eapdtw_b200
