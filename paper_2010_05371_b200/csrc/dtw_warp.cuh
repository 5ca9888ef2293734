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
//     test_dtw.cpp:183-201 and :267-289.  Liveness inside the loop is tested
//     on the high 32 bits only (hi(v) <= hi(ub)), which keeps a SUPERSET of
//     the live cells (sound); the returned value is checked exactly.
//   * KILL=true replaces dead cells by +inf with an exact test; it is used
//     with the per-row thresholds of a cumulative bound (row_threshold,
//     dtw.cpp:81-86), whose thresholds grow with the row so a dead value must
//     not come back.
//
// Shared-memory contract (both arrays padded so no index is ever clamped):
//   qsp    : column series, qsp[j] for j in [1, lc]; qsp[j] = +inf for
//            j in [-kPadL, 0] and [lc+1, lc+kPadR]   (an out-of-range column
//            costs (c - inf)^2 = +inf, which masks the matrix edges for free)
//   rowbuf : lc+2 doubles plus the same padding; owned by the warp.
#pragma once
#include <cfloat>
#include <climits>
#include <cstdint>
#include <cuda_runtime.h>

namespace eapdtw_b200 {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kPadL = 32;  // left padding of qsp / rowbuf (doubles)
constexpr int kPadR = 40;  // right padding

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
//   qsp        : padded column series (see contract above)
//   w          : effective half window (effective_window, dtw.cpp:57-62)
//   get_ub()   : current threshold, re-read at every strip (warp-uniform)
//   rowthr(u,i): per-row threshold given the strip ub (identity without a cb)
//   rowbuf     : padded per-warp scratch (see contract above)
//   cells      : incremented (by lane 0) with the number of evaluated cells
template <bool KILL, class RowFn, class UbFn, class RowThrFn>
__device__ double warp_dtw(const RowFn& rowval, int lr, const double* __restrict__ qsp, int lc,
                           int w, UbFn&& get_ub, RowThrFn&& rowthr, double* __restrict__ rowbuf,
                           unsigned long long& cells) {
  const int lane = threadIdx.x & 31;
  const double INF = d_inf();
  for (int k = lane; k <= lc + 1; k += 32) rowbuf[k] = k == 0 ? 0.0 : INF;
  __syncwarp();
  // Band |i - j| <= w.  With w >= lr every (i, j) is inside it; the offset
  // d = j - i + w is then shifted so the same unsigned test always passes.
  const bool banded = w < lr;
  const int w2 = banded ? 2 * w : INT_MAX / 2;
  const int woff = banded ? w : INT_MAX / 4;
  int lo = 0, hi = 0;  // live column range of the row held in rowbuf (row i0-1)
  int written = 0;     // highest rowbuf column that may hold a non-inf value
  unsigned cnt = 0;
  double ub_last = INF;

  for (int i0 = 1; i0 <= lr; i0 += 32) {
    const double ub_strip = get_ub();
    const int i = i0 + lane;
    const bool active = i <= lr;
    // Clamp to the largest finite double so an infinite threshold never
    // makes an unreachable (+inf) cell "live".
    const double ub = fmin(rowthr(ub_strip, i), DBL_MAX);
    ub_last = __shfl_sync(kFull, ub, min(31, lr - i0));
    const int ub_hi = __double2hiint(ub);
    // Inactive rows (past lr) see c = +inf: all their cells are +inf.
    const double c = active ? rowval(i - 1) : INF;
    const int wl = min(31, lr - i0);  // writer lane: the last row of the strip
    const int jb = max(lo, 1);
    double top_prev = (lane == 0 && jb - 1 >= lo && jb - 1 <= hi) ? rowbuf[jb - 1] : INF;
    int j = jb - lane;
    int d = j - i + woff;
    double v = INF;
    bool fin = !active;
    unsigned finmask = __ballot_sync(kFull, fin);
    int newlo = -1, newhi = -1;
    int t = 0;
    for (;; ++t) {
      double top = __shfl_up_sync(kFull, v, 1);
      if (lane == 0) top = rowbuf[j];
      const double diag = top_prev;
      top_prev = top;
      const bool inb = static_cast<unsigned>(d) <= static_cast<unsigned>(w2);
      double nv = __dadd_rn(sq_cost(c, qsp[j]), dmin2(v, dmin2(top, diag)));
      nv = inb ? nv : INF;
      bool live;
      if (KILL) {
        live = nv <= ub;
        nv = live ? nv : INF;
      } else {
        live = __double2hiint(nv) <= ub_hi;  // nv >= 0: superset of nv <= ub
      }
      if (lane == wl) rowbuf[j] = nv;
      v = nv;
      cnt += (inb && !fin) ? 1u : 0u;
      const bool upf = lane == 0 ? (j > hi) : ((finmask >> (lane - 1)) & 1u);
      fin = fin || j > lc || d > w2 || (upf && !live);
      finmask = __ballot_sync(kFull, fin);
      const unsigned lm = __ballot_sync(kFull, live);
      if ((lm >> wl) & 1u) {
        const int jw = jb + t - wl;
        if (newlo < 0) newlo = jw;
        newhi = jw;
      }
      if (finmask == kFull) break;
      ++j;
      ++d;
    }
    // The writer lane stopped at column jb + t - wl; anything it wrote in an
    // earlier strip beyond that is stale and must read as +inf.
    const int wend = jb + t - wl;
    for (int k = max(wend + 1, 0) + lane; k <= min(written, lc + 1); k += 32) rowbuf[k] = INF;
    written = max(wend, 0);
    __syncwarp();
    if (newhi < 0) {  // the last row of the strip has no live cell: borders collided
      lo = -1;
      break;
    }
    lo = newlo;
    hi = newhi;
  }
  for (int off = 16; off > 0; off >>= 1) cnt += __shfl_xor_sync(kFull, cnt, off);
  if (lane == 0) cells += cnt;
  if (lo < 0 || hi != lc) return INF;
  const double r = rowbuf[lc];
  return r <= ub_last ? r : INF;
}

}  // namespace eapdtw_b200
