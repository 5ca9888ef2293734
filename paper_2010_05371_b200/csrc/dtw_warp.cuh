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

#ifdef EAPDTW_PHASE_CLOCKS
__device__ unsigned long long g_dbg[16];  // strip steps, strips, per-bin DTWs / steps
#endif

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
// The record's distance only decreases, so one 8-byte load (single-copy
// atomic) rejects a d above it without touching the CAS; otherwise the loop
// starts from the guess {that distance, ~0} rather than a separately loaded
// index, which could tear into a (new d, old idx) pair and drop a lower-index
// tie: every comparison below uses a record the 16-byte CAS returned
// atomically (or the guess, which the CAS checks).  (A CAS for every result
// serialised the warm start's many finite results on one address: +1.9 ms.)
__device__ __forceinline__ void best_record_update(BestRecord* rec, double d,
                                                   unsigned long long idx) {
  const double d_now = *reinterpret_cast<volatile double*>(&rec->d);
  if (d > d_now) return;
  BestRecord cur{d_now, ~0ull};
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
//   rowraw(k)  : raw value of row k (0-based); loaded one strip ahead
//   rownorm(x) : row value used by the DP (identity, or the exact z-norm)
//   lr         : number of rows (the longer series, reference orient dtw.cpp:48-52)
//   qsp        : padded column series (see contract above)
//   w          : effective half window (effective_window, dtw.cpp:57-62)
//   get_ub()   : current threshold (warp-uniform); read one strip ahead
//   rowthr(u,i,i0): row i's threshold given the strip ub (identity without a cb);
//                 called once per strip by every lane (i0: the strip's first row)
//   rowbuf     : padded per-warp scratch (see contract above)
//   cells      : incremented (by lane 0) with the number of evaluated cells
// LEFT: pruning from the left only -- left_prune_scan (dtw.cpp:130-182): a
// row starts at the first live column of the row above (next_start) and is
// evaluated to the end of its band (no right border from dead cells); an
// all-dead row abandons.  Same result contract (exact iff <= ub, else +inf),
// more cells than EAPrunedDTW.
template <bool KILL, bool LEFT = false, class RawFn, class NormFn, class UbFn, class RowThrFn>
__device__ double warp_dtw(const RawFn& rowraw, const NormFn& rownorm, int lr,
                           const double* __restrict__ qsp, int lc, int w, UbFn&& get_ub,
                           RowThrFn&& rowthr, double* __restrict__ rowbuf,
                           unsigned long long& cells) {
  const int lane = threadIdx.x & 31;
  const double INF = d_inf();
  for (int k = lane; k <= lc + 1; k += 32) rowbuf[k] = k == 0 ? 0.0 : INF;
  // Band |i - j| <= w.  With w >= lr every (i, j) is inside it.
  const bool banded = w < lr;
  int lo = 0, hi = 0;  // live column range of the row held in rowbuf (row i0-1)
  int written = 0;     // highest rowbuf column that may hold a non-inf value
  unsigned cnt = 0;
  double ub_last = INF;
  double ub_next = get_ub();
  double x_next = lane < lr ? rowraw(lane) : 0.0;
  __syncwarp();

#ifdef EAPDTW_PHASE_CLOCKS
  int dbg_strips = 0;
  unsigned long long dbg_steps = 0;
#endif
  for (int i0 = 1; i0 <= lr; i0 += 32) {
#ifdef EAPDTW_PHASE_CLOCKS
    if (lane == 0) atomicAdd(&g_dbg[1], 1ull);
    ++dbg_strips;
#endif
    const double ub_strip = ub_next;
    const int i = i0 + lane;
    const bool active = i <= lr;
    const double x = x_next;
    if (i0 + 32 <= lr) {  // prefetch the next strip's threshold and row values
      ub_next = get_ub();
      x_next = i + 32 <= lr ? rowraw(i + 31) : 0.0;
    }
    // Clamp to the largest finite double so an infinite threshold never
    // makes an unreachable (+inf) cell "live".
    const double ub = fmin(rowthr(ub_strip, i, i0), DBL_MAX);
    const int wl = min(31, lr - i0);  // writer lane: the last row of the strip
    ub_last = __shfl_sync(kFull, ub, wl);
    const int ub_hi = __double2hiint(ub);
    // Inactive rows (past lr) see c = +inf: all their cells are +inf.
    const double c = active ? rownorm(x) : INF;
    const int jb = max(lo, 1);
    // Row i's band columns [bl, bh]; the lane is finished once j > bh.
    const int bl = banded ? max(1, i - w) : 1;
    const int bh = active ? (banded ? min(lc, i + w) : lc) : -1;
    double top_prev = (lane == 0 && jb - 1 >= lo && jb - 1 <= hi) ? rowbuf[jb - 1] : INF;
    int j = jb - lane;
    const double* qp = qsp + j;
    double* rp = rowbuf + j;
    double v = INF;
    // Finished lanes as a warp-uniform bit mask F (bit L = lane L).  Lane L
    // is finished once its cell is dead and its upstream row (lane L-1; for
    // lane 0 the row buffer, dead beyond column hi) was finished one step
    // earlier -- every later cell of the row is then dead -- or once it is
    // past its band.  Per step only the dead/alive ballot is per-lane; the
    // chain  F |= D & (F << 1 | lane-0 bit)  is uniform bit arithmetic, and
    // the past-band test runs once per 4 steps (a lane past its band is
    // noticed up to 3 columns late: cells computed exactly anyway).
    unsigned finmask = __ballot_sync(kFull, !active);
    int jf = active ? lc + 1 : j - 1;  // last column computed before finishing
    const bool writer = lane == wl;
    const bool is0 = lane == 0;
    const unsigned span = static_cast<unsigned>(bh - bl);
    int jr = j - bl;
    int j0 = jb;  // lane 0's column (warp-uniform)

    // One wavefront step at column j+u.  RANGE: apply the band test (a block
    // of 4 steps with every lane inside its band skips it).
    auto step = [&](auto range_tag, int u) {
      constexpr bool RANGE = decltype(range_tag)::value;
      const double sh = __shfl_up_sync(kFull, v, 1);
      const double top = is0 ? rp[u] : sh;
      const double diag = top_prev;
      top_prev = top;
      double nv = __dadd_rn(sq_cost(c, qp[u]), dmin2(v, dmin2(top, diag)));
      if (RANGE) nv = static_cast<unsigned>(jr + u) <= span ? nv : INF;
      bool dead;
      if (KILL) {
        dead = !(nv <= ub);
        nv = dead ? INF : nv;
      } else {
        dead = __double2hiint(nv) > ub_hi;  // nv >= 0: live is a superset of nv <= ub
      }
      if (writer) rp[u] = nv;
      v = nv;
      const unsigned dm = __ballot_sync(kFull, dead);
      if (!LEFT) finmask |= dm & ((finmask << 1) | (j0 + u > hi ? 1u : 0u));
    };

    for (;;) {
      const unsigned before = finmask;
      {
        step(std::true_type{}, 0);
        step(std::true_type{}, 1);
        step(std::true_type{}, 2);
        step(std::true_type{}, 3);
        finmask |= __ballot_sync(kFull, jr + 3 > static_cast<int>(span));
      }
      if (((finmask & ~before) >> lane) & 1u) jf = j + 3;
#ifdef EAPDTW_PHASE_CLOCKS
      dbg_steps += 4;
#endif
      if (finmask == kFull) break;
      j += 4;
      jr += 4;
      j0 += 4;
      qp += 4;
      rp += 4;
    }
    // All lanes advanced T = j - (jb - lane) + 4 steps; the writer's last
    // column is jb - wl + T - 1.  Anything it wrote in an earlier strip beyond
    // that is stale and must read as +inf.
    const int wend = jb - wl + (j - (jb - lane)) + 3;
    for (int k = max(wend + 1, 0) + lane; k <= written; k += 32) rowbuf[k] = INF;
    written = min(max(wend, 0), lc + 1);
    // Cells this lane evaluated inside its band before finishing.
    const int c0 = max(jb, bl), c1 = min(jf, bh);
    cnt += active && c1 >= c0 ? static_cast<unsigned>(c1 - c0 + 1) : 0u;
    __syncwarp();
    // Live range of the new last row, read back from rowbuf (columns [jb, wend]).
    const int wcol1 = min(wend, lc);
    const int ubl_hi = __double2hiint(ub_last);
    int nlo = INT_MAX, nhi = -1;
    for (int k0 = jb; k0 <= wcol1; k0 += 32) {
      const int k = k0 + lane;
      bool lv = false;
      if (k <= wcol1) {
        const double rv = rowbuf[k];
        lv = KILL ? rv <= ub_last : __double2hiint(rv) <= ubl_hi;
      }
      const unsigned bm = __ballot_sync(kFull, lv);
      if (bm) {
        if (nlo == INT_MAX) nlo = k0 + __ffs(bm) - 1;
        nhi = k0 + 31 - __clz(bm);
      }
    }
    if (nhi < 0) {  // the last row of the strip has no live cell: borders collided
      lo = -1;
      break;
    }
    lo = nlo;
    hi = nhi;
  }
#ifdef EAPDTW_PHASE_CLOCKS
  if (lane == 0) {
    atomicAdd(&g_dbg[0], dbg_steps);
    const int bin = dbg_strips <= 1 ? 0 : dbg_strips <= 2 ? 1 : dbg_strips <= 4 ? 2 : dbg_strips <= 8 ? 3 : dbg_strips <= 16 ? 4 : 5;
    atomicAdd(&g_dbg[2 + bin], 1ull);
    atomicAdd(&g_dbg[8 + bin], dbg_steps);
  }
#endif
  for (int off = 16; off > 0; off >>= 1) cnt += __shfl_xor_sync(kFull, cnt, off);
  if (lane == 0) cells += cnt;
  if (lo < 0 || hi != lc) return INF;
  const double r = rowbuf[lc];
  return r <= ub_last ? r : INF;
}


}  // namespace eapdtw_b200
