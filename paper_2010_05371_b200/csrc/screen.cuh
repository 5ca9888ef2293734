// screen.cuh -- lane-per-candidate DTW prefix screen (phase A).
//
// Most candidates that survive the lower bounds still die within a few DTW
// rows (at the converged threshold 50-85% of them are
// dead by row 16).  Evaluating those with a whole warp wastes the warp's
// pipeline fill; here each LANE runs the first R rows of its own candidate,
// 32 candidates per warp in lockstep, with the row kept in registers.
//
// The DP is evaluated in band coordinates e = i - j over a fixed window
// e in [e_lo, e_hi] (C slots).  Within a row, cell e depends on cell e+1 of the
// same row (left), e-1 (top) and e (diag) of the previous row, so one
// in-place sweep from high e to low e updates the row.  All lanes are on the
// same row, so the query value q[i - e] is a shared-memory broadcast.
//
// Soundness: the values are exact DP values (same rounding as warp_dtw) as
// long as every live cell stays inside the window.  The top of the window
// (e_hi = min(w, R-1)) is a true matrix/band edge; if a live cell ever sits on
// the low slot while e_lo is not the band edge, the lane is marked OVERFLOW
// and is never killed.  Otherwise a row with no live cell (tested on the high
// word: a superset of v <= ub) proves every later cell dead: KILL.
#pragma once
#include "dtw_warp.cuh"

namespace eapdtw_b200 {

// Returns true iff the candidate is proven to exceed ub (all cells of some row
// within the first `rows` rows are > ub).  c_of(r) gives the lane's row value
// for 1-based row r.  `active` lanes only; inactive lanes return false.
// Window [e_lo, e_lo + C) of band offsets for the first `rows` rows: the
// whole reachable range [max(-w, 1-m), min(w, rows-1)] when it fits, else C
// slots around the diagonal (holding e = 0, the corner).  e_hi is the last
// slot that can hold a matrix/band cell.
template <int C>
__device__ __forceinline__ void screen_window(int rows, int m, int w, int& e_lo, int& e_hi) {
  const int top = min(w, rows - 1);
  const int bot = max(-w, 1 - m);
  if (top - bot + 1 <= C) {
    e_lo = max(bot, top - C + 1);
  } else {
    e_lo = max(bot, -(C / 2));
    if (e_lo + C - 1 > top) e_lo = max(bot, top - C + 1);
  }
  e_hi = min(top, e_lo + C - 1);
}

template <int C, bool NARROW, class RowFn>
__device__ bool screen_prefix_impl(bool active, const RowFn& c_of, int rows, const double* qsp,
                                   int m, int w, double ub, unsigned& nrow_done) {
  const double INF = d_inf();
  int e_lo, e_hi;
  screen_window<C>(rows, m, w, e_lo, e_hi);
  const bool lo_is_edge = e_lo <= -w || e_lo <= 1 - m;
  const bool hi_is_edge = e_lo + C - 1 >= min(w, rows - 1);
  const int ub_hi = __double2hiint(fmin(ub, DBL_MAX));
  double V[C];
#pragma unroll
  for (int s = 0; s < C; ++s) V[s] = INF;
  // Row 0 holds the corner (0,0) = 0 at e = 0, the diag of cell (1,1).
  const int s0 = 0 - e_lo;
#pragma unroll
  for (int s = 0; s < C; ++s)
    if (s == s0) V[s] = 0.0;
  bool dead = false, overflow = false;
  const int nrows = min(rows, m);
  unsigned done = 0;
  for (int r = 1; r <= nrows; ++r) {
    const bool run = active && !dead && !overflow;
    done += run ? 1u : 0u;
    const double c = run ? c_of(r) : INF;
    // slot s <-> e = e_lo + s <-> column j = r - e; q pointer at slot 0
    const double* qr = qsp + (r - e_lo);
    bool any = false;
    double left = INF;  // cell above the window top: outside the band / matrix
#pragma unroll
    for (int s = C - 1; s >= 0; --s) {
      const double top = s > 0 ? V[s - 1] : INF;  // previous row, e - 1
      double nv = __dadd_rn(sq_cost(c, qr[-s]), dmin2(left, dmin2(top, V[s])));
      if (NARROW && e_lo + s > e_hi) nv = INF;  // slots past a narrow band's top
      V[s] = nv;
      left = nv;
      any |= __double2hiint(nv) <= ub_hi;
    }
    // a live cell on a window edge that is not a band/matrix edge: the live
    // region may leave the window, so this lane can no longer be killed
    if (!lo_is_edge && __double2hiint(V[0]) <= ub_hi) overflow = true;
    if (!hi_is_edge && __double2hiint(V[C - 1]) <= ub_hi) overflow = true;
    if (!any) dead = true;
    if (!__any_sync(kFull, active && !dead && !overflow)) break;
  }
  nrow_done = done;
  return active && dead && !overflow;
}

// Returns true iff the candidate is proven to exceed ub: every cell of some
// row among the first `rows` rows is > ub, with the live region never leaving
// the window.  c_of(r) gives the lane's (exact) row value for 1-based row r.
// nrow_done receives the rows this lane evaluated.
template <int C, class RowFn>
__device__ bool screen_prefix(bool active, const RowFn& c_of, int rows, const double* qsp, int m,
                              int w, double ub, unsigned& nrow_done) {
  int e_lo, e_hi;
  screen_window<C>(rows, m, w, e_lo, e_hi);
  if (e_lo + C - 1 > e_hi)
    return screen_prefix_impl<C, true>(active, c_of, rows, qsp, m, w, ub, nrow_done);
  return screen_prefix_impl<C, false>(active, c_of, rows, qsp, m, w, ub, nrow_done);
}

}  // namespace eapdtw_b200
