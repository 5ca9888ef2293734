// dtw_ad.cuh -- anti-diagonal warp engine for exactly-rounded pruned DTW.
//
// Same contract as warp_dtw (dtw_warp.cuh): the returned value is the full-DP
// value bit-for-bit when it is <= ub, +inf otherwise (sound pruning,
// SURVEY.md A.4); every cell is fl(fl(fl(a-b)^2) + min(left, top, diag)).
// Only the schedule differs.
//
// Cells are indexed by anti-diagonal d = i + j and band offset e = i - j.  The
// warp owns a window of 64*K consecutive offsets [E0, E0 + 64K): lane L holds
// e = E0 + 2KL + 2k + p (k < K, parity p).  One "pair" of steps updates
// anti-diagonal d0 (the p = 0 cells) and then d0 + 1 (p = 1), with
//
//   cell (d, e) <- left (d-1, e+1), top (d-1, e-1), diag (d-2, e)
//
// so every dependency stays in the lane's registers except one value per step
// that crosses to a neighbour lane (__shfl_up of the top for p = 0,
// __shfl_down of the left for p = 1).  All 32 lanes work on every step (no
// strip fill/drain), and the live region -- which follows the warping path,
// i.e. stays near a constant e -- rarely moves relative to the lanes.  Row and
// column values come from padded shared arrays (+inf outside the matrix).
//
// After each pair one ballot tells which lanes hold a live cell (tested on
// the high word: a superset of v <= ub, hence sound).  Two dead anti-diagonals
// in a row mean every later cell is dead: abandon.  A live cell in the lowest
// (highest) lane means the region may leave the window: the window shifts by
// one lane if the other end is dead; if both ends are live the region is
// wider than the window and the engine reports kAdOverflow -- the caller then
// re-runs the candidate with a wider window or the strip engine.
#pragma once
#include <type_traits>

#include "dtw_warp.cuh"

namespace eapdtw_b200 {

constexpr int kAdOk = 0;
constexpr int kAdOverflow = 1;

// Padding (elements) on each side of the row / column arrays: every row or
// column the window touches lies within 32K + 2 of a live cell (the window
// always holds one), and lazy row fills run up to 33 rows further.
__host__ __device__ constexpr int ad_pad(int K) { return 32 * K + 40; }

// rowsp : per-warp row-value buffer, indices [1 - ad_pad(K), lr + ad_pad(K)];
//         filled lazily (normalised rows; +inf outside [1, lr]).
// qsp   : padded column series, +inf outside [1, lc], same padding.
template <int K, class RawFn, class NormFn, class UbFn>
__device__ int warp_dtw_ad(const RawFn& rowraw, const NormFn& rownorm, int lr,
                           const double* __restrict__ qsp, int lc, int w, UbFn&& get_ub,
                           double* __restrict__ rowsp, double& result,
                           unsigned long long& cells) {
  const int lane = threadIdx.x & 31;
  const double INF = d_inf();
  constexpr int WN = 64 * K;  // window width in band offsets
  constexpr int PAD = ad_pad(K);

  // Band in e = i - j, intersected with the matrix.
  const bool banded = w < lr;
  const int emin = banded ? max(-w, 1 - lc) : 1 - lc;
  const int emax = banded ? min(w, lr - 1) : lr - 1;
  // Initial window: centred on e = 0 (the corner), clamped to the band.
  int E0 = -32 * K;
  if (E0 + WN - 1 > emax) E0 = emax - WN + 1;
  if (E0 < emin) E0 = emin;
  const bool covers = E0 <= emin && E0 + WN - 1 >= emax;  // window holds the whole band

  for (int k = lane; k < PAD; k += 32) rowsp[-k] = INF;  // rows 0, -1, ... (left pad)
  int filled = 0;  // rows [1, filled] (and +inf beyond lr) are valid in rowsp

  double V0[K], V1[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    V0[k] = INF;
    V1[k] = INF;
  }
  {  // anti-diagonal 0 holds the DP corner (0,0) = 0 at e = 0
    const int off = -E0;
    if (off / (2 * K) == lane) {
      const int k0 = (off % (2 * K)) >> 1;
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (k == k0) {
          if (off & 1) V1[k] = 0.0;
          else V0[k] = 0.0;
        }
    }
  }
  // The first pair's parity-0 anti-diagonal is the first d >= 1 with
  // d == E0 (mod 2); anti-diagonal 0 (or 1, all +inf) is the prior state.
  int d0 = ((E0 & 1) == 0) ? 2 : 1;
  const int dfin = lr + lc;
  double ub = fmin(get_ub(), DBL_MAX);
  double ub_pref = ub;
  int ub_hi = __double2hiint(ub);
  unsigned long long cnt = 0;

  // oob bit (2k+p): the cell's offset lies outside the band (possible only
  // when the window is not strictly inside it); recomputed after a shift.
  unsigned oob = 0;
  auto compute_oob = [&]() {
    oob = 0;
    if (!banded) return;
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const int e = E0 + 2 * K * lane + 2 * k + p;
        if (e > w || e < -w) oob |= 1u << (2 * k + p);
      }
  };
  compute_oob();
  bool masked = __any_sync(kFull, oob != 0);

  // One pair of anti-diagonals; MASK selects the band-edge variant.
  auto pair = [&](auto mask_tag, const double* crow, const double* qcol) -> bool {
    constexpr bool MASK = decltype(mask_tag)::value;
    double cr[K + 1], qv[K];
#pragma unroll
    for (int k = 0; k <= K; ++k) cr[k] = crow[k];
#pragma unroll
    for (int k = 0; k < K; ++k) qv[k] = qcol[-k];
    bool any = false;
    // parity 0: anti-diagonal d0
    double up = __shfl_up_sync(kFull, V1[K - 1], 1);
    if (lane == 0) up = INF;
    double N0[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const double top = k > 0 ? V1[k - 1] : up;
      double nv = __dadd_rn(sq_cost(cr[k], qv[k]), dmin2(V1[k], dmin2(top, V0[k])));
      if (MASK && ((oob >> (2 * k)) & 1u)) nv = INF;
      N0[k] = nv;
      any |= __double2hiint(nv) <= ub_hi;
    }
#pragma unroll
    for (int k = 0; k < K; ++k) V0[k] = N0[k];
    // parity 1: anti-diagonal d0 + 1
    double dn = __shfl_down_sync(kFull, V0[0], 1);
    if (lane == 31) dn = INF;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const double left = k < K - 1 ? V0[k + 1] : dn;
      double nv = __dadd_rn(sq_cost(cr[k + 1], qv[k]), dmin2(left, dmin2(V0[k], V1[k])));
      if (MASK && ((oob >> (2 * k + 1)) & 1u)) nv = INF;
      V1[k] = nv;
      any |= __double2hiint(nv) <= ub_hi;
    }
    return any;
  };

  // Evaluated cells are counted per window segment (between shifts): for each
  // of the lane's offsets e, the anti-diagonals d in [d_seg, d_last] with
  // d == e (mod 2) whose cell lies inside the matrix (and band).
  int d_seg = ((E0 & 1) == 0) ? 2 : 1;
  auto count_segment = [&](int d_last) {
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const int e = E0 + 2 * K * lane + 2 * k + p;
        if (banded && (e > w || e < -w)) continue;
        int lo = max(d_seg, max(2 + e, 2 - e));
        int hi = min(d_last, min(2 * lr - e, 2 * lc + e));
        if (((lo - e) & 1) != 0) ++lo;
        if (((hi - e) & 1) != 0) --hi;
        if (hi >= lo) cnt += static_cast<unsigned long long>(((hi - lo) >> 1) + 1);
      }
  };

  int status = kAdOk;
  for (;;) {
    // ---- per block of 4 pairs: lazy row fill and threshold refresh
    const int a0 = (d0 + E0) >> 1;  // exact: d0 == E0 (mod 2)
    if (filled < a0 + 32 * K + 6) {
      do {  // normalise the next 32 rows, one per lane
        const int r = filled + 1 + lane;
        rowsp[r] = r <= lr ? rownorm(rowraw(r - 1)) : INF;
        filled += 32;
      } while (filled < a0 + 32 * K + 6);
      __syncwarp();
    }
    ub = fmin(ub_pref, DBL_MAX);  // load issued one block earlier
    ub_hi = __double2hiint(ub);
    ub_pref = get_ub();
    const double* crow = rowsp + (a0 + K * lane);
    const double* qcol = qsp + (a0 - E0 - K * lane);
    bool stop = false, shifted = false;
#pragma unroll 1
    for (int t = 0; t < 4; ++t) {
      const bool any = masked ? pair(std::true_type{}, crow + t, qcol + t)
                              : pair(std::false_type{}, crow + t, qcol + t);
      if (dfin <= d0 + 1) {  // the final cell (lr, lc) is on this pair
        const int off = (lr - lc) - E0;
        double r = INF;
        if (off >= 0 && off < WN) {
          const int src = off / (2 * K), kk = (off % (2 * K)) >> 1;
          double mine = INF;
#pragma unroll
          for (int k = 0; k < K; ++k)
            if (k == kk) mine = (off & 1) ? V1[k] : V0[k];
          r = __shfl_sync(kFull, mine, src);
        }
        result = r <= ub ? r : INF;
        count_segment(d0 + 1);
        stop = true;
        break;
      }
      const unsigned lm = __ballot_sync(kFull, any);
      if (lm == 0u) {  // two consecutive dead anti-diagonals: nothing later can live
        result = INF;
        count_segment(d0 + 1);
        stop = true;
        break;
      }
      d0 += 2;
      if (!covers && ((lm & 1u) | (lm >> 31))) {
        const bool lo_live = (lm & 1u) && E0 > emin;
        const bool hi_live = (lm >> 31) && E0 + WN - 1 < emax;
        if ((lo_live && (lm >> 31)) || (hi_live && (lm & 1u))) {
          count_segment(d0 - 1);
          status = kAdOverflow;  // live region wider than the window
          stop = true;
          break;
        }
        if (lo_live || hi_live) {
          count_segment(d0 - 1);
          d_seg = d0;
#pragma unroll
          for (int k = 0; k < K; ++k) {
            const double x0 = lo_live ? __shfl_up_sync(kFull, V0[k], 1)
                                      : __shfl_down_sync(kFull, V0[k], 1);
            const double x1 = lo_live ? __shfl_up_sync(kFull, V1[k], 1)
                                      : __shfl_down_sync(kFull, V1[k], 1);
            const bool edge = lo_live ? lane == 0 : lane == 31;
            V0[k] = edge ? INF : x0;
            V1[k] = edge ? INF : x1;
          }
          E0 += lo_live ? -2 * K : 2 * K;
          compute_oob();
          masked = __any_sync(kFull, oob != 0);
          shifted = true;  // pointers change: restart the block
          break;
        }
      }
    }
    if (stop) break;
    (void)shifted;
  }
  for (int off = 16; off > 0; off >>= 1) cnt += __shfl_xor_sync(kFull, cnt, off);
  if (lane == 0) cells += cnt;
  return status;
}

}  // namespace eapdtw_b200
