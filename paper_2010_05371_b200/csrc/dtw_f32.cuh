// dtw_f32.cuh -- FP32 screening pass in front of the exact FP64 pruned DTW.
//
// Almost every DTW the search starts is abandoned (cfg4: all but ~60 of 3.8 M
// tasks).  Proving "this candidate's DTW exceeds ub" does not need the exact
// FP64 value, only a sound bound, so the strip engine of dtw_warp.cuh is run
// here in FP32 (1 SHFL instead of 2 per step, FMNMX3 instead of 2 DSETP + 4
// selects, FP32 latency and the 128-lane FP32 pipe) against a threshold that
// is INFLATED by the worst-case FP32 error.  A candidate this pass abandons
// is abandoned by the reference too; every other candidate is re-evaluated by
// the exact FP64 engine (warp_dtw), so results keep the reference's bits.
//
// Soundness.  Let P be the argmin path of the FP64 DP
// (dtw.cpp:115 semantics) and S*(P) the real-arithmetic sum of its exact
// costs (c_i - q_j)^2 over the FP64 values c_i, q_j.  The FP64 DP value of a
// cell on P is the rounded sum of P's prefix, so S*(prefix) <= v64 (1 + e64),
// e64 = (2L + 8) 2^-53, L = lr + lc.  The FP32 pass uses cf = fl32(c') with
// c' = (x - mean) * rcp(sd) in FP64, |cf - c| <= u' |c|, u' = 2^-24 + 2^-49,
// and qf = fl32(q).  Each FP32 cost is <= (1+u)^3 (|c - q| + u'(|c|+|q|))^2 and
// the DP adds one rounding per cell, so by Minkowski's inequality the FP32
// value of the cell is <= (1+u)^(L+3) (sqrt(S*) + u' sqrt(L) (cmax + qmax))^2.
// Hence, with the FP64 engine's liveness threshold t of a row,
//     T32(t) = a (sqrt(t) + b)^2,   a >= (1 + e64)(1+u)^(L+4),
//                                   b >= u' sqrt(L) (cmax + qmax),
// evaluated with upward rounding, keeps every cell the FP64 engine would keep
// on P live.  cmax is enforced per strip: a row value with |cf| > cmax aborts
// the pass ("undecided", so the FP64 engine runs).
#pragma once
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cuda_runtime.h>

#include <type_traits>

#include "dtw_warp.cuh"


namespace eapdtw_b200 {

__device__ __forceinline__ float f_inf() { return __int_as_float(0x7f800000); }

// FP32 three-input minimum (FMNMX3 on sm_100a).
__device__ __forceinline__ float fmin3f(float a, float b, float c) {
  float d;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// T32 = a (sqrt(t) + b)^2 rounded up, clamped to FLT_MAX (an infinite or huge
// threshold never makes a +inf cell live).
struct F32Guard {
  float a, b;
};
__device__ __forceinline__ float f32_threshold(double t, F32Guard g) {
  const float tf = __double2float_ru(t);  // +inf when t > FLT_MAX
  const float s = __fadd_ru(__fsqrt_ru(tf), g.b);
  return fminf(__fmul_ru(__fmul_ru(s, s), g.a), FLT_MAX);
}

// Host: the guard constants for series lengths lr, lc and value bounds.
// vfac: each FP32 value is within vfac * u' of the FP64 one (1 for the DTW's
// rounded conversions; 4 for the Keogh terms' convert-multiply chain).
static inline F32Guard make_f32_guard(int lr, int lc, double cmax, double qmax,
                                      double vfac = 1.0) {
  const double L = static_cast<double>(lr) + lc;
  const double u = 0x1.0p-24, up = vfac * (0x1.0p-24 + 0x1.0p-49);
  const double e64 = (2.0 * L + 8.0) * 0x1.0p-53;
  // (1+u)^(L+4) <= exp((L+4) u); margins absorb the host's own rounding
  const double a = (1.0 + e64) * std::exp((L + 4.0) * u) * (1.0 + 0x1.0p-40);
  const double b = up * std::sqrt(L) * (cmax + qmax) * (1.0 + 0x1.0p-40) + 1e-18;
  F32Guard g;
  g.a = std::nextafter(static_cast<float>(a), FLT_MAX);
  g.b = std::nextafter(static_cast<float>(b), FLT_MAX);
  return g;
}

// The inverse: a lower bound on the exact value v given its FP32 sum x <= a
// (sqrt(v) + b)^2, i.e. v >= (sqrt(x / a) - b)^2 (rounded down; 0 if negative).
__device__ __forceinline__ float f32_lower(float x, F32Guard g) {
  const float s = __fsub_rd(__fsqrt_rd(__fdiv_rd(x, g.a)), g.b);
  return s > 0.0f ? __fmul_rd(s, s) : 0.0f;
}

// Per-step band test of banded pairs: off (cfg4 sweep 41.5 -> 39.4 ms, all
// parity tests green); see f32_strip_run.
#ifndef EAPDTW_F32_BANDTEST
#define EAPDTW_F32_BANDTEST 0
#endif
constexpr bool kF32BandTest = EAPDTW_F32_BANDTEST != 0;

constexpr int kF32Undecided = 1;  // a row value exceeded cmax: run the FP64 engine

// FP32 screening strip engine: the schedule of warp_dtw<false> (dtw_warp.cuh)
// on floats, resumable strip by strip (F32Strip holds the state between
// strips), so a caller can probe a pair in both directions (f32_probe_pair).
//   rowraw(k)  : raw value of row k (0-based); loaded one strip ahead
//   rownorm(x) : the row value as float (|value| <= cmax checked here)
//   qsp        : padded float column series (kPadL / kPadR of +inf)
//   rowthr(u, i, i0): float threshold of row i given the strip's ub (double)
//   rowbuf     : padded per-warp float scratch (its own per direction)
// REV: the pair is processed reversed -- row k of the pass is the caller's
// rowraw(k) (the caller reverses the rows), column j is qsp[lc + 1 - j].
// The DTW of the reversed pair is the same real sum over the reversed paths,
// and the band |i - j| <= w maps onto itself, so the screen's soundness
// argument (above) holds unchanged; only the evaluation order differs.
// BLK: wavefront steps per block of finish bookkeeping (ballots, finish
// masks, loop counters).  8 in the search and in NN1 (measured against 4:
// cfg4 -2%, cfg3-nolb -3%, cfg5 -9%, NN1 being ALU-pipe bound; 16: cfg5 +1%):
// the per-block work is amortised over twice the cells at the cost of up to 4
// more steps at a strip's end.
// UNB: also instantiate the unbounded-band path without the per-step band
// test (NN1); the search kernel keeps one copy of the step loop (i-cache:
// the second copy cost the cfg4 sweep ~4 ms).
// Warp-uniform, so a caller can keep it in memory between strip runs.
struct F32Strip {
  int lo, hi;     // live column range of the row held in rowbuf (row i0 - 1); lo < 0: dead
  int written;    // highest rowbuf column that may hold a non-inf value
  int i0;         // first row of the next strip
  unsigned cnt;   // evaluated cells (warp total)
  float ub_last;  // threshold of the row held in rowbuf
  float slack;    // ub_last - min of that row (after a strip run with want_slack)
  float vmin;     // that minimum (over every cell of the row the strip evaluated)
  int status;     // 0, or kF32Undecided
};

__device__ inline void f32_strip_begin(F32Strip& s, int lc, float* __restrict__ rowbuf) {
  const int lane = threadIdx.x & 31;
  const float INF = f_inf();
  for (int k = lane; k <= lc + 1; k += 32) rowbuf[k] = k == 0 ? 0.0f : INF;
  s.lo = 0;
  s.hi = 0;
  s.written = 0;
  s.i0 = 1;
  s.cnt = 0;
  s.ub_last = INF;
  s.slack = INF;
  s.vmin = 0.0f;
  s.status = 0;
  __syncwarp();
}

// Runs up to max_strips strips (all: lr).  Stops early when the borders
// collide (s.lo < 0: proven > ub) or a row value exceeds cmax.
template <int BLK, bool UNB, bool REV, class RawFn, class NormFn, class UbFn, class RowThrFn>
__device__ void f32_strip_run(F32Strip& s, int max_strips, bool want_slack, const RawFn& rowraw,
                              const NormFn& rownorm, int lr, const float* __restrict__ qsp, int lc,
                              int w, float cmax, UbFn&& get_ub, RowThrFn&& rowthr,
                              float* __restrict__ rowbuf) {
  const int lane = threadIdx.x & 31;
  const float INF = f_inf();
  const bool banded = w < lr;
  int lo = s.lo, hi = s.hi, written = s.written;
  unsigned cnt = 0;
  float ub_last = s.ub_last;
  int i0 = s.i0;
  // the first strip's threshold and row values (then one strip ahead)
  double ub_next = get_ub();
  double x_next = i0 + lane <= lr ? rowraw(i0 - 1 + lane) : 0.0;
#ifdef EAPDTW_PHASE_CLOCKS
  int dbg_strips = 0;
  unsigned long long dbg_steps = 0;
#endif

  for (int ns = 0; ns < max_strips && i0 <= lr && lo >= 0; ++ns, i0 += 32) {
#ifdef EAPDTW_PHASE_CLOCKS
    if (lane == 0) atomicAdd(&g_dbg[1], 1ull);
    ++dbg_strips;
#endif
    const double ub_strip = ub_next;
    const int i = i0 + lane;
    const bool active = i <= lr;
    const double x = x_next;
    if (i0 + 32 <= lr) {
      ub_next = get_ub();
      x_next = i + 32 <= lr ? rowraw(i + 31) : 0.0;
    }
    const float ub = rowthr(ub_strip, i, i0);
    const int wl = min(31, lr - i0);
    ub_last = __shfl_sync(kFull, ub, wl);
    const float c = active ? rownorm(x) : INF;
    if (__any_sync(kFull, active && !(fabsf(c) <= cmax))) {
      s.status = kF32Undecided;
      break;
    }
    const int jb = max(lo, 1);
    const int bl = banded ? max(1, i - w) : 1;
    const int bh = active ? (banded ? min(lc, i + w) : lc) : -1;
    float top_prev = (lane == 0 && jb - 1 >= lo && jb - 1 <= hi) ? rowbuf[jb - 1] : INF;
    int j = jb - lane;
    // column j of the pass: qsp[j] forward, qsp[lc + 1 - j] reversed
    const float* qp = REV ? qsp + (lc + 1 - j) : qsp + j;
    float* rp = rowbuf + j;
    float v = INF;
    unsigned finmask = __ballot_sync(kFull, !active);
    int jf = active ? lc + 1 : j - 1;
    const bool writer = lane == wl;
    const bool is0 = lane == 0;
    const unsigned span = static_cast<unsigned>(bh - bl);
    int jr = j - bl;
    int j0 = jb;

    // One wavefront step at column j+u (RANGE: with the band test).  Every
    // lane loads its row-buffer cell (only lane 0 uses it as its top): one
    // select instead of a predicated load and two moves.  Deadness is
    // accumulated over the block of steps (alld).  The cost and the
    // accumulation are one FFMA (d*d + min, one rounding where the T32 bound
    // allows two).
    // The block's column values and row-buffer cells are loaded up front
    // (qb, rbb): the compiler cannot move a load above the writer's store to
    // the same shared array, and the per-step load latency was the largest
    // stall of the loop (ncu).  Reading rowbuf early is safe: the writer
    // (lane wl >= 0) writes column j0 - wl + u at step u, lane 0 reads column
    // j0 + u, so a column is read before it is written.
    float qb[BLK], rbb[BLK];
    auto step = [&](auto range_tag, int u, bool& alld) {
      constexpr bool RANGE = decltype(range_tag)::value;
      const float sh = __shfl_up_sync(kFull, v, 1);
      const float top = is0 ? rbb[u] : sh;
      const float diag = top_prev;
      top_prev = top;
      float d = __fsub_rn(c, qb[u]);
      // the band test masks the difference (off the step's dependency
      // chain): inf * inf + min(...) = +inf
      if (RANGE) d = static_cast<unsigned>(jr + u) <= span ? d : INF;
      const float nv = __fmaf_rn(d, d, fmin3f(v, top, diag));
      if (writer) rp[u] = nv;
      v = nv;
      alld = alld && nv > ub;
    };

    for (;;) {
      const unsigned before = finmask;
      bool alld = true;
#pragma unroll
      for (int u = 0; u < BLK; ++u) {
        qb[u] = REV ? qp[-u] : qp[u];
        rbb[u] = rp[u];
      }
      // Unbounded band: the band is the whole row, and the +inf padding of
      // qsp (dtw_warp.cuh) already makes every out-of-range column cost +inf,
      // so the per-step band test (3 ALU-pipe ops per cell) is dropped.
      // EAPDTW_F32_BANDTEST=0: no per-step band test for banded pairs
      // either.  Cells beyond a lane's band edges then take real costs: the
      // DP of a wider band, a lower bound of the banded one, so an abandon is
      // still sound (the exact engine applies the band); lanes still finish
      // at their right band edge (finmask below).
      if ((UNB && !banded) || !kF32BandTest) {
#pragma unroll
        for (int u = 0; u < BLK; ++u) step(std::false_type{}, u, alld);
      } else {
#pragma unroll
        for (int u = 0; u < BLK; ++u) step(std::true_type{}, u, alld);
      }
      // Finished lanes, once per block (conservative): lane L is finished
      // after step u if it was dead in all BLK steps and lane L-1 (lane 0:
      // the row buffer, dead beyond column hi) was finished after step u-1.
      // BLK chained updates, one per step, with the block's all-dead mask D.
      const unsigned D = __ballot_sync(kFull, alld);
      if constexpr (BLK == 8 || BLK == 16) {
        // Closed form of the BLK chained updates (same result; identity
        // checked in tests/test_finish_mask.py): a lane of D finishes if a
        // run of D lanes joins it to a seed within reach.  Seeds: lanes just
        // above a finished lane (reach BLK-1 more lanes), and lane 0 once
        // the row buffer is dead, from step u0 = hi - j0 + 1 on (reach
        // BLK-1-u0).  Bounded propagation through D by doubling (1 + 2 + 4
        // [+ 8]).  Measured: cfg4 -3%, cfg3-nolb -2%, cfg5 -7.5% (ALU-pipe work).
        unsigned G = (finmask << 1) & D;
        unsigned P = D;
#pragma unroll
        for (int sh = 1; sh < BLK; sh *= 2) {
          G |= P & (G << sh);
          if (2 * sh < BLK) P &= P << sh;
        }
        const int u0 = max(0, hi - j0 + 1);
        if (u0 < BLK) {
          const int run = __ffs(~D) - 1;  // D's trailing ones (-1: all 32)
          const int k = min(run < 0 ? 32 : run, BLK - u0);
          G |= k >= 32 ? kFull : ((1u << k) - 1u);
        }
        finmask |= G;
      } else {
#pragma unroll
        for (int u = 0; u < BLK; ++u) finmask |= D & ((finmask << 1) | (j0 + u > hi ? 1u : 0u));
      }
      finmask |= __ballot_sync(kFull, jr + (BLK - 1) > static_cast<int>(span));
      if (((finmask & ~before) >> lane) & 1u) jf = j + (BLK - 1);
#ifdef EAPDTW_PHASE_CLOCKS
      dbg_steps += BLK;
#endif
      if (finmask == kFull) break;
      j += BLK;
      jr += BLK;
      j0 += BLK;
      qp += REV ? -BLK : BLK;
      rp += BLK;
    }
    const int wend = jb - wl + (j - (jb - lane)) + (BLK - 1);
    for (int k = max(wend + 1, 0) + lane; k <= written; k += 32) rowbuf[k] = INF;
    written = min(max(wend, 0), lc + 1);
    const int c0 = max(jb, bl), c1 = min(jf, bh);
    cnt += active && c1 >= c0 ? static_cast<unsigned>(c1 - c0 + 1) : 0u;
    __syncwarp();
    const int wcol1 = min(wend, lc);
    int nlo = INT_MAX, nhi = -1;
    float vmin = INF;
    for (int k0 = jb; k0 <= wcol1; k0 += 32) {
      const int k = k0 + lane;
      const float rv = k <= wcol1 ? rowbuf[k] : INF;
      vmin = fminf(vmin, rv);
      const unsigned bm = __ballot_sync(kFull, rv <= ub_last);
      if (bm) {
        if (nlo == INT_MAX) nlo = k0 + __ffs(bm) - 1;
        nhi = k0 + 31 - __clz(bm);
      }
    }
    if (want_slack) {
      for (int off = 16; off > 0; off >>= 1) vmin = fminf(vmin, __shfl_xor_sync(kFull, vmin, off));
      s.slack = ub_last - vmin;
      s.vmin = vmin;
    }
    if (nhi < 0) {
      lo = -1;
      i0 += 32;
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
  s.lo = lo;
  s.hi = hi;
  s.written = written;
  s.i0 = i0;
  s.cnt += cnt;
  s.ub_last = ub_last;
}

// The pass's outcome: +inf if proven > ub (or undecided: status), else the
// FP32 value of the final cell.  Adds the evaluated cells to `cells`.
__device__ inline float f32_strip_end(F32Strip& s, int lc, const float* __restrict__ rowbuf,
                                      unsigned long long& cells, int& status) {
  const int lane = threadIdx.x & 31;
  if (lane == 0) cells += s.cnt;
  s.cnt = 0;
  __syncwarp();
  status = s.status;
  if (s.status != 0 || s.lo < 0 || s.hi != lc) return f_inf();
  const float r = rowbuf[lc];
  return r <= s.ub_last ? r : f_inf();
}

// One whole FP32 pass, forward.
template <int BLK = 4, bool UNB = false, class RawFn, class NormFn, class UbFn, class RowThrFn>
__device__ float warp_dtw_f32(const RawFn& rowraw, const NormFn& rownorm, int lr,
                              const float* __restrict__ qsp, int lc, int w, float cmax,
                              UbFn&& get_ub, RowThrFn&& rowthr, float* __restrict__ rowbuf,
                              unsigned long long& cells, int& status) {
  F32Strip s;
  f32_strip_begin(s, lc, rowbuf);
  f32_strip_run<BLK, UNB, false>(s, lr, false, rowraw, rownorm, lr, qsp, lc, w, cmax, get_ub,
                                 rowthr, rowbuf);
  return f32_strip_end(s, lc, rowbuf, cells, status);
}

// Probe both directions, continue the likelier to die.  The FP32 pass runs
// `probe` strips forward and `probe` strips on the reversed pair (its own row
// buffer rowbuf_r), then finishes the direction whose last row has the
// smaller slack (threshold minus the row's smallest value: the closer to an
// all-dead row).  A pair the screen will abandon is abandoned by whichever
// direction gets there first; the cfg4 design study (tools/live_study.c)
// measured 1.7x fewer live cells than forward alone (the death rows of the
// two directions are heavy-tailed and weakly correlated).  probe = 0: the
// forward pass alone.  Returns +inf when proven > ub; otherwise a value (or
// status kF32Undecided): run the exact engine.  (One inlined strip loop per
// direction: the phases share it.)
// st: two F32Strip in shared memory (the warp's): the inactive direction's
// state stays there, not in registers (the search kernel is at its register
// budget; local memory would miss L1 under the large shared-memory carve-out).
// on_pick(use_r, vmin): called once both probes are alive, before the chosen
// direction continues, with the minimum of the DROPPED direction's frontier
// row: every path pays at least that (less the FP32 error) inside the rows
// the dropped probe covered, which the caller may add to the continuing
// direction's cumulative bound (kernels.cu: run_dtw).  If it did (returns
// true), the bound no longer holds inside those rows: the continuing pass
// stops before them, undecided if still alive.
struct NoPick {
  __device__ bool operator()(bool, float) const { return false; }
};
template <int BLK, bool UNB, class RawF, class RawR, class NormFn, class UbFn, class ThrF, class ThrR,
          class PickFn = NoPick>
__device__ float f32_probe_pair(const RawF& raw_f, const RawR& raw_r, const NormFn& rownorm, int lr,
                                const float* __restrict__ qsp, int lc, int w, float cmax,
                                UbFn&& get_ub, ThrF&& thr_f, ThrR&& thr_r,
                                float* __restrict__ rowbuf_f, float* __restrict__ rowbuf_r,
                                int probe, F32Strip* st, unsigned long long& cells, int& status,
                                PickFn&& on_pick = NoPick{}) {
  F32Strip& f = st[0];
  F32Strip& r = st[1];
  f32_strip_begin(f, lc, rowbuf_f);
  if (probe <= 0 || lr <= 32 * probe) probe = 0;
  bool use_r = false, limited = false;
  // phase 0: forward probe (or the whole forward pass); 1: reversed probe;
  // 2: the rest of the chosen direction
  for (int phase = 0; phase < 3; ++phase) {
    if (phase == 1) {
      if (probe == 0 || f.lo < 0 || f.status != 0) break;
      f32_strip_begin(r, lc, rowbuf_r);
    }
    if (phase == 2) {
      use_r = r.lo < 0 || r.status != 0 || r.slack < f.slack;
      if (r.lo >= 0 && r.status == 0) limited = on_pick(use_r, use_r ? f.vmin : r.vmin);
      int unused;
      if (use_r) f32_strip_end(f, lc, rowbuf_f, cells, unused);  // the dropped direction's cells count
      else f32_strip_end(r, lc, rowbuf_r, cells, unused);
    }
    const bool rev = phase == 1 || (phase == 2 && use_r);
    // (limited: the whole strips before the last 32 * probe rows)
    const int n = (phase < 2 && probe > 0) ? probe : (limited ? (lr - 32 * probe) / 32 - probe : lr);
    if (rev)
      f32_strip_run<BLK, UNB, true>(r, n, phase == 1, raw_r, rownorm, lr, qsp, lc, w, cmax, get_ub,
                                    thr_r, rowbuf_r);
    else
      f32_strip_run<BLK, UNB, false>(f, n, phase == 0, raw_f, rownorm, lr, qsp, lc, w, cmax,
                                     get_ub, thr_f, rowbuf_f);
    if (phase == 0 && probe == 0) break;
  }
  if (limited) {
    F32Strip& c = use_r ? r : f;
    if (c.status == 0 && c.lo >= 0 && c.i0 <= lr) c.status = kF32Undecided;
    __syncwarp();
  }
  return use_r ? f32_strip_end(r, lc, rowbuf_r, cells, status)
               : f32_strip_end(f, lc, rowbuf_f, cells, status);
}

}  // namespace eapdtw_b200
