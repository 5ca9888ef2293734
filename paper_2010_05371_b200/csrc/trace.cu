// trace.cu -- per-cell event capture of one DTW on the device (KernelTrace,
// dtw.hpp:42-57; the CLI's `trace` subcommand, eapdtw_cli.cpp:91-108).
//
// A debugging path, not a throughput path: one thread walks the DP matrix row
// by row in the reference's event order and appends every event (cell,
// discard point, pruning point, abandon) to a device log, so the log can be
// compared line for line with the reference's write_trace_csv.  The three
// schedules follow dtw.cpp:95-122 (full), :130-182 (left prune) and :197-296
// (EAPrunedDTW); values use the production kernels' arithmetic (explicitly
// rounded DSUB/DMUL/DADD, no FMA), so the traced cell values are the ones the
// warp engine computes.  The log is bounded by the caller's capacity; the
// number of events is always returned so a caller can size a retry.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace eapdtw_b200 {

namespace {

struct Log {
  TraceEvent* ev;
  long long cap;
  long long n = 0;
  unsigned long long cells = 0;
  long long last_row = 0, last_col = 0;

  __device__ void put(unsigned kind, long long i, long long j, double v) {
    if (n < cap) {
      TraceEvent e;
      e.kind = kind;
      e.pad_ = 0;
      e.row = static_cast<unsigned long long>(i);
      e.col = static_cast<unsigned long long>(j);
      e.value = v;
      ev[n] = e;
    }
    ++n;
  }
  __device__ void cell(long long i, long long j, double v) {
    ++cells;
    last_row = i;
    last_col = j;
    put(kTraceCell, i, j, v);
  }
  __device__ void discard(long long i, long long j, double v) { put(kTraceDiscard, i, j, v); }
  __device__ void pruning_point(long long i, long long j) {
    put(kTracePruningPoint, i, j, __longlong_as_double(0x7ff0000000000000LL));
  }
  __device__ void abandon() {
    put(kTraceAbandon, last_row, last_col, __longlong_as_double(0x7ff0000000000000LL));
  }
};

__device__ __forceinline__ double cost(double a, double b) {
  const double d = __dsub_rn(a, b);
  return __dmul_rn(d, d);
}
__device__ __forceinline__ double dmin2(double a, double b) { return b < a ? b : a; }
__device__ __forceinline__ double dmin3(double a, double b, double c) { return dmin2(a, dmin2(b, c)); }

__global__ void trace_kernel(int algo, const double* __restrict__ rows, long long lr,
                             const double* __restrict__ cols, long long lc, long long w, double ub,
                             double* __restrict__ buf, TraceEvent* __restrict__ ev, long long cap,
                             unsigned long long* __restrict__ hdr, double* __restrict__ result) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double INF = __longlong_as_double(0x7ff0000000000000LL);
  Log log{ev, cap};
  double* prev = buf;
  double* curr = buf + lc + 1;
  for (long long k = 0; k < 2 * (lc + 1); ++k) buf[k] = INF;
  curr[0] = 0.0;
  double out = INF;
  bool done = false;

  // band limits of row i (dtw.cpp:77, :104-105)
  auto band_lo = [&](long long i) { return i > w ? i - w : 1LL; };
  auto band_hi = [&](long long i) { return lc < i + w ? lc : i + w; };

  if (algo == 0) {  // full_scan: every band cell, three-way minimum
    for (long long i = 1; i <= lr; ++i) {
      double* t = prev; prev = curr; curr = t;
      const double ri = rows[i - 1];
      const long long j0 = band_lo(i), j1 = band_hi(i);
      curr[j0 - 1] = INF;
      for (long long j = j0; j <= j1; ++j) {
        const double v = __dadd_rn(cost(ri, cols[j - 1]), dmin3(curr[j - 1], prev[j], prev[j - 1]));
        curr[j] = v;
        log.cell(i, j, v);
      }
      if (j1 + 1 <= lc) curr[j1 + 1] = INF;
    }
    out = curr[lc];
  } else if (algo == 1) {  // left_prune_scan: a discard run moves the row start
    long long start = 1;
    for (long long i = 1; i <= lr && !done; ++i) {
      double* t = prev; prev = curr; curr = t;
      const double ri = rows[i - 1];
      const long long j0 = start > band_lo(i) ? start : band_lo(i);
      const long long j1 = band_hi(i);
      start = j0;
      long long j = j0;
      curr[j - 1] = INF;
      for (; j == start && j <= j1; ++j) {  // the run: top and diagonal only
        const double v = __dadd_rn(cost(ri, cols[j - 1]), dmin2(prev[j], prev[j - 1]));
        curr[j] = v;
        log.cell(i, j, v);
        if (v > ub) {
          ++start;
          log.discard(i, j, v);
        }
      }
      if (j > j1 && j == start) {  // the run consumed the reachable row
        log.abandon();
        done = true;
        break;
      }
      for (; j <= j1; ++j) {
        const double v = __dadd_rn(cost(ri, cols[j - 1]), dmin3(curr[j - 1], prev[j], prev[j - 1]));
        curr[j] = v;
        log.cell(i, j, v);
      }
      if (j1 + 1 <= lc) curr[j1 + 1] = INF;
    }
    if (!done) {
      if (curr[lc] <= ub) {
        out = curr[lc];
      } else {
        log.abandon();
      }
    }
  } else {  // ea_pruned_scan: left border (discard run) + right border (pruning point)
    long long start = 1, ppr = 1, pp = 0;
    log.pruning_point(0, 1);
    for (long long i = 1; i <= lr && !done; ++i) {
      double* t = prev; prev = curr; curr = t;
      const double ri = rows[i - 1];
      const long long j0 = start > band_lo(i) ? start : band_lo(i);
      const long long j1 = band_hi(i);
      start = j0;
      long long j = j0;
      curr[j - 1] = INF;
      if (j0 > ppr) {  // row starts inside the pruned area
        log.abandon();
        done = true;
        break;
      }
      for (; j == start && j < ppr; ++j) {  // discard run before the old pruning point
        const double v = __dadd_rn(cost(ri, cols[j - 1]), dmin2(prev[j], prev[j - 1]));
        curr[j] = v;
        log.cell(i, j, v);
        if (v > ub) {
          ++start;
          log.discard(i, j, v);
        } else {
          pp = j + 1;
        }
      }
      for (; j < ppr; ++j) {  // three-way scan up to the old pruning point
        const double v = __dadd_rn(cost(ri, cols[j - 1]), dmin3(curr[j - 1], prev[j], prev[j - 1]));
        curr[j] = v;
        log.cell(i, j, v);
        if (v <= ub) pp = j + 1;
      }
      if (j <= j1) {  // the old pruning point's column
        const double d = cost(ri, cols[j - 1]);
        if (j == start) {  // after a discard run only the diagonal is left
          const double v = __dadd_rn(d, prev[j - 1]);
          curr[j] = v;
          log.cell(i, j, v);
          if (v <= ub) {
            pp = j + 1;
          } else {
            log.abandon();
            done = true;
            break;
          }
        } else {
          const double v = __dadd_rn(d, dmin2(curr[j - 1], prev[j - 1]));
          curr[j] = v;
          log.cell(i, j, v);
          if (v <= ub) pp = j + 1;
        }
        ++j;
      } else if (j == start) {
        log.abandon();
        done = true;
        break;
      }
      for (; j == pp && j <= j1; ++j) {  // past it: left neighbour only
        const double v = __dadd_rn(cost(ri, cols[j - 1]), curr[j - 1]);
        curr[j] = v;
        log.cell(i, j, v);
        if (v <= ub) ++pp;
      }
      if (j1 + 1 <= lc) curr[j1 + 1] = INF;
      if (pp <= j1) log.pruning_point(i, pp);
      ppr = pp;
    }
    if (!done) {
      if (ppr > lc) {
        out = curr[lc];
      } else {
        log.abandon();
      }
    }
  }
  hdr[0] = static_cast<unsigned long long>(log.n);
  hdr[1] = log.cells;
  *result = out;
}

}  // namespace

cudaError_t launch_trace(int algo, const double* rows, long long lr, const double* cols,
                         long long lc, long long w, double ub, double* buf, TraceEvent* ev,
                         long long cap, unsigned long long* hdr, double* result,
                         cudaStream_t stream) {
  trace_kernel<<<1, 32, 0, stream>>>(algo, rows, lr, cols, lc, w, ub, buf, ev, cap, hdr, result);
  return cudaGetLastError();
}

}  // namespace eapdtw_b200
