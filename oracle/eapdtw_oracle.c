/*
 * eapdtw_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * path; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
 * may load it.  The product library (paper_2010_05371_b200/) never links,
 * loads or calls anything under oracle/.
 *
 * It restates, in plain C11 with IEEE double arithmetic and NO floating-point
 * contraction (built with -ffp-contract=off), the algorithms of the reference
 * (paths relative to /root/reference/proj):
 *   - full_scan              src/dtw.cpp:95-122
 *   - left_prune_scan        src/dtw.cpp:130-182
 *   - ea_pruned_scan         src/dtw.cpp:197-296   (EAPrunedDTW, four stages)
 *   - orient / effective_window / check_cumulative_bound  src/dtw.cpp:48-86
 *   - compute_envelope       src/lower_bounds.cpp:9-49 (restated as a direct
 *                            max/min scan: the envelope values are exact
 *                            max/min, so any sweep order gives equal bits)
 *   - lb_kim_fl / lb_keogh / cumulative_bound  src/lower_bounds.cpp:51-103
 *   - RunningStats / znormalize_into            include/eapdtw/search.hpp:16-42,
 *                                               src/search.cpp:25-46
 *   - cascade_decision / similarity_search      src/search.cpp:63-210
 *   - the cfg1 pairwise loop and the cfg5 NN1 loop (harness loops over
 *     ea_pruned_dtw_windowed / ea_pruned_dtw).
 *
 * Parity is pinned in tests/test_oracle.py against the reference's own
 * fixtures (test_dtw.cpp worked example, acceptance.cpp goldens) and against
 * the reference library itself compiled into oracle/_ref/ (oracle/Makefile).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_ENOMEM 3
#define ORC_UNBOUNDED ((size_t)-1)

static const double PINF = 1.0 / 0.0;

/* squared_cost: include/eapdtw/dtw.hpp:60-63 */
static inline double sq_cost(double a, double b) {
  const double d = a - b;
  return d * d;
}
static inline double dmin(double a, double b) { return b < a ? b : a; }
static inline double min3(double a, double b, double c) { return dmin(a, dmin(b, c)); }
static inline size_t zmin(size_t a, size_t b) { return a < b ? a : b; }
static inline size_t zmax(size_t a, size_t b) { return a > b ? a : b; }
/* band_start: src/dtw.cpp:77 */
static inline size_t band_start(size_t i, size_t w) { return i > w ? i - w : 1; }

/* row_threshold: src/dtw.cpp:81-86 */
static inline double row_threshold(double ub, const double* cb, size_t cb_len, size_t i, size_t w,
                                   size_t lr) {
  if (cb_len == 0) return ub;
  const size_t k = zmin(i + w, lr);
  const double t = ub - cb[k - 1];
  return t > 0.0 ? t : 0.0; /* std::max(0.0, t) */
}

/* full_scan: src/dtw.cpp:95-122 (row-by-row DP on a double buffer) */
double orc_full_scan(const double* rows, size_t lr, const double* cols, size_t lc, size_t w,
                     uint64_t* cells) {
  double* buf = (double*)malloc(2 * (lc + 1) * sizeof(double));
  if (!buf) return NAN;
  for (size_t k = 0; k < 2 * (lc + 1); ++k) buf[k] = PINF;
  double* prev = buf;
  double* curr = buf + lc + 1;
  curr[0] = 0.0;
  uint64_t n = 0;
  for (size_t i = 1; i <= lr; ++i) {
    double* t = prev; prev = curr; curr = t;
    const double ri = rows[i - 1];
    const size_t js = band_start(i, w);
    const size_t je = zmin(lc, i + w);
    curr[js - 1] = PINF;
    for (size_t j = js; j <= je; ++j) {
      curr[j] = sq_cost(ri, cols[j - 1]) + min3(curr[j - 1], prev[j], prev[j - 1]);
      ++n;
    }
    if (je + 1 <= lc) curr[je + 1] = PINF;
  }
  const double r = curr[lc];
  free(buf);
  if (cells) *cells += n;
  return r;
}

/* left_prune_scan: src/dtw.cpp:130-182 */
double orc_left_prune_scan(const double* rows, size_t lr, const double* cols, size_t lc, size_t w,
                           double ub, uint64_t* cells) {
  double* buf = (double*)malloc(2 * (lc + 1) * sizeof(double));
  if (!buf) return NAN;
  for (size_t k = 0; k < 2 * (lc + 1); ++k) buf[k] = PINF;
  double* prev = buf;
  double* curr = buf + lc + 1;
  curr[0] = 0.0;
  uint64_t n = 0;
  size_t next_start = 1;
  double result;
  for (size_t i = 1; i <= lr; ++i) {
    double* t = prev; prev = curr; curr = t;
    const double ri = rows[i - 1];
    const size_t js = zmax(next_start, band_start(i, w));
    const size_t je = zmin(lc, i + w);
    next_start = js;
    size_t j = js;
    curr[j - 1] = PINF;
    for (; j == next_start && j <= je; ++j) { /* stage 1: discard run */
      const double v = sq_cost(ri, cols[j - 1]) + dmin(prev[j], prev[j - 1]);
      curr[j] = v;
      ++n;
      if (v > ub) ++next_start;
    }
    if (j > je && j == next_start) { result = PINF; goto done; }
    for (; j <= je; ++j) { /* stage 2 */
      curr[j] = sq_cost(ri, cols[j - 1]) + min3(curr[j - 1], prev[j], prev[j - 1]);
      ++n;
    }
    if (je + 1 <= lc) curr[je + 1] = PINF;
  }
  result = curr[lc] <= ub ? curr[lc] : PINF;
done:
  free(buf);
  if (cells) *cells += n;
  return result;
}

/* ea_pruned_scan: src/dtw.cpp:197-296.  EAPrunedDTW: left border via the
 * discard run (next_start), right border via the pruning point pp which
 * persists across rows; abandon when the borders collide. */
double orc_ea_pruned_scan(const double* rows, size_t lr, const double* cols, size_t lc, size_t w,
                          double ub_global, const double* cb, size_t cb_len, uint64_t* cells) {
  double* buf = (double*)malloc(2 * (lc + 1) * sizeof(double));
  if (!buf) return NAN;
  for (size_t k = 0; k < 2 * (lc + 1); ++k) buf[k] = PINF;
  double* prev = buf;
  double* curr = buf + lc + 1;
  curr[0] = 0.0;
  uint64_t n = 0;
  size_t next_start = 1, prev_pp = 1, pp = 0;
  double result = PINF;

  for (size_t i = 1; i <= lr; ++i) {
    double* t = prev; prev = curr; curr = t;
    const double ri = rows[i - 1];
    const double ub = row_threshold(ub_global, cb, cb_len, i, w, lr);
    const size_t js = zmax(next_start, band_start(i, w));
    const size_t je = zmin(lc, i + w);
    next_start = js;
    size_t j = js;
    curr[j - 1] = PINF;
    if (js > prev_pp) goto abandon; /* row starts inside the pruned area */

    for (; j == next_start && j < prev_pp; ++j) { /* stage 1 */
      const double v = sq_cost(ri, cols[j - 1]) + dmin(prev[j], prev[j - 1]);
      curr[j] = v;
      ++n;
      if (v > ub) ++next_start; else pp = j + 1;
    }
    for (; j < prev_pp; ++j) { /* stage 2 */
      const double v = sq_cost(ri, cols[j - 1]) + min3(curr[j - 1], prev[j], prev[j - 1]);
      curr[j] = v;
      ++n;
      if (v <= ub) pp = j + 1;
    }
    if (j <= je) { /* stage 3, at the previous pruning point */
      const double d = sq_cost(ri, cols[j - 1]);
      if (j == next_start) {
        const double v = d + prev[j - 1];
        curr[j] = v;
        ++n;
        if (v <= ub) pp = j + 1; else goto abandon;
      } else {
        const double v = d + dmin(curr[j - 1], prev[j - 1]);
        curr[j] = v;
        ++n;
        if (v <= ub) pp = j + 1;
      }
      ++j;
    } else if (j == next_start) {
      goto abandon;
    }
    for (; j == pp && j <= je; ++j) { /* stage 4, left only */
      const double v = sq_cost(ri, cols[j - 1]) + curr[j - 1];
      curr[j] = v;
      ++n;
      if (v <= ub) ++pp;
    }
    if (je + 1 <= lc) curr[je + 1] = PINF;
    prev_pp = pp;
  }
  if (prev_pp > lc) result = curr[lc];
abandon:
  free(buf);
  if (cells) *cells += n;
  return result;
}

/* orient (src/dtw.cpp:48-52): longer series on rows, first argument wins ties.
 * effective_window (src/dtw.cpp:57-62).  Returns 0 when no path fits. */
static int orient_window(const double** a, size_t* la, const double** b, size_t* lb,
                         size_t window, size_t* w_out) {
  if (*la < *lb) {
    const double* tp = *a; *a = *b; *b = tp;
    size_t tl = *la; *la = *lb; *lb = tl;
  }
  const size_t lr = *la, lc = *lb;
  if (window == ORC_UNBOUNDED) { *w_out = lr; return 1; }
  if (lr - lc > window) return 0;
  *w_out = window >= lc ? lr : window;
  return 1;
}

/* check_cumulative_bound: src/dtw.cpp:64-75 */
static int check_cb(const double* cb, size_t cb_len, size_t lr) {
  if (cb_len == 0) return ORC_OK;
  if (cb_len != lr) return ORC_EINVAL;
  for (size_t k = 0; k + 1 < cb_len; ++k)
    if (!(cb[k] >= cb[k + 1])) return ORC_EINVAL;
  if (cb[cb_len - 1] != 0.0) return ORC_EINVAL;
  return ORC_OK;
}

/* Entry points (src/dtw.cpp:304-396).  algo: 0 full (windowed), 1 left-prune,
 * 2 EAPrunedDTW.  window == ORC_UNBOUNDED means Band::unbounded(). */
int orc_dtw(int algo, const double* a, size_t la, const double* b, size_t lb, size_t window,
            double ub, const double* cb, size_t cb_len, double* out, uint64_t* cells) {
  if (la == 0 || lb == 0) return ORC_EINVAL;
  size_t w;
  const size_t lr = la >= lb ? la : lb;
  if (algo == 2) {
    const int e = check_cb(cb, cb_len, lr);
    if (e) return e;
  }
  if (!orient_window(&a, &la, &b, &lb, window, &w)) { *out = PINF; return ORC_OK; }
  switch (algo) {
    case 0: *out = orc_full_scan(a, la, b, lb, w, cells); break;
    case 1: *out = orc_left_prune_scan(a, la, b, lb, w, ub, cells); break;
    case 2: *out = orc_ea_pruned_scan(a, la, b, lb, w, ub, cb, cb_len, cells); break;
    default: return ORC_EINVAL;
  }
  return ORC_OK;
}

/* compute_envelope: src/lower_bounds.cpp:9-49.  Upper/lower = max/min over
 * [j-w, j+w] clamped to [0, l). */
int orc_compute_envelope(const double* s, size_t l, size_t window, double* upper, double* lower) {
  if (l == 0) return ORC_EINVAL;
  const size_t w = window == ORC_UNBOUNDED ? l : zmin(window, l);
  for (size_t j = 0; j < l; ++j) {
    const size_t lo = j > w ? j - w : 0;
    const size_t hi = zmin(l - 1, j + w);
    double mx = s[lo], mn = s[lo];
    for (size_t k = lo + 1; k <= hi; ++k) {
      if (s[k] > mx) mx = s[k];
      if (s[k] < mn) mn = s[k];
    }
    upper[j] = mx;
    lower[j] = mn;
  }
  return ORC_OK;
}

/* lb_kim_fl: src/lower_bounds.cpp:51-55 */
int orc_lb_kim_fl(const double* q, const double* c, size_t l, double* out) {
  if (l < 2) return ORC_EINVAL;
  *out = sq_cost(q[0], c[0]) + sq_cost(q[l - 1], c[l - 1]);
  return ORC_OK;
}

/* lb_keogh: src/lower_bounds.cpp:57-88.  order may be NULL (natural order);
 * contributions (length l) is zero-filled then written per visited position. */
double orc_lb_keogh(const double* upper, const double* lower, const double* x, size_t l,
                    double abandon_above, const size_t* order, double* contrib, int* abandoned) {
  double total = 0.0;
  if (contrib) memset(contrib, 0, l * sizeof(double));
  if (abandoned) *abandoned = 0;
  for (size_t k = 0; k < l; ++k) {
    const size_t j = order ? order[k] : k;
    double d = 0.0;
    if (x[j] > upper[j]) d = sq_cost(x[j], upper[j]);
    else if (x[j] < lower[j]) d = sq_cost(x[j], lower[j]);
    total += d;
    if (contrib) contrib[j] = d;
    if (total > abandon_above) {
      if (abandoned) *abandoned = 1;
      break;
    }
  }
  return total;
}

/* cumulative_bound: src/lower_bounds.cpp:90-103 */
int orc_cumulative_bound(const double* c, size_t l, double* cb) {
  if (l == 0) return ORC_OK;
  for (size_t k = 0; k < l; ++k) cb[k] = 0.0;
  if (c[l - 1] < 0.0) return ORC_EINVAL;
  for (size_t k = l - 1; k-- > 0;) {
    if (c[k] < 0.0) return ORC_EINVAL;
    cb[k] = cb[k + 1] + c[k + 1];
  }
  return ORC_OK;
}

/* RunningStats (include/eapdtw/search.hpp:16-42, src/search.cpp:25-35) */
typedef struct { double sum, sumsq; size_t count; } orc_stats;

static orc_stats stats_over(const double* x, size_t n) {
  orc_stats s = {0.0, 0.0, n};
  for (size_t i = 0; i < n; ++i) {
    s.sum += x[i];
    s.sumsq += x[i] * x[i];
  }
  return s;
}
static inline double stats_mean(const orc_stats* s) { return s->sum / (double)s->count; }
static inline double stats_sd(const orc_stats* s) {
  const double m = stats_mean(s);
  const double v = s->sumsq / (double)s->count - m * m;
  return sqrt(v > 0.0 ? v : 0.0);
}

/* znormalize_into: src/search.cpp:37-46 (kMinStddev = 1e-12, :13) */
static void znorm_into(const double* src, size_t n, const orc_stats* st, double* dst) {
  const double m = stats_mean(st);
  const double s = stats_sd(st);
  if (s < 1e-12) {
    for (size_t i = 0; i < n; ++i) dst[i] = 0.0;
    return;
  }
  for (size_t i = 0; i < n; ++i) dst[i] = (src[i] - m) / s;
}

int orc_znormalize(const double* src, size_t n, double* dst) {
  if (n == 0) return ORC_EINVAL;
  const orc_stats st = stats_over(src, n);
  znorm_into(src, n, &st, dst);
  return ORC_OK;
}

/* Sliding stats chain exactly as similarity_search runs it (search.cpp:156-168,
 * reset every 100000 slides, :16).  Writes mean[s] and sd[s] for every start. */
int orc_sliding_stats(const double* ref, size_t n, size_t m, double* mean, double* sd) {
  if (m == 0 || m > n) return ORC_EINVAL;
  orc_stats st = stats_over(ref, m);
  size_t since = 0;
  for (size_t s = 0; s + m <= n; ++s) {
    if (s > 0) {
      st.sum += ref[s + m - 1];
      st.sumsq += ref[s + m - 1] * ref[s + m - 1];
      st.sum -= ref[s - 1];
      st.sumsq -= ref[s - 1] * ref[s - 1];
      if (++since == 100000) {
        st = stats_over(ref + s, m);
        since = 0;
      }
    }
    mean[s] = stats_mean(&st);
    sd[s] = stats_sd(&st);
  }
  return ORC_OK;
}

typedef struct {
  uint64_t location;
  double distance_sq;
  int32_t found;
  int32_t pad_;
  uint64_t candidates_total, pruned_kim, pruned_keogh_eq, pruned_keogh_ec, dtw_calls,
      dtw_abandoned, dp_cells_evaluated;
  double elapsed_seconds;
} orc_search_result;

/* similarity_search + cascade_decision: src/search.cpp:63-210.
 * algo: 0 full, 1 left-prune, 2 EAPrunedDTW (search.hpp:56). */
int orc_similarity_search(const double* ref, size_t n, const double* query, size_t qlen,
                          size_t query_length, double ratio, int algo, int use_lb, int tighten,
                          orc_search_result* out) {
  const size_t m = query_length == 0 ? qlen : query_length;
  if (m == 0 || m > qlen) return ORC_EINVAL;
  if (m > n) return ORC_EINVAL;
  const double wf = floor(ratio * (double)m); /* window_cells_for: search.cpp:18-21 */
  const size_t w = wf <= 0.0 ? 0 : (size_t)wf;
  memset(out, 0, sizeof(*out));
  out->distance_sq = PINF;

  double* qn = (double*)malloc(m * sizeof(double));
  double* qu = (double*)malloc(m * sizeof(double));
  double* ql = (double*)malloc(m * sizeof(double));
  size_t* order = (size_t*)malloc(m * sizeof(size_t));
  double* cn = (double*)malloc(m * sizeof(double));
  double* ceq = (double*)malloc(m * sizeof(double));
  double* cec = (double*)malloc(m * sizeof(double));
  double* cu = (double*)malloc(m * sizeof(double));
  double* cl = (double*)malloc(m * sizeof(double));
  double* cb = (double*)malloc(m * sizeof(double));
  if (!qn || !qu || !ql || !order || !cn || !ceq || !cec || !cu || !cl || !cb) return ORC_ENOMEM;

  {
    const orc_stats qs = stats_over(query, m);
    znorm_into(query, m, &qs, qn);
  }
  orc_compute_envelope(qn, m, w, qu, ql);
  /* order: by descending |q|, index ascending on ties (search.cpp:143-149);
   * insertion sort keeps it dependency-free and exact. */
  for (size_t k = 0; k < m; ++k) order[k] = k;
  for (size_t k = 1; k < m; ++k) {
    const size_t v = order[k];
    const double fv = fabs(qn[v]);
    size_t p = k;
    while (p > 0) {
      const size_t u = order[p - 1];
      const double fu = fabs(qn[u]);
      if (fu > fv || (fu == fv && u < v)) break;
      order[p] = u;
      --p;
    }
    order[p] = v;
  }

  orc_stats st = stats_over(ref, m);
  size_t since = 0;
  int found = 0;
  double best = PINF;
  size_t loc = 0;
  for (size_t s = 0; s + m <= n; ++s) {
    if (s > 0) {
      st.sum += ref[s + m - 1];
      st.sumsq += ref[s + m - 1] * ref[s + m - 1];
      st.sum -= ref[s - 1];
      st.sumsq -= ref[s - 1] * ref[s - 1];
      if (++since == 100000) {
        st = stats_over(ref + s, m);
        since = 0;
      }
    }
    ++out->candidates_total;
    const double* craw = ref + s;
    size_t cb_len = 0;
    const double ub = found ? best : PINF;
    if (!use_lb) {
      znorm_into(craw, m, &st, cn);
    } else {
      const double mean = stats_mean(&st);
      const double sd = stats_sd(&st);
      const int constant = sd < 1e-12;
      if (m >= 2) {
        const double c0 = constant ? 0.0 : (craw[0] - mean) / sd;
        const double cl_ = constant ? 0.0 : (craw[m - 1] - mean) / sd;
        const double kim = sq_cost(qn[0], c0) + sq_cost(qn[m - 1], cl_);
        if (kim > ub) { ++out->pruned_kim; continue; }
      }
      znorm_into(craw, m, &st, cn);
      const double eq = orc_lb_keogh(qu, ql, cn, m, ub, order, ceq, NULL);
      if (eq > ub) { ++out->pruned_keogh_eq; continue; }
      orc_compute_envelope(cn, m, w, cu, cl);
      const double ec = orc_lb_keogh(cu, cl, qn, m, ub, order, cec, NULL);
      if (ec > ub) { ++out->pruned_keogh_ec; continue; }
      if (tighten) {
        orc_cumulative_bound(eq > ec ? ceq : cec, m, cb);
        cb_len = m;
      }
    }
    ++out->dtw_calls;
    double d = PINF;
    uint64_t c = 0;
    orc_dtw(algo, cn, m, qn, m, w, ub, cb, cb_len, &d, &c);
    out->dp_cells_evaluated += c;
    if (d == PINF) { ++out->dtw_abandoned; continue; }
    if (!found || d < best) {
      found = 1;
      best = d;
      loc = s;
    }
  }
  out->found = found;
  out->location = loc;
  out->distance_sq = best;
  free(qn); free(qu); free(ql); free(order); free(cn); free(ceq); free(cec); free(cu); free(cl);
  free(cb);
  return ORC_OK;
}

/* cfg1 harness loop: out[p] = ea_pruned_dtw_windowed(a_p, b_p, Band::cells(w), ub[p])
 * (dtw.cpp:377-385).  ub may be NULL (+inf). */
int orc_pairwise(const double* a, const double* b, size_t npairs, size_t len, size_t window,
                 const double* ub, double* out, uint64_t* cells) {
  for (size_t p = 0; p < npairs; ++p) {
    const int e = orc_dtw(2, a + p * len, len, b + p * len, len, window, ub ? ub[p] : PINF, NULL,
                          0, &out[p], cells);
    if (e) return e;
  }
  return ORC_OK;
}

/* cfg5 harness loop: for each query a running cutoff,
 * d = ea_pruned_dtw_windowed(db[k], q, band, bsf); strict < keeps the lowest index. */
int orc_nn1(const double* queries, size_t nq, const double* db, size_t nd, size_t len,
            size_t window, uint64_t* argmin, double* dist, uint64_t* cells) {
  for (size_t q = 0; q < nq; ++q) {
    double bsf = PINF;
    uint64_t arg = 0;
    for (size_t k = 0; k < nd; ++k) {
      double d;
      const int e = orc_dtw(2, db + k * len, len, queries + q * len, len, window, bsf, NULL, 0,
                            &d, cells);
      if (e) return e;
      if (d < bsf) {
        bsf = d;
        arg = k;
      }
    }
    argmin[q] = arg;
    dist[q] = bsf;
  }
  return ORC_OK;
}

/* ---- benchmark data generator (not a reference algorithm) -------------------
 * x0 = 0, x[i+1] = x[i] + N(0,1): std::mt19937_64 (the C++ standard fixes its
 * output stream: word 64, n 312, m 156, r 31, a 0xB5026F5AA96619E9, tempering
 * u 29 / s 17 / t 37 / l 43, init multiplier 6364136223846793005) mapped to
 * (0,1) as (k >> 11 + 0.5) 2^-53 and Box-Muller with both variates used -- the
 * same definition as the product's eapdtw_random_walk_normal, restated here so
 * bench.py's reference arm generates its inputs without loading the product
 * library.  tests/test_oracle.py checks the two agree bit for bit. */
typedef struct {
  uint64_t mt[312];
  int idx;
} orc_mt64;

static void mt64_seed(orc_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(orc_mt64* g) {
  const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t y = (g->mt[i] & upper) | (g->mt[(i + 1) % 312] & lower);
      uint64_t v = g->mt[(i + 156) % 312] ^ (y >> 1);
      if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = v;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

int orc_random_walk_normal(size_t n, uint64_t seed, double* out) {
  if (n == 0 || !out) return ORC_EINVAL;
  orc_mt64* g = (orc_mt64*)malloc(sizeof(orc_mt64));
  if (!g) return ORC_ENOMEM;
  mt64_seed(g, seed);
  double x = 0.0;
  out[0] = 0.0;
  size_t i = 1;
  while (i < n) {
    const double u1 = ((double)(mt64_next(g) >> 11) + 0.5) * 0x1.0p-53;
    const double u2 = ((double)(mt64_next(g) >> 11) + 0.5) * 0x1.0p-53;
    const double rad = sqrt(-2.0 * log(u1));
    const double th = 6.283185307179586 * u2;
    x += rad * cos(th);
    out[i++] = x;
    if (i < n) {
      x += rad * sin(th);
      out[i++] = x;
    }
  }
  free(g);
  return ORC_OK;
}
