/* live_study.c -- where the pruned DTW's live cells sit (design study for the
 * FP32 screen's schedule; not product code).
 *
 * cfg4 shape: the first N points of the bench reference, m = 1024, w = 205,
 * threshold ub fixed at the full search's final distance.  Every candidate
 * that survives LB_Kim (corners) -> LB_Keogh EQ -> LB_Keogh EC (the
 * reference's cascade, search.cpp:63-107) is run through the DP with the
 * reference's row thresholds (ub - cb[min(i+w, m) - 1], dtw.cpp:81-86) and
 * dead cells killed.  Per row: the live column range [lo, hi] in diagonal
 * offsets e = j - i.  Reported: rows survived, live cells, the live offset
 * width per row (histogram) and its maximum per task, and the drift of the
 * range centre.
 *
 *   gcc -O2 -fopenmp -o /tmp/live_study tools/live_study.c oracle/eapdtw_oracle.c -lm
 *   /tmp/live_study N ub
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

int orc_random_walk_normal(size_t n, uint64_t seed, double* out);
int orc_sliding_stats(const double* ref, size_t n, size_t m, double* mean, double* sd);
int orc_znormalize(const double* src, size_t n, double* dst);
int orc_compute_envelope(const double* s, size_t l, size_t window, double* upper, double* lower);
double orc_lb_keogh(const double* upper, const double* lower, const double* x, size_t l,
                    double abandon_above, const size_t* order, double* contrib, int* abandoned);
int orc_cumulative_bound(const double* c, size_t l, double* cb);

/* Pruned DP (dead cells killed) with row thresholds ub - cb[min(i+w, m) - 1]:
   returns rows survived, adds live cells to *cells. */
static _Thread_local double g_extra = 0.0; static _Thread_local size_t g_kk_limit = 0;
static int pruned_rows(const double* c, const double* qn, const double* cbnd, size_t m, size_t w,
                       double ub, double* prev, double* cur, long long* cells, int* rowcells,
                       double* slack) {
  for (size_t j = 0; j <= m + 1; ++j) prev[j] = INFINITY;
  prev[0] = 0.0;
  int rows = 0;
  for (size_t i = 1; i <= m; ++i) {
    const size_t kk = (i + w < m ? i + w : m) - 1;
    double thr = ub - cbnd[kk];
    if (g_extra > 0 && kk <= g_kk_limit) thr -= g_extra;
    if (thr < 0) thr = 0;
    int any = 0;
    double vmin = INFINITY;
    const size_t bl = i > w ? i - w : 1, bh = i + w < m ? i + w : m;
    for (size_t j = 0; j <= m + 1; ++j) cur[j] = INFINITY;
    for (size_t j = bl; j <= bh; ++j) {
      double mn = prev[j - 1];
      if (prev[j] < mn) mn = prev[j];
      if (cur[j - 1] < mn) mn = cur[j - 1];
      if (mn == INFINITY) continue;
      const double d = c[i - 1] - qn[j - 1];
      const double v = d * d + mn;
      if (v > thr) continue;
      cur[j] = v;
      ++*cells;
      ++any;
      if (v < vmin) vmin = v;
    }
    if (rowcells) rowcells[i] = any;
    if (slack) slack[i] = thr - vmin;
    if (!any) break;
    ++rows;
    double* t = prev;
    prev = cur;
    cur = t;
  }
  return rows;
}

static const double* g_q;
static int cmp_order(const void* a, const void* b) {
  const size_t i = *(const size_t*)a, j = *(const size_t*)b;
  const double fa = fabs(g_q[i]), fb = fabs(g_q[j]);
  if (fa != fb) return fa > fb ? -1 : 1;
  return i < j ? -1 : 1;
}

int main(int argc, char** argv) {
  const size_t N = argc > 1 ? (size_t)atol(argv[1]) : 2000000;
  const double ub = argc > 2 ? atof(argv[2]) : 3.748871965313156;
  const size_t m = 1024, w = 205;
  double* ref = malloc(N * 8);
  double* q = malloc(m * 8);
  orc_random_walk_normal(N, 20261019ULL, ref);
  orc_random_walk_normal(m, 20261020ULL, q);
  double* qn = malloc(m * 8);
  orc_znormalize(q, m, qn);
  double *qu = malloc(m * 8), *ql = malloc(m * 8);
  orc_compute_envelope(qn, m, w, qu, ql);
  size_t* order = malloc(m * sizeof(size_t));
  for (size_t k = 0; k < m; ++k) order[k] = k;
  g_q = qn;
  qsort(order, m, sizeof(size_t), cmp_order);
  const size_t nc = N - m + 1;
  double *mean = malloc(nc * 8), *sd = malloc(nc * 8);
  orc_sliding_stats(ref, N, m, mean, sd);

  long long tasks = 0, cells = 0, rows_sum = 0;
  long long whist[12] = {0};          /* per-row live width: <=16,32,48,64,88,104,128,144,192,256,384,>384 */
  long long maxhist[12] = {0};        /* per-task max width */
  long long cells_by_max[12] = {0};   /* live cells, by the task's max width */
  const int edges[11] = {16, 32, 48, 64, 88, 104, 128, 144, 192, 256, 384};
  long long rowhist[12] = {0}, rowcells[12] = {0}; /* rows survived: 0,1,2,<=4,8,16,32,64,128,256,512,>512 */
  long long eqrow_hist[12] = {0}; /* the same with EQ-only thresholds (rows < 16 only) */
  long long drift_hist[8] = {0};      /* |centre(i) - centre(i-16)| per 16 rows: <=2,4,8,16,32,64,128,>128 */
  /* by d / ub of the task (full banded DTW): <=1, 1.1, 1.25, 1.5, 2, 3, >3 */
  long long dr_tasks[7] = {0}, dr_cells[7] = {0}, imp_tasks = 0, imp_cells = 0;
  long long rev_rows = 0, rev_cells = 0, min_rows = 0, min_cells2 = 0, best_cells = 0, pred_cells = 0;
  long long pk_cells[4][2] = {{0}};  /* probe k = 16, 32, 64, 128 rows both ways: [by slack, by live count] */
  const int pks[4] = {16, 32, 64, 128};
  long long comb_cells = 0, comb_plain = 0;
  long long greedy_cells[3] = {0};
  long long alt_cells[3] = {0};  /* K = 32: slack/T, extrapolated death row, slack at 32 + width */  /* strip-granular races: greedy least-slack (S = 16, 32, 64) */
  const double dedges[6] = {1.0, 1.1, 1.25, 1.5, 2.0, 3.0};
#pragma omp parallel reduction(+ : comb_cells, comb_plain, rowhist[:12], rowcells[:12], eqrow_hist[:12], tasks, cells, rows_sum, whist[:12], maxhist[:12], cells_by_max[:12], drift_hist[:8], dr_tasks[:7], dr_cells[:7], imp_tasks, imp_cells, rev_rows, rev_cells, min_rows, min_cells2, best_cells, pred_cells, pk_cells[:4][:2], greedy_cells[:3], alt_cells[:3])
  {
    double *c = malloc(m * 8), *cu = malloc(m * 8), *cl = malloc(m * 8);
    double *ceq = malloc(m * 8), *cec = malloc(m * 8), *cbnd = malloc(m * 8), *cbig = malloc(m * 8);
    double *prev = malloc((m + 2) * 8), *cur = malloc((m + 2) * 8);
    int* cen = malloc((m + 1) * sizeof(int));
#pragma omp for schedule(dynamic, 4096)
    for (size_t s = 0; s < nc; ++s) {
      const double mu = mean[s], sg = sd[s];
      if (sg < 1e-12) continue;
      const double c0 = (ref[s] - mu) / sg, cl0 = (ref[s + m - 1] - mu) / sg;
      const double kim = (qn[0] - c0) * (qn[0] - c0) + (qn[m - 1] - cl0) * (qn[m - 1] - cl0);
      if (kim > ub) continue;
      for (size_t k = 0; k < m; ++k) c[k] = (ref[s + k] - mu) / sg;
      int ab = 0;
      const double teq = orc_lb_keogh(qu, ql, c, m, ub, order, ceq, &ab);
      if (ab) continue;
      orc_compute_envelope(c, m, w, cu, cl);
      const double tec = orc_lb_keogh(cu, cl, qn, m, ub, order, cec, &ab);
      if (ab) continue;
      orc_cumulative_bound(tec > teq ? cec : ceq, m, cbnd);
      /* the DP with killed dead cells; rows = candidate, cols = query */
      ++tasks;
      for (size_t j = 0; j <= m + 1; ++j) prev[j] = INFINITY;
      prev[0] = 0.0;
      int maxw = 0, rows = 0;
      long long tc = 0;
      for (size_t i = 1; i <= m; ++i) {
        const size_t kk = (i + w < m ? i + w : m) - 1;
        double thr = ub - cbnd[kk];
        if (thr < 0) thr = 0;
        cur[0] = INFINITY;
        int lo = 1 << 30, hi = -1;
        const size_t bl = i > w ? i - w : 1, bh = i + w < m ? i + w : m;
        for (size_t j = 1; j <= m + 1; ++j) cur[j] = INFINITY;
        for (size_t j = bl; j <= bh; ++j) {
          double mn = prev[j - 1];
          if (prev[j] < mn) mn = prev[j];
          if (cur[j - 1] < mn) mn = cur[j - 1];
          if (mn == INFINITY) continue;
          const double d = c[i - 1] - qn[j - 1];
          const double v = d * d + mn;
          if (v > thr) continue;
          cur[j] = v;
          ++tc;
          if ((int)j < lo) lo = (int)j;
          hi = (int)j;
        }
        if (hi < 0) break;
        ++rows;
        const int wd = hi - lo + 1;
        int b = 0;
        while (b < 11 && wd > edges[b]) ++b;
        whist[b]++;
        if (wd > maxw) maxw = wd;
        cen[i] = (lo + hi) / 2 - (int)i;
        if (i > 16 && i % 16 == 0) {
          const int dd = abs(cen[i] - cen[i - 16]);
          int db = 0;
          while (db < 7 && dd > (2 << db)) ++db;
          drift_hist[db]++;
        }
        double* t = prev;
        prev = cur;
        cur = t;
      }
      cells += tc;
      rows_sum += rows;
      {
        const int redges[11] = {0, 1, 2, 4, 8, 16, 32, 64, 128, 256, 512};
        int rb = 0;
        while (rb < 11 && rows > redges[rb]) ++rb;
        rowhist[rb]++;
        rowcells[rb] += tc;
        /* EQ-only thresholds, first 16 rows */
        orc_cumulative_bound(ceq, m, cbig);
        long long c2 = 0;
        /* thr(i) = ub - sum_{k >= i} ceq[k] (EQ terms are per row: rows after i still to pay) */
        double suf = 0; 
        double* sufa = cbig; /* reuse: suffix sums */
        for (size_t k = m; k-- > 0;) { suf += ceq[k]; sufa[k] = suf; }
        for (size_t j = 0; j <= m + 1; ++j) prev[j] = INFINITY;
        prev[0] = 0.0;
        int r2 = 0;
        for (size_t i = 1; i <= 16; ++i) {
          double thr = ub - (i < m ? sufa[i] : 0.0);
          int any = 0;
          const size_t bl = i > w ? i - w : 1, bh = i + w < m ? i + w : m;
          for (size_t j = 0; j <= m + 1; ++j) cur[j] = INFINITY;
          for (size_t j = bl; j <= bh && j <= i + 40; ++j) {
            double mn = prev[j - 1];
            if (prev[j] < mn) mn = prev[j];
            if (cur[j - 1] < mn) mn = cur[j - 1];
            if (mn == INFINITY) continue;
            const double d = c[i - 1] - qn[j - 1];
            const double v = d * d + mn;
            if (v > thr) continue;
            cur[j] = v; ++any;
          }
          if (!any) break;
          ++r2;
          double* t = prev; prev = cur; cur = t;
        }
        rb = 0;
        while (rb < 11 && r2 > redges[rb]) ++rb;
        eqrow_hist[rb]++;
      }
      {  /* full banded DTW of the task, and LB_Improved (Lemire) both ways */
        for (size_t j = 0; j <= m + 1; ++j) prev[j] = INFINITY;
        prev[0] = 0.0;
        for (size_t i = 1; i <= m; ++i) {
          const size_t bl = i > w ? i - w : 1, bh = i + w < m ? i + w : m;
          for (size_t j = 0; j <= m + 1; ++j) cur[j] = INFINITY;
          for (size_t j = bl; j <= bh; ++j) {
            double mn = prev[j - 1];
            if (prev[j] < mn) mn = prev[j];
            if (cur[j - 1] < mn) mn = cur[j - 1];
            const double d = c[i - 1] - qn[j - 1];
            cur[j] = d * d + mn;
          }
          double* t = prev;
          prev = cur;
          cur = t;
        }
        const double dfull = prev[m];
        int b = 0;
        while (b < 6 && dfull / ub > dedges[b]) ++b;
        dr_tasks[b]++;
        dr_cells[b] += tc;
        /* LB_Improved(q, c): Keogh EQ total + Keogh of q against the envelope of
           the projection of c onto q's envelope */
        double* h = cbig;
        for (size_t k = 0; k < m; ++k) h[k] = c[k] > qu[k] ? qu[k] : (c[k] < ql[k] ? ql[k] : c[k]);
        double *hu = cu, *hl = cl;
        orc_compute_envelope(h, m, w, hu, hl);
        double e2 = 0;
        for (size_t k = 0; k < m; ++k) {
          const double x = qn[k];
          if (x > hu[k]) e2 += (x - hu[k]) * (x - hu[k]);
          else if (x < hl[k]) e2 += (x - hl[k]) * (x - hl[k]);
        }
        {  /* the same pruned DP on the reversed pair (thresholds from the reversed contributions) */
          double *rc = malloc(m * 8), *rq = malloc(m * 8), *rcon = malloc(m * 8), *rcb = malloc(m * 8);
          const double* con = tec > teq ? cec : ceq;
          for (size_t k = 0; k < m; ++k) {
            rc[k] = c[m - 1 - k];
            rq[k] = qn[m - 1 - k];
            rcon[k] = con[m - 1 - k];
          }
          orc_cumulative_bound(rcon, m, rcb);
          long long rcc = 0, fcc = 0;
          int *rcf = calloc(m + 2, sizeof(int)), *rcr = calloc(m + 2, sizeof(int));
          double *slf = malloc((m + 2) * 8), *slr = malloc((m + 2) * 8);
          for (size_t k = 0; k <= m + 1; ++k) slf[k] = slr[k] = -1;
          pruned_rows(c, qn, cbnd, m, w, ub, prev, cur, &fcc, rcf, slf);
          const int rr = pruned_rows(rc, rq, rcb, m, w, ub, prev, cur, &rcc, rcr, slr);
          for (int pi = 0; pi < 4; ++pi) {
            const int K = pks[pi];
            long long pf = 0, pr = 0;  /* cells in the first K rows */
            for (int k = 1; k <= K && k <= (int)m; ++k) {
              pf += rcf[k];
              pr += rcr[k];
            }
            const int fdead = rcf[K] == 0, rdead = rcr[K] == 0;
            for (int crit = 0; crit < 2; ++crit) {
              long long cost;
              if (fdead || rdead) cost = fdead && rdead ? pf + pr : (fdead ? 2 * pf : 2 * pr);
              else {
                int pick_rev = crit == 0 ? slr[K] < slf[K] : rcr[K] < rcf[K];
                cost = pf + pr + (pick_rev ? rcc - pr : fcc - pf);
              }
              /* when one died within K rows, the other was run only as long */
              if (fdead && !rdead) cost = pf + (pr < pf ? pr : pf) + 0;
              if (rdead && !fdead) cost = pr + (pf < pr ? pf : pr);
              pk_cells[pi][crit] += cost;
            }
          }
          {
            const int K = 32;
            long long pf = 0, pr = 0;
            for (int k = 1; k <= K; ++k) {
              pf += rcf[k];
              pr += rcr[k];
            }
            const int fdead = rcf[K] == 0, rdead = rcr[K] == 0;
            for (int crit = 0; crit < 3; ++crit) {
              long long cost;
              if (fdead || rdead) {
                cost = fdead && rdead ? pf + pr : (fdead ? pf + (pr < pf ? pr : pf) : pr + (pf < pr ? pf : pr));
              } else {
                const double tf = ub - cbnd[K + w - 1], tr = ub - rcb[K + w - 1];
                double sf = slf[K], sr = slr[K];
                int pick_rev;
                if (crit == 0) pick_rev = sr / tr < sf / tf;
                else if (crit == 1) {
                  const double gf = (slf[K / 2] - sf) / (K / 2), gr = (slr[K / 2] - sr) / (K / 2);
                  const double df = gf > 0 ? sf / gf : 1e30, dr = gr > 0 ? sr / gr : 1e30;
                  pick_rev = dr < df;
                } else pick_rev = sr * rcr[K] < sf * rcf[K];
                cost = pf + pr + (pick_rev ? rcc - pr : fcc - pf);
              }
              alt_cells[crit] += cost;
            }
          }
          {  /* probe 32 both ways, pick by slack, continue with the other probe's excess added to cb */
            const int K = 32;
            long long pf = 0, pr = 0;
            for (int k = 1; k <= K; ++k) { pf += rcf[k]; pr += rcr[k]; }
            const int fdead = rcf[K] == 0, rdead = rcr[K] == 0;
            long long cost, plain;
            if (fdead || rdead) {
              cost = fdead && rdead ? pf + pr : (fdead ? pf + (pr < pf ? pr : pf) : pr + (pf < pr ? pf : pr));
              plain = cost;
            } else {
              const int pick_rev = slr[K] < slf[K];
              const size_t kkK = (K + w < m ? K + w : m) - 1;
              plain = pf + pr + (pick_rev ? rcc - pr : fcc - pf);
              long long tcells = 0;
              if (!pick_rev) {
                /* forward continues; reverse probe's frontier minimum replaces the last 32 positions' bound */
                const double rmin = (ub - rcb[kkK]) - slr[K];
                const double tail = cbnd[m - 33];
                g_extra = rmin > tail ? rmin - tail : 0.0;
                g_kk_limit = m - 33;
                pruned_rows(c, qn, cbnd, m, w, ub, prev, cur, &tcells, NULL, NULL);
              } else {
                const double fmin = (ub - cbnd[kkK]) - slf[K];
                const double head = rcb[m - 33];
                g_extra = fmin > head ? fmin - head : 0.0;
                g_kk_limit = m - 33;
                pruned_rows(rc, rq, rcb, m, w, ub, prev, cur, &tcells, NULL, NULL);
              }
              g_extra = 0.0;
              const long long own = pick_rev ? pr : pf;
              cost = pf + pr + (tcells > own ? tcells - own : 0);
            }
            comb_cells += cost;
            comb_plain += plain;
          }
          /* greedy race: after one strip each, always advance the direction
             with less slack at its frontier; stop when either dies */
          for (int gi = 0; gi < 3; ++gi) {
            const int S = 16 << gi;
            int a = 0, b = 0;  /* rows done fwd / rev */
            long long cost = 0;
            int dead = 0;
            for (int it = 0; !dead; ++it) {
              int adv_rev;
              if (it == 0) adv_rev = 0;
              else if (it == 1) adv_rev = 1;
              else adv_rev = slr[b] < slf[a];
              int* rc_ = adv_rev ? rcr : rcf;
              int* fr = adv_rev ? &b : &a;
              for (int k = 0; k < S && !dead; ++k) {
                const int row = *fr + 1;
                if (row > (int)m) { dead = 1; break; }
                cost += rc_[row];
                *fr = row;
                if (rc_[row] == 0) dead = 1;
              }
            }
            greedy_cells[gi] += cost;
          }
          free(rcf); free(rcr); free(slf); free(slr);
          rev_rows += rr;
          rev_cells += rcc;
          min_rows += rr < rows ? rr : rows;
          /* racing both directions at equal speed costs 2 x the cells of the
             shorter one (approximated by rows) */
          min_cells2 += rr < rows ? 2 * rcc : 2 * tc;
          best_cells += rcc < tc ? rcc : tc;
          /* predictor: the direction whose first 64 rows carry more of the
             bound's mass (its thresholds start lower) */
          double pf = 0, pr = 0;
          for (size_t k = 0; k < 64; ++k) {
            pf += con[k];
            pr += con[m - 1 - k];
          }
          pred_cells += pr > pf ? rcc : tc;
          free(rc); free(rq); free(rcon); free(rcb);
        }
        double imp = teq + e2;
        if (imp > ub) {
          imp_tasks++;
          imp_cells += tc;
        }
      }
      int b = 0;
      while (b < 11 && maxw > edges[b]) ++b;
      maxhist[b]++;
      cells_by_max[b] += tc;
    }
    free(c); free(cu); free(cl); free(ceq); free(cec); free(cbnd); free(cbig);
    free(prev); free(cur); free(cen);
  }
  printf("N %zu candidates %zu DTW tasks %lld (%.3f%%), rows/task %.1f, live cells/task %.0f\n", N, nc,
         tasks, 100.0 * tasks / nc, (double)rows_sum / tasks, (double)cells / tasks);
  printf("width edges   <=16 32 48 64 88 104 128 144 192 256 384 >384\n");
  printf("rows by width:");
  for (int b = 0; b < 12; ++b) printf(" %lld", whist[b]);
  printf("\ntasks by max width:");
  for (int b = 0; b < 12; ++b) printf(" %lld", maxhist[b]);
  printf("\nlive cells by task max width (%%):");
  for (int b = 0; b < 12; ++b) printf(" %.1f", 100.0 * cells_by_max[b] / cells);
  printf("\nrows survived (0,1,2,<=4,8,16,32,64,128,256,512,>512): tasks");
  for (int b = 0; b < 12; ++b) printf(" %lld", rowhist[b]);
  printf(" | cells %%");
  for (int b = 0; b < 12; ++b) printf(" %.1f", 100.0 * rowcells[b] / cells);
  printf("\nEQ-only thresholds, rows survived of the first 16:");
  for (int b = 0; b < 12; ++b) printf(" %lld", eqrow_hist[b]);
  printf("\ncentre drift per 16 rows (<=2,4,8,16,32,64,128,>128):");
  for (int b = 0; b < 8; ++b) printf(" %lld", drift_hist[b]);
  printf("\nby d/ub (<=1,1.1,1.25,1.5,2,3,>3): tasks");
  for (int b = 0; b < 7; ++b) printf(" %lld", dr_tasks[b]);
  printf(" | live cells %%");
  for (int b = 0; b < 7; ++b) printf(" %.1f", 100.0 * dr_cells[b] / cells);
  printf("\nreverse direction: rows/task %.1f live cells/task %.0f | min(fwd, rev) rows/task %.1f | race both (2x shorter) cells/task %.0f",
         (double)rev_rows / tasks, (double)rev_cells / tasks, (double)min_rows / tasks, (double)min_cells2 / tasks);
  printf("\nbest direction (oracle) cells/task %.0f | predicted direction cells/task %.0f",
         (double)best_cells / tasks, (double)pred_cells / tasks);
  for (int pi = 0; pi < 4; ++pi)
    printf("\nprobe %d rows both ways, then the one with less slack: %.0f cells/task, fewer live: %.0f",
           pks[pi], (double)pk_cells[pi][0] / tasks, (double)pk_cells[pi][1] / tasks);
  printf("\ngreedy least-slack race, strips of 16/32/64 rows: %.0f %.0f %.0f cells/task",
         (double)greedy_cells[0] / tasks, (double)greedy_cells[1] / tasks, (double)greedy_cells[2] / tasks);
  printf("\nprobe 32 + other probe's excess in cb: %.0f cells/task (plain probe 32: %.0f)", (double)comb_cells / tasks, (double)comb_plain / tasks);
  printf("\nK=32 criteria: slack/T %.0f, extrapolated death %.0f, slack*live %.0f cells/task",
         (double)alt_cells[0] / tasks, (double)alt_cells[1] / tasks, (double)alt_cells[2] / tasks);
  printf("\nLB_Improved(EQ) > ub: %lld tasks (%.1f%%), %.1f%% of live cells\n", imp_tasks,
         100.0 * imp_tasks / tasks, 100.0 * imp_cells / cells);
  return 0;
}
