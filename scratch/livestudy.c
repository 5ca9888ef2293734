// Live-region study: for LB survivors of cfg4, per-row live ranges of the
// pruned DTW (cells with value <= thr(row)), in band coordinates e = j - i.
// usage: livestudy Z.bin Q.bin CB.bin m w ub count
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

int main(int argc, char** argv) {
  const int m = atoi(argv[4]), w = atoi(argv[5]);
  const double ub = atof(argv[6]);
  const int cnt = atoi(argv[7]);
  FILE* per = argc > 8 && argv[8][0] != '-' ? fopen(argv[8], "w") : NULL;
  double* CC = NULL;
  if (argc > 9) { CC = malloc(sizeof(double) * m * cnt); FILE* g = fopen(argv[9], "rb"); if (fread(CC, 8, (size_t)m * cnt, g)) {} fclose(g); }
  long long cells_before = 0;
  double* Z = malloc(sizeof(double) * m * cnt);
  double* Q = malloc(sizeof(double) * m);
  double* CB = malloc(sizeof(double) * m * cnt);
  FILE* f = fopen(argv[1], "rb"); fread(Z, 8, (size_t)m * cnt, f); fclose(f);
  f = fopen(argv[2], "rb"); fread(Q, 8, m, f); fclose(f);
  f = fopen(argv[3], "rb"); fread(CB, 8, (size_t)m * cnt, f); fclose(f);
  double* prev = malloc(sizeof(double) * (m + 2));
  double* cur = malloc(sizeof(double) * (m + 2));
  long long hist_rows[12] = {0};    // rows survived, log2 bins
  long long width_hist[10] = {0};   // per-row live width: <=8,16,24,32,48,64,96,128,256,>256
  long long span32_hist[10] = {0};  // per 32-row strip: span of live e (max-min+1)
  long long span8_hist[10] = {0};   // per 8-row group
  long long cells = 0, rows_total = 0;
  const int edges[9] = {8, 16, 24, 32, 48, 64, 96, 128, 256};
  for (int c = 0; c < cnt; ++c) {
    const double* z = Z + (size_t)c * m;
    const double* cb = CB + (size_t)c * m;
    for (int j = 0; j <= m + 1; ++j) prev[j] = INFINITY;
    prev[0] = 0.0;
    int rows = 0;
    int smin32 = 1 << 30, smax32 = -(1 << 30), smin8 = 1 << 30, smax8 = -(1 << 30);
    for (int i = 1; i <= m; ++i) {
      const double thr = ub - cb[i - 1];
      cur[0] = INFINITY;
      int lo = 1 << 30, hi = -1;
      const int bl = i - w > 1 ? i - w : 1, bh = i + w < m ? i + w : m;
      for (int j = 1; j <= m; ++j) {
        if (j < bl || j > bh) { cur[j] = INFINITY; continue; }
        const double d = z[i - 1] - Q[j - 1];
        double mn = prev[j - 1];
        if (prev[j] < mn) mn = prev[j];
        if (cur[j - 1] < mn) mn = cur[j - 1];
        double v = d * d + mn;
        double t2 = thr;
        if (CC) { double cc = CC[(size_t)c * m + j - 1]; double tc = ub - cc; if (tc < t2) t2 = tc; }
        if (v > t2) v = INFINITY;
        cur[j] = v;
        if (v != INFINITY) { if (j < lo) lo = j; hi = j; ++cells; }
      }
      if (hi < 0) break;
      ++rows;
      int width = hi - lo + 1, b = 0;
      while (b < 9 && width > edges[b]) ++b;
      width_hist[b]++;
      const int elo = lo - i, ehi = hi - i;
      if (elo < smin32) smin32 = elo;
      if (ehi > smax32) smax32 = ehi;
      if (elo < smin8) smin8 = elo;
      if (ehi > smax8) smax8 = ehi;
      if (i % 32 == 0) {
        int s = smax32 - smin32 + 1; b = 0; while (b < 9 && s > edges[b]) ++b; span32_hist[b]++;
        smin32 = 1 << 30; smax32 = -(1 << 30);
      }
      if (i % 8 == 0) {
        int s = smax8 - smin8 + 1; b = 0; while (b < 9 && s > edges[b]) ++b; span8_hist[b]++;
        smin8 = 1 << 30; smax8 = -(1 << 30);
      }
      double* t = prev; prev = cur; cur = t;
    }
    rows_total += rows;
    if (per) fprintf(per, "%d %lld\n", rows, cells - cells_before);
    cells_before = cells;
    int b = 0; while ((1 << b) < rows + 1 && b < 11) ++b;
    hist_rows[b]++;
  }
  printf("candidates %d, rows/cand %.1f, live cells/cand %.0f, cells/row %.1f\n", cnt,
         (double)rows_total / cnt, (double)cells / cnt, (double)cells / rows_total);
  printf("rows survived (<=2^b):");
  for (int b = 0; b < 12; ++b) printf(" %lld", hist_rows[b]);
  printf("\nrow width  (<=8,16,24,32,48,64,96,128,256,>256):");
  for (int b = 0; b < 10; ++b) printf(" %lld", width_hist[b]);
  printf("\n8-row span:");
  for (int b = 0; b < 10; ++b) printf(" %lld", span8_hist[b]);
  printf("\n32-row span:");
  for (int b = 0; b < 10; ++b) printf(" %lld", span32_hist[b]);
  printf("\n");
  if (per) fclose(per);
  return 0;
}
