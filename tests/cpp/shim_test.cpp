// Drop-in check of include/eapdtw_b200.hpp: the reference's own worked example
// and contract cases (proj/tests/test_dtw.cpp:53-149, test_search.cpp:143-158)
// written against the B200 shim, exactly as a reference caller would.
#include <cstdio>
#include <vector>

#include "eapdtw_b200.hpp"

using namespace eapdtw_b200;

static int failures = 0;
#define CHECK(x)                                            \
  do {                                                      \
    if (!(x)) {                                             \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #x); \
      ++failures;                                           \
    }                                                       \
  } while (0)

int main() {
  const Series s(std::vector<double>{3, 1, 4, 4, 1, 1});
  const Series t(std::vector<double>{1, 3, 2, 1, 2, 2});
  CHECK(dtw_full(s, t) == 9.0);
  CHECK(dtw_windowed(s, t, Band::cells(0)) == 23.0);
  CHECK(ea_pruned_dtw(s, t, 9.0) == 9.0);
  CHECK(is_pruned(ea_pruned_dtw(s, t, 6.0)));
  CHECK(is_pruned(ea_pruned_dtw_windowed(s, t, Band::cells(0), 22.0)));
  CHECK(ea_pruned_dtw_windowed(s, t, Band::cells(0), 23.0) == 23.0);
  CHECK(dtw_left_prune(s.view(), t.view(), 9.0) == 9.0);
  {  // KernelTrace capture (test_dtw.cpp / cli_tests.cpp:176-204): eap at ub 6
     // abandons at (5,3) = 7; the full kernel evaluates all 36 cells, (6,6) = 9
    KernelTrace tr;
    tr.capture_cells = true;
    CHECK(is_pruned(ea_pruned_dtw(s.view(), t.view(), 6.0, tr)));
    CHECK(tr.abandon_cell && tr.abandon_cell->row == 5 && tr.abandon_cell->col == 3);
    CHECK(!tr.cells.empty() && tr.cells.back().value == 7.0);
    CHECK(tr.cells_evaluated == tr.cells.size());
    CHECK(!tr.discard_points.empty() && !tr.pruning_points.empty());
    KernelTrace fu;
    fu.capture_cells = true;
    CHECK(dtw_full(s.view(), t.view(), fu) == 9.0);
    CHECK(fu.cells.size() == 36 && fu.cells.back().row == 6 && fu.cells.back().col == 6);
    KernelTrace lp;
    lp.capture_cells = true;
    CHECK(is_pruned(dtw_left_prune(s.view(), t.view(), 6.0, lp)));
    CHECK(lp.abandon_cell && lp.abandon_cell->row == 5);
  }
  bool threw = false;
  try {
    const std::vector<double> bad = {1.0, 0.0};
    (void)ea_pruned_dtw_windowed(s.view(), t.view(), Band::unbounded(), 10.0, bad);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
  threw = false;
  try {
    Series empty(std::vector<double>{});
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);

  // exact normalised copy at distance 0 (integer samples keep sums exact)
  std::vector<double> ref(2000), q(48);
  unsigned long long x = 12345;
  for (auto& v : ref) { x = x * 6364136223846793005ull + 1442695040888963407ull; v = double((x >> 33) % 13) - 6.0; }
  for (auto& v : q) { x = x * 6364136223846793005ull + 1442695040888963407ull; v = double((x >> 33) % 13) - 6.0; }
  for (int k = 0; k < 48; ++k) ref[700 + k] = q[k];
  SearchConfig cfg;
  cfg.window_ratio = 0.1;
  const SearchResult r = similarity_search(Series(ref), Series(q), cfg);
  CHECK(r.best.found);
  CHECK(r.best.location == 700);
  CHECK(r.best.distance_sq == 0.0);
  CHECK(r.report.candidates_total == 2000 - 48 + 1);
  CHECK(r.report.candidates_total == r.report.pruned_kim + r.report.pruned_keogh_eq +
                                         r.report.pruned_keogh_ec + r.report.dtw_calls);
  std::printf("report: total=%zu kim=%zu eq=%zu ec=%zu calls=%zu abandoned=%zu cells=%zu\n",
              r.report.candidates_total, r.report.pruned_kim, r.report.pruned_keogh_eq,
              r.report.pruned_keogh_ec, r.report.dtw_calls, r.report.dtw_abandoned,
              r.report.dp_cells_evaluated);
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
