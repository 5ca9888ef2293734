// The multi-device C ABI through the shim (eapdtw_b200::MultiDevice), N = 1:
// the same answers as the single-device calls, exactly as a reference caller
// of similarity_search / the NN1 loop would drive it.
#include <cstdio>
#include <vector>

#include "eapdtw_b200.hpp"

using namespace eapdtw_b200;

static int failures = 0;
#define CHECK(x)                                              \
  do {                                                        \
    if (!(x)) {                                               \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #x); \
      ++failures;                                             \
    }                                                         \
  } while (0)

int main() {
  MultiDevice mg(std::vector<int>{0});
  CHECK(mg.device_count() == 1);
  const Series ref = random_walk(250000, 20260809);
  const Series q = random_walk(512, 414243);
  for (const double ratio : {0.05, 0.2}) {
    SearchConfig cfg;
    cfg.query_length = 200;
    cfg.window_ratio = ratio;
    const SearchResult one = similarity_search(ref, q, cfg);
    for (const int batches : {1, 3}) {
      const SearchResult multi = mg.similarity_search(ref, q, cfg, batches);
      CHECK(multi.best.found == one.best.found);
      CHECK(multi.best.location == one.best.location);
      CHECK(multi.best.distance_sq == one.best.distance_sq);
      CHECK(multi.report.candidates_total == one.report.candidates_total);
    }
  }
  // NN1: 8 queries x 500 rows of length 64, unbounded band
  const std::size_t len = 64, nq = 8, nd = 500;
  std::vector<double> qs, db;
  for (std::size_t k = 0; k < nq; ++k) {
    const Series s = random_walk(len, 1000 + k);
    const RunningStats st = RunningStats::over(s.view());
    std::vector<double> z(len);
    znormalize_into(s.view(), st, z);
    qs.insert(qs.end(), z.begin(), z.end());
  }
  for (std::size_t k = 0; k < nd; ++k) {
    const Series s = random_walk(len, 5000 + k);
    std::vector<double> z(len);
    znormalize_into(s.view(), RunningStats::over(s.view()), z);
    db.insert(db.end(), z.begin(), z.end());
  }
  std::vector<std::size_t> arg;
  std::vector<double> dist;
  mg.nn1(qs, db, len, Band::unbounded(), arg, dist, 3);
  for (std::size_t i = 0; i < nq; ++i) {  // the reference's loop: strict <, first index wins
    double best = PRUNED;
    std::size_t at = 0;
    const std::span<const double> qi(qs.data() + i * len, len);
    for (std::size_t k = 0; k < nd; ++k) {
      const double d = ea_pruned_dtw(std::span<const double>(db.data() + k * len, len), qi, best);
      if (d < best) {
        best = d;
        at = k;
      }
    }
    CHECK(arg[i] == at);
    CHECK(dist[i] == best);
  }
  if (failures == 0) std::printf("OK\n");
  return failures == 0 ? 0 : 1;
}
