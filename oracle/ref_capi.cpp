// ref_capi.cpp -- extern "C" shim over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY (see oracle/eapdtw_oracle.c header).  oracle/Makefile
// compiles the reference's own hot-path sources in place
// (/root/reference/proj/src/{dtw,lower_bounds,search}.cpp) together with this
// file into oracle/_ref/libeapdtw_ref.so.  Nothing here re-implements the
// algorithm: every function forwards to the reference entry point it names.
// It exists so Python tests can (a) pin the C restatement against the real
// reference, and (b) time the reference on the host cores as the CPU baseline
// (bench.py --impl reference / cpu_baseline).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <mutex>
#include <random>
#include <span>
#include <stdexcept>
#include <thread>
#include <vector>

#include "eapdtw/dtw.hpp"
#include "eapdtw/io.hpp"
#include "eapdtw/lower_bounds.hpp"
#include "eapdtw/search.hpp"
#include "eapdtw/series.hpp"

using namespace eapdtw;

namespace {
constexpr int kOk = 0;
constexpr int kInval = 1;
constexpr int kOther = 2;
constexpr std::size_t kUnbounded = static_cast<std::size_t>(-1);

Band band_of(std::size_t w) { return w == kUnbounded ? Band::unbounded() : Band::cells(w); }

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return kOk;
  } catch (const std::invalid_argument&) {
    return kInval;
  } catch (...) {
    return kOther;
  }
}
}  // namespace

extern "C" {

struct ref_search_result {
  uint64_t location;
  double distance_sq;
  int32_t found;
  int32_t pad_;
  uint64_t candidates_total, pruned_kim, pruned_keogh_eq, pruned_keogh_ec, dtw_calls,
      dtw_abandoned, dp_cells_evaluated;
  double elapsed_seconds;
};

// dtw.hpp:69-99; algo 0 dtw_windowed, 1 dtw_left_prune_windowed, 2 ea_pruned_dtw_windowed
int ref_dtw(int algo, const double* a, size_t la, const double* b, size_t lb, size_t window,
            double ub, const double* cb, size_t cb_len, double* out, uint64_t* cells) {
  return guarded([&] {
    std::span<const double> sa(a, la), sb(b, lb);
    KernelTrace tr;
    const Band band = band_of(window);
    switch (algo) {
      case 0: *out = dtw_windowed(sa, sb, band, tr); break;
      case 1: *out = dtw_left_prune_windowed(sa, sb, band, ub, tr); break;
      case 2: *out = ea_pruned_dtw_windowed(sa, sb, band, ub, std::span<const double>(cb, cb_len), tr); break;
      default: throw std::invalid_argument("algo");
    }
    if (cells) *cells += tr.cells_evaluated;
  });
}

int ref_ea_pruned_dtw(const double* a, size_t la, const double* b, size_t lb, double ub,
                      double* out) {
  return guarded([&] { *out = ea_pruned_dtw(std::span<const double>(a, la), std::span<const double>(b, lb), ub); });
}

// lower_bounds.hpp:25
int ref_compute_envelope(const double* s, size_t l, size_t window, double* upper, double* lower) {
  return guarded([&] {
    const Envelope e = compute_envelope(std::span<const double>(s, l), band_of(window));
    std::copy(e.upper.begin(), e.upper.end(), upper);
    std::copy(e.lower.begin(), e.lower.end(), lower);
  });
}

// lower_bounds.hpp:52-54
int ref_lb_keogh(const double* upper, const double* lower, const double* x, size_t l,
                 double abandon_above, const size_t* order, double* total, double* contrib,
                 int* abandoned) {
  return guarded([&] {
    Envelope env;
    env.upper.assign(upper, upper + l);
    env.lower.assign(lower, lower + l);
    const BoundResult r = lb_keogh(env, std::span<const double>(x, l), abandon_above,
                                   order ? std::span<const std::size_t>(order, l) : std::span<const std::size_t>{});
    *total = r.total;
    if (contrib) std::copy(r.contributions.begin(), r.contributions.end(), contrib);
    if (abandoned) *abandoned = r.abandoned ? 1 : 0;
  });
}

int ref_cumulative_bound(const double* c, size_t l, double* cb) {
  return guarded([&] {
    const auto v = cumulative_bound(std::span<const double>(c, l));
    std::copy(v.begin(), v.end(), cb);
  });
}

// io.hpp random_walk (io.cpp:124-137): the reference's seeded test data.
int ref_random_walk(size_t n, uint64_t seed, double* out) {
  return guarded([&] {
    const Series s = random_walk(n, seed);
    std::copy(s.begin(), s.end(), out);
  });
}

// search.hpp:46 with RunningStats::over
int ref_znormalize(const double* src, size_t n, double* dst) {
  return guarded([&] {
    std::span<const double> s(src, n);
    znormalize_into(s, RunningStats::over(s), std::span<double>(dst, n));
  });
}

static void fill_result(const SearchResult& r, ref_search_result* out) {
  std::memset(out, 0, sizeof(*out));
  out->location = r.best.location;
  out->distance_sq = r.best.distance_sq;
  out->found = r.best.found ? 1 : 0;
  out->candidates_total = r.report.candidates_total;
  out->pruned_kim = r.report.pruned_kim;
  out->pruned_keogh_eq = r.report.pruned_keogh_eq;
  out->pruned_keogh_ec = r.report.pruned_keogh_ec;
  out->dtw_calls = r.report.dtw_calls;
  out->dtw_abandoned = r.report.dtw_abandoned;
  out->dp_cells_evaluated = r.report.dp_cells_evaluated;
  out->elapsed_seconds = r.report.elapsed_seconds;
}

// search.hpp:118-119
int ref_similarity_search(const double* ref, size_t n, const double* query, size_t qlen,
                          size_t query_length, double ratio, int algo, int use_lb, int tighten,
                          ref_search_result* out) {
  return guarded([&] {
    SearchConfig cfg;
    cfg.query_length = query_length;
    cfg.window_ratio = ratio;
    cfg.algorithm = static_cast<Algo>(algo);
    cfg.use_lower_bounds = use_lb != 0;
    cfg.tighten_ub = tighten != 0;
    const SearchResult r = similarity_search(Series(std::vector<double>(ref, ref + n)),
                                             Series(std::vector<double>(query, query + qlen)), cfg);
    fill_result(r, out);
  });
}

// CPU-baseline harness: the reference search sharded over host threads.
// Shard starts are multiples of 100000 candidates (the stats reset interval,
// search.cpp:16) and each shard carries an (m-1)-point halo, so every shard
// reproduces the unsharded stats chain; merge = (distance, lowest index).
// Each shard runs the unmodified similarity_search on its slice.
int ref_similarity_search_threads(const double* ref, size_t n, const double* query, size_t qlen,
                                  size_t query_length, double ratio, int algo, int use_lb,
                                  int tighten, int threads, ref_search_result* out) {
  const size_t m = query_length == 0 ? qlen : query_length;
  if (m == 0 || m > qlen || m > n) return kInval;
  const size_t ncand = n - m + 1;
  const size_t seg = 100000;
  const size_t nseg = (ncand + seg - 1) / seg;
  if (threads < 1) threads = 1;
  std::vector<ref_search_result> parts(nseg);
  std::vector<int> rc(nseg, 0);
  std::atomic<size_t> next{0};
  auto worker = [&] {
    for (;;) {
      const size_t k = next.fetch_add(1);
      if (k >= nseg) return;
      const size_t s0 = k * seg;
      const size_t s1 = std::min(ncand, s0 + seg);
      rc[k] = ref_similarity_search(ref + s0, (s1 - s0) + m - 1, query, qlen, m, ratio, algo,
                                    use_lb, tighten, &parts[k]);
      parts[k].location += s0;
    }
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) pool.emplace_back(worker);
  for (auto& t : pool) t.join();
  ref_search_result best{};
  best.distance_sq = std::numeric_limits<double>::infinity();
  for (size_t k = 0; k < nseg; ++k) {
    if (rc[k]) return rc[k];
    const auto& p = parts[k];
    if (p.found && (!best.found || p.distance_sq < best.distance_sq)) {
      best.found = 1;
      best.distance_sq = p.distance_sq;
      best.location = p.location;
    }
    best.candidates_total += p.candidates_total;
    best.pruned_kim += p.pruned_kim;
    best.pruned_keogh_eq += p.pruned_keogh_eq;
    best.pruned_keogh_ec += p.pruned_keogh_ec;
    best.dtw_calls += p.dtw_calls;
    best.dtw_abandoned += p.dtw_abandoned;
    best.dp_cells_evaluated += p.dp_cells_evaluated;
    best.elapsed_seconds += p.elapsed_seconds;
  }
  *out = best;
  return kOk;
}

// cfg1 harness: pairs split over threads, each pair ea_pruned_dtw_windowed.
int ref_pairwise_threads(const double* a, const double* b, size_t npairs, size_t len,
                         size_t window, const double* ub, int threads, double* out,
                         uint64_t* cells) {
  std::atomic<size_t> next{0};
  std::atomic<uint64_t> total{0};
  std::atomic<int> err{0};
  auto worker = [&] {
    uint64_t local = 0;
    for (;;) {
      const size_t p = next.fetch_add(1);
      if (p >= npairs) break;
      const int e = ref_dtw(2, a + p * len, len, b + p * len, len, window,
                            ub ? ub[p] : std::numeric_limits<double>::infinity(), nullptr, 0,
                            &out[p], &local);
      if (e) err = e;
    }
    total += local;
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < std::max(1, threads); ++t) pool.emplace_back(worker);
  for (auto& t : pool) t.join();
  if (cells) *cells = total;
  return err;
}

// cfg5 harness: queries split over threads; per query a running cutoff over
// the database with ea_pruned_dtw_windowed (strict < keeps the lowest index).
int ref_nn1_threads(const double* queries, size_t nq, const double* db, size_t nd, size_t len,
                    size_t window, int threads, uint64_t* argmin, double* dist, uint64_t* cells) {
  std::atomic<size_t> next{0};
  std::atomic<uint64_t> total{0};
  std::atomic<int> err{0};
  auto worker = [&] {
    uint64_t local = 0;
    for (;;) {
      const size_t q = next.fetch_add(1);
      if (q >= nq) break;
      double bsf = std::numeric_limits<double>::infinity();
      uint64_t arg = 0;
      for (size_t k = 0; k < nd; ++k) {
        double d;
        const int e = ref_dtw(2, db + k * len, len, queries + q * len, len, window, bsf, nullptr,
                              0, &d, &local);
        if (e) err = e;
        if (d < bsf) {
          bsf = d;
          arg = k;
        }
      }
      argmin[q] = arg;
      dist[q] = bsf;
    }
    total += local;
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < std::max(1, threads); ++t) pool.emplace_back(worker);
  for (auto& t : pool) t.join();
  if (cells) *cells = total;
  return err;
}

// ---- file formats (io.cpp), used only to generate tests/golden/io_golden.json ----

// io.cpp:50-55; writes at most cap-1 chars + NUL
int ref_format_double(double v, char* buf, size_t cap) {
  return guarded([&] {
    const std::string s = format_double(v);
    std::snprintf(buf, cap, "%s", s.c_str());
  });
}

// io.cpp:57-74 (SearchReport/BestSoFar from a ref_search_result)
int ref_emit_stats(const ref_search_result* r, const char* path) {
  return guarded([&] {
    SearchReport rep;
    rep.candidates_total = r->candidates_total;
    rep.pruned_kim = r->pruned_kim;
    rep.pruned_keogh_eq = r->pruned_keogh_eq;
    rep.pruned_keogh_ec = r->pruned_keogh_ec;
    rep.dtw_calls = r->dtw_calls;
    rep.dtw_abandoned = r->dtw_abandoned;
    rep.dp_cells_evaluated = r->dp_cells_evaluated;
    rep.elapsed_seconds = r->elapsed_seconds;
    BestSoFar best;
    best.location = r->location;
    best.distance_sq = r->distance_sq;
    best.found = r->found != 0;
    emit_stats(rep, best, path);
  });
}

// io.cpp:17-42; on failure copies the exception message into err
int ref_load_series(const char* path, double* out, size_t cap, size_t* n, char* err,
                    size_t errcap) {
  try {
    const Series s = load_series(path);
    *n = s.length();
    std::copy_n(s.begin(), std::min(cap, s.length()), out);
    return kOk;
  } catch (const std::exception& e) {
    std::snprintf(err, errcap, "%s", e.what());
    return kOther;
  }
}

// run_trace (eapdtw_cli.cpp:91-108) generalised to a band: the traced kernel
// (dtw.hpp:69-99 KernelTrace overloads) + write_trace_csv (io.cpp:76-122).
int ref_trace_csv(int algo, const double* a, size_t la, const double* b, size_t lb, size_t window,
                  double ub, const char* path, double* out, uint64_t* cells) {
  return guarded([&] {
    std::span<const double> sa(a, la), sb(b, lb);
    KernelTrace trace;
    trace.capture_cells = true;
    const Band band = band_of(window);
    switch (algo) {
      case 0: *out = dtw_windowed(sa, sb, band, trace); break;
      case 1: *out = dtw_left_prune_windowed(sa, sb, band, ub, trace); break;
      case 2: *out = ea_pruned_dtw_windowed(sa, sb, band, ub, {}, trace); break;
      default: throw std::invalid_argument("algo");
    }
    *cells = trace.cells_evaluated;
    write_trace_csv(trace, path);
  });
}

// io.cpp:44-48
int ref_save_series(const double* s, size_t n, const char* path) {
  return guarded([&] { save_series(Series(std::vector<double>(s, s + n)), path); });
}

}  // extern "C"
