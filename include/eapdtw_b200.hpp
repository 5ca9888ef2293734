// eapdtw_b200.hpp -- the reference's public C++ API (proj/include/eapdtw/*.hpp)
// re-exposed on top of the B200 C ABI (eapdtw_b200.h).  Header-only; link with
// libeapdtw_b200.so.
//
// Same names, argument meaning and error behaviour as the reference, so a
// caller of the reference switches by changing the namespace:
//   eapdtw::ea_pruned_dtw_windowed (dtw.hpp:93-99)  -> eapdtw_b200::ea_pruned_dtw_windowed
//   eapdtw::ea_pruned_dtw          (dtw.hpp:85-87)  -> eapdtw_b200::ea_pruned_dtw
//   eapdtw::dtw_windowed           (dtw.hpp:72-74)  -> eapdtw_b200::dtw_windowed
//   eapdtw::dtw_left_prune(_windowed) (dtw.hpp:76-83) -> same names (the GPU
//        left-pruning schedule, left_prune_scan dtw.cpp:130-182)
//   eapdtw::similarity_search      (search.hpp:118-119) -> eapdtw_b200::similarity_search
//   lower_bounds.hpp (Envelope, compute_envelope, lb_kim_fl, BoundResult,
//        lb_keogh, cumulative_bound), search.hpp (RunningStats,
//        znormalize_into, cascade_decision, tighten_threshold) and io.hpp's
//        random_walk -> same names.
// Every overload that takes a KernelTrace runs the device trace kernel
// (eapdtw_trace: one thread, the reference's schedule and event order), so
// cells_evaluated, discard / pruning points and the abandon cell have the
// reference's meaning; the other overloads run the production kernels.
// include/compat/eapdtw/*.hpp map the reference's include paths and
// namespace onto this header.
// Invalid input throws std::invalid_argument exactly where the reference does;
// a CUDA failure throws std::runtime_error.  There is no CPU fallback.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <limits>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "eapdtw_b200.h"

namespace eapdtw_b200 {

inline constexpr double PRUNED = std::numeric_limits<double>::infinity();  // series.hpp:16
[[nodiscard]] inline bool is_pruned(double v) { return v == PRUNED; }      // series.hpp:18

namespace detail {
inline void check(int rc) {
  if (rc == EAPDTW_OK) return;
  const std::string msg = eapdtw_last_error();
  if (rc == EAPDTW_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error("eapdtw_b200: " + msg);
}

// One context per host thread (the C ABI serialises calls per context).
struct ThreadContext {
  eapdtw_ctx* ctx = nullptr;
  explicit ThreadContext(int device) { check(eapdtw_ctx_create(&ctx, device)); }
  ~ThreadContext() { eapdtw_ctx_destroy(ctx); }
  ThreadContext(const ThreadContext&) = delete;
  ThreadContext& operator=(const ThreadContext&) = delete;
};

inline eapdtw_ctx* context() {
  thread_local ThreadContext tc(0);
  return tc.ctx;
}
}  // namespace detail

// series.hpp:22-50
class Series {
 public:
  explicit Series(std::vector<double> samples) : samples_(std::move(samples)) {
    if (samples_.empty()) throw std::invalid_argument("Series: empty input");
    for (std::size_t i = 0; i < samples_.size(); ++i)
      if (!std::isfinite(samples_[i]))
        throw std::invalid_argument("Series: non-finite sample at index " + std::to_string(i));
  }
  [[nodiscard]] std::size_t length() const { return samples_.size(); }
  [[nodiscard]] double operator[](std::size_t i) const { return samples_[i]; }
  [[nodiscard]] const double* data() const { return samples_.data(); }
  [[nodiscard]] std::span<const double> view() const { return samples_; }
  [[nodiscard]] const std::vector<double>& samples() const { return samples_; }

 private:
  std::vector<double> samples_;
};

// dtw.hpp:60-63
[[nodiscard]] inline double squared_cost(double a, double b) {
  const double d = a - b;
  return d * d;
}

// dtw.hpp:16-23
struct Band {
  static constexpr std::size_t unbounded_window = EAPDTW_UNBOUNDED_WINDOW;
  std::size_t window = unbounded_window;
  [[nodiscard]] static constexpr Band unbounded() { return Band{unbounded_window}; }
  [[nodiscard]] static constexpr Band cells(std::size_t w) { return Band{w}; }
  [[nodiscard]] constexpr bool is_unbounded() const { return window == unbounded_window; }
};

// dtw.hpp:27-57.  Counters are always kept; with capture_cells set, the call
// runs the device trace (eapdtw_trace: one thread, the reference's event
// order) and fills cells / discard_points / pruning_points / abandon_cell.
struct CellRef {
  std::size_t row = 0;
  std::size_t col = 0;
  friend bool operator==(const CellRef&, const CellRef&) = default;
};
struct TraceCell {
  std::size_t row = 0;
  std::size_t col = 0;
  double value = 0.0;
};
struct KernelTrace {
  std::size_t cells_evaluated = 0;
  bool capture_cells = false;
  std::vector<TraceCell> cells;
  std::vector<CellRef> discard_points;
  std::vector<CellRef> pruning_points;
  std::optional<CellRef> abandon_cell;
  void reset() {
    cells_evaluated = 0;
    cells.clear();
    discard_points.clear();
    pruning_points.clear();
    abandon_cell.reset();
  }
};

namespace detail {
// algo: EAPDTW_ALGO_FULL / _LEFT_PRUNE / _EA_PRUNED
inline double traced(int algo, std::span<const double> a, std::span<const double> b,
                     std::size_t window, double ub, KernelTrace& trace) {
  const std::size_t lr = std::max(a.size(), b.size()), lc = std::min(a.size(), b.size());
  std::vector<eapdtw_trace_event> ev(2 * (lr + 2) * (lc + 2) + 8);
  std::size_t n = 0;
  uint64_t cells = 0;
  double out = PRUNED;
  check(eapdtw_trace(context(), algo, a.data(), a.size(), b.data(), b.size(), window, ub,
                     ev.data(), ev.size(), &n, &cells, &out));
  trace.cells_evaluated += cells;
  for (std::size_t k = 0; k < std::min(n, ev.size()); ++k) {
    const eapdtw_trace_event& e = ev[k];
    switch (e.kind) {
      case 0: trace.cells.push_back({e.row, e.col, e.value}); break;
      case 1: trace.discard_points.push_back({e.row, e.col}); break;
      case 2: trace.pruning_points.push_back({e.row, e.col}); break;
      default: trace.abandon_cell = CellRef{e.row, e.col}; break;
    }
  }
  return out;
}
}  // namespace detail

// --- DTW kernels, span level (dtw.hpp:69-99)
[[nodiscard]] inline double ea_pruned_dtw_windowed(std::span<const double> a,
                                                   std::span<const double> b, Band band, double ub,
                                                   std::span<const double> cumulative_bound,
                                                   KernelTrace& trace) {
  if (cumulative_bound.empty())
    return detail::traced(EAPDTW_ALGO_EA_PRUNED, a, b, band.window, ub, trace);
  double out = PRUNED;
  uint64_t cells = 0;
  detail::check(eapdtw_ea_pruned_dtw_windowed(detail::context(), a.data(), a.size(), b.data(),
                                              b.size(), band.window, ub, cumulative_bound.data(),
                                              cumulative_bound.size(), &out, &cells));
  trace.cells_evaluated += cells;
  return out;
}
[[nodiscard]] inline double ea_pruned_dtw_windowed(std::span<const double> a,
                                                   std::span<const double> b, Band band, double ub,
                                                   std::span<const double> cumulative_bound = {}) {
  double out = PRUNED;
  uint64_t cells = 0;
  detail::check(eapdtw_ea_pruned_dtw_windowed(detail::context(), a.data(), a.size(), b.data(),
                                              b.size(), band.window, ub, cumulative_bound.data(),
                                              cumulative_bound.size(), &out, &cells));
  return out;
}
[[nodiscard]] inline double ea_pruned_dtw(std::span<const double> a, std::span<const double> b,
                                          double ub) {
  return ea_pruned_dtw_windowed(a, b, Band::unbounded(), ub);
}
[[nodiscard]] inline double ea_pruned_dtw(std::span<const double> a, std::span<const double> b,
                                          double ub, KernelTrace& trace) {
  return ea_pruned_dtw_windowed(a, b, Band::unbounded(), ub, {}, trace);
}
[[nodiscard]] inline double dtw_windowed(std::span<const double> a, std::span<const double> b,
                                         Band band, KernelTrace& trace) {
  return detail::traced(EAPDTW_ALGO_FULL, a, b, band.window, PRUNED, trace);
}
[[nodiscard]] inline double dtw_windowed(std::span<const double> a, std::span<const double> b,
                                         Band band) {
  double out = PRUNED;
  uint64_t cells = 0;
  detail::check(eapdtw_dtw_windowed(detail::context(), a.data(), a.size(), b.data(), b.size(),
                                    band.window, &out, &cells));
  return out;
}
[[nodiscard]] inline double dtw_full(std::span<const double> a, std::span<const double> b) {
  return dtw_windowed(a, b, Band::unbounded());
}
[[nodiscard]] inline double dtw_full(std::span<const double> a, std::span<const double> b,
                                     KernelTrace& trace) {
  return dtw_windowed(a, b, Band::unbounded(), trace);
}
// Left pruning (left_prune_scan, dtw.cpp:130-182): the GPU's left-border-only
// schedule; same result contract as EAPrunedDTW (exact iff <= ub, else PRUNED).
[[nodiscard]] inline double dtw_left_prune_windowed(std::span<const double> a,
                                                    std::span<const double> b, Band band,
                                                    double ub, KernelTrace& trace) {
  return detail::traced(EAPDTW_ALGO_LEFT_PRUNE, a, b, band.window, ub, trace);
}
[[nodiscard]] inline double dtw_left_prune_windowed(std::span<const double> a,
                                                    std::span<const double> b, Band band,
                                                    double ub) {
  double out = PRUNED;
  uint64_t cells = 0;
  detail::check(eapdtw_dtw_left_prune_windowed(detail::context(), a.data(), a.size(), b.data(),
                                               b.size(), band.window, ub, &out, &cells));
  return out;
}
[[nodiscard]] inline double dtw_left_prune(std::span<const double> a, std::span<const double> b,
                                           double ub) {
  return dtw_left_prune_windowed(a, b, Band::unbounded(), ub);
}
[[nodiscard]] inline double dtw_left_prune(std::span<const double> a, std::span<const double> b,
                                           double ub, KernelTrace& trace) {
  return dtw_left_prune_windowed(a, b, Band::unbounded(), ub, trace);
}

// Series-level conveniences (dtw.hpp:103-135)
[[nodiscard]] inline double ea_pruned_dtw_windowed(const Series& a, const Series& b, Band band,
                                                   double ub,
                                                   std::span<const double> cumulative_bound = {}) {
  return ea_pruned_dtw_windowed(a.view(), b.view(), band, ub, cumulative_bound);
}
[[nodiscard]] inline double ea_pruned_dtw(const Series& a, const Series& b, double ub) {
  return ea_pruned_dtw(a.view(), b.view(), ub);
}
[[nodiscard]] inline double dtw_windowed(const Series& a, const Series& b, Band band) {
  return dtw_windowed(a.view(), b.view(), band);
}
[[nodiscard]] inline double dtw_full(const Series& a, const Series& b) {
  return dtw_full(a.view(), b.view());
}
[[nodiscard]] inline double dtw_left_prune(const Series& a, const Series& b, double ub) {
  return dtw_left_prune(a.view(), b.view(), ub);
}
[[nodiscard]] inline double ea_pruned_dtw(const Series& a, const Series& b, double ub,
                                          KernelTrace& trace) {
  return ea_pruned_dtw(a.view(), b.view(), ub, trace);
}
[[nodiscard]] inline double dtw_left_prune(const Series& a, const Series& b, double ub,
                                           KernelTrace& trace) {
  return dtw_left_prune(a.view(), b.view(), ub, trace);
}

// --- lower bounds (lower_bounds.hpp:12-63), on the device
struct Envelope {
  std::vector<double> upper;
  std::vector<double> lower;
  std::size_t window = 0;
  [[nodiscard]] std::size_t length() const { return upper.size(); }
};
[[nodiscard]] inline Envelope compute_envelope(std::span<const double> series, Band band) {
  Envelope env;
  env.upper.resize(series.size());
  env.lower.resize(series.size());
  detail::check(eapdtw_compute_envelope(detail::context(), series.data(), series.size(), band.window,
                                        env.upper.data(), env.lower.data()));
  env.window = band.is_unbounded() ? series.size() : std::min(band.window, series.size());
  return env;
}
[[nodiscard]] inline Envelope compute_envelope(const Series& series, Band band) {
  return compute_envelope(series.view(), band);
}
[[nodiscard]] inline double lb_kim_fl(std::span<const double> q, std::span<const double> c) {
  if (q.size() != c.size()) throw std::invalid_argument("lb_kim_fl: length mismatch");
  double out = 0.0;
  detail::check(eapdtw_lb_kim_fl(detail::context(), q.data(), c.data(), q.size(), &out));
  return out;
}
[[nodiscard]] inline double lb_kim_fl(const Series& q, const Series& c) {
  return lb_kim_fl(q.view(), c.view());
}
struct BoundResult {
  double total = 0.0;
  std::vector<double> contributions;
  bool abandoned = false;
};
[[nodiscard]] inline BoundResult lb_keogh(const Envelope& env, std::span<const double> series,
                                          double abandon_above = PRUNED,
                                          std::span<const std::size_t> order = {}) {
  if (env.upper.size() != env.lower.size()) throw std::invalid_argument("lb_keogh: malformed envelope");
  if (env.length() != series.size()) throw std::invalid_argument("lb_keogh: length mismatch");
  if (!order.empty() && order.size() != series.size())
    throw std::invalid_argument("lb_keogh: order/series length mismatch");
  BoundResult res;
  res.contributions.assign(series.size(), 0.0);
  int ab = 0;
  detail::check(eapdtw_lb_keogh(detail::context(), env.upper.data(), env.lower.data(),
                                series.data(), series.size(), abandon_above,
                                order.empty() ? nullptr : order.data(), &res.total,
                                res.contributions.data(), &ab));
  res.abandoned = ab != 0;
  return res;
}
[[nodiscard]] inline BoundResult lb_keogh(const Envelope& env, const Series& series,
                                          double abandon_above = PRUNED,
                                          std::span<const std::size_t> order = {}) {
  return lb_keogh(env, series.view(), abandon_above, order);
}
[[nodiscard]] inline std::vector<double> cumulative_bound(std::span<const double> contributions) {
  std::vector<double> cb(contributions.size(), 0.0);
  detail::check(eapdtw_cumulative_bound(detail::context(), contributions.data(),
                                        contributions.size(), cb.data()));
  return cb;
}

// --- search (search.hpp:16-119)
struct RunningStats {  // search.hpp:16-42
  double sum = 0.0;
  double sum_of_squares = 0.0;
  std::size_t count = 0;
  [[nodiscard]] static RunningStats over(std::span<const double> window) {
    RunningStats s;
    detail::check(eapdtw_running_stats_over(window.data(), window.size(), &s.sum,
                                            &s.sum_of_squares));
    s.count = window.size();
    return s;
  }
  void add(double x) {
    sum += x;
    sum_of_squares += x * x;
    ++count;
  }
  void remove(double x) {
    sum -= x;
    sum_of_squares -= x * x;
    --count;
  }
  [[nodiscard]] double mean() const { return sum / static_cast<double>(count); }
  [[nodiscard]] double variance() const {
    const double m = mean();
    const double v = sum_of_squares / static_cast<double>(count) - m * m;
    return v > 0.0 ? v : 0.0;
  }
  [[nodiscard]] double stddev() const { return std::sqrt(variance()); }
};
// search.hpp:46 (search.cpp:37-46)
inline void znormalize_into(std::span<const double> src, const RunningStats& stats,
                            std::span<double> dst) {
  detail::check(eapdtw_znormalize_into(src.data(), src.size(), stats.sum, stats.sum_of_squares,
                                       stats.count, dst.data()));
}
[[nodiscard]] inline Series znormalize(const Series& s, const RunningStats& stats) {
  std::vector<double> out(s.length());
  znormalize_into(s.view(), stats, out);
  return Series(std::move(out));
}

struct BestSoFar {
  std::size_t location = 0;
  double distance_sq = PRUNED;
  bool found = false;
};
enum class Algo : std::uint8_t { full, left_prune, ea_pruned };
[[nodiscard]] inline std::string to_string(Algo a) {  // search.cpp:52-60
  switch (a) {
    case Algo::full: return "full";
    case Algo::left_prune: return "lp";
    case Algo::ea_pruned: return "eap";
  }
  return "?";
}
struct SearchConfig {
  std::size_t query_length = 0;
  double window_ratio = 0.1;
  Algo algorithm = Algo::ea_pruned;
  bool use_lower_bounds = true;
  bool tighten_ub = true;
};
struct SearchReport {
  std::size_t candidates_total = 0;
  std::size_t pruned_kim = 0;
  std::size_t pruned_keogh_eq = 0;
  std::size_t pruned_keogh_ec = 0;
  std::size_t dtw_calls = 0;
  std::size_t dtw_abandoned = 0;
  std::size_t dp_cells_evaluated = 0;
  double elapsed_seconds = 0.0;
};
struct SearchResult {
  BestSoFar best;
  SearchReport report;
};

[[nodiscard]] inline SearchResult similarity_search(const Series& reference, const Series& query,
                                                    const SearchConfig& cfg) {
  eapdtw_search_config c{cfg.query_length, cfg.window_ratio, static_cast<int32_t>(cfg.algorithm),
                         cfg.use_lower_bounds ? 1 : 0, cfg.tighten_ub ? 1 : 0, 0};
  eapdtw_search_result r{};
  detail::check(eapdtw_similarity_search(detail::context(), reference.data(), reference.length(),
                                         query.data(), query.length(), &c, &r));
  SearchResult out;
  out.best = {static_cast<std::size_t>(r.location), r.distance_sq, r.found != 0};
  out.report = {r.candidates_total, r.pruned_kim,  r.pruned_keogh_eq,   r.pruned_keogh_ec,
                r.dtw_calls,        r.dtw_abandoned, r.dp_cells_evaluated, r.elapsed_seconds};
  return out;
}

// One host thread driving several GPUs (eapdtw_multi_*, NCCL between them):
// the same similarity_search over 100000-aligned reference shards, and the
// NN1 loop over a row-split database.
class MultiDevice {
 public:
  explicit MultiDevice(const std::vector<int>& devices) {
    detail::check(eapdtw_multi_create(&mg_, devices.data(), static_cast<int>(devices.size())));
  }
  ~MultiDevice() { eapdtw_multi_destroy(mg_); }
  MultiDevice(const MultiDevice&) = delete;
  MultiDevice& operator=(const MultiDevice&) = delete;
  [[nodiscard]] int device_count() const { return eapdtw_multi_device_count(mg_); }
  [[nodiscard]] SearchResult similarity_search(const Series& reference, const Series& query,
                                               const SearchConfig& cfg, int batches = 8) {
    eapdtw_search_config c{cfg.query_length, cfg.window_ratio,
                           static_cast<int32_t>(cfg.algorithm), cfg.use_lower_bounds ? 1 : 0,
                           cfg.tighten_ub ? 1 : 0, 0};
    eapdtw_search_result r{};
    detail::check(eapdtw_multi_similarity_search(mg_, reference.data(), reference.length(),
                                                 query.data(), query.length(), &c, batches, &r));
    SearchResult out;
    out.best = {static_cast<std::size_t>(r.location), r.distance_sq, r.found != 0};
    out.report = {r.candidates_total, r.pruned_kim,  r.pruned_keogh_eq,   r.pruned_keogh_ec,
                  r.dtw_calls,        r.dtw_abandoned, r.dp_cells_evaluated, r.elapsed_seconds};
    return out;
  }
  // queries: nq x len, db: nd x len (row-major); argmin / dist per query.
  void nn1(std::span<const double> queries, std::span<const double> db, std::size_t len,
           Band band, std::vector<std::size_t>& argmin, std::vector<double>& dist,
           int batches = 4) {
    const std::size_t nq = queries.size() / len, nd = db.size() / len;
    std::vector<uint64_t> a(nq);
    dist.assign(nq, PRUNED);
    detail::check(eapdtw_multi_nn1(mg_, queries.data(), nq, db.data(), nd, len, band.window,
                                   batches, a.data(), dist.data(), nullptr));
    argmin.assign(a.begin(), a.end());
  }

 private:
  eapdtw_multi* mg_ = nullptr;
};

// search.hpp:85-114: the cascade of one candidate, composed from the device
// helpers above in the reference's order (search.cpp:63-107).
enum class CascadeTier : std::uint8_t { none, kim, keogh_eq, keogh_ec };
struct CascadeWorkspace {
  std::vector<double> candidate_norm;
  std::vector<double> contrib_eq;
  std::vector<double> contrib_ec;
  std::vector<double> cumulative;
};
[[nodiscard]] inline CascadeTier cascade_decision(std::span<const double> query_norm,
                                                  const Envelope& query_env,
                                                  std::span<const std::size_t> order,
                                                  std::span<const double> candidate_raw,
                                                  const RunningStats& stats, const BestSoFar& bsf,
                                                  const SearchConfig& cfg, CascadeWorkspace& ws) {
  const std::size_t m = query_norm.size();
  ws.candidate_norm.resize(m);
  ws.cumulative.clear();
  if (!cfg.use_lower_bounds) {
    znormalize_into(candidate_raw, stats, ws.candidate_norm);
    return CascadeTier::none;
  }
  const double ub = bsf.found ? bsf.distance_sq : PRUNED;
  const double mean = stats.mean();
  const double sd = stats.stddev();
  const bool constant = sd < 1e-12;  // kMinStddev, search.cpp:13
  if (m >= 2) {
    const double c0 = constant ? 0.0 : (candidate_raw.front() - mean) / sd;
    const double cl = constant ? 0.0 : (candidate_raw.back() - mean) / sd;
    const double kim = squared_cost(query_norm.front(), c0) + squared_cost(query_norm.back(), cl);
    if (kim > ub) return CascadeTier::kim;
  }
  znormalize_into(candidate_raw, stats, ws.candidate_norm);
  const BoundResult eq = lb_keogh(query_env, ws.candidate_norm, ub, order);
  if (eq.total > ub) return CascadeTier::keogh_eq;
  ws.contrib_eq = eq.contributions;
  const Envelope cand_env = compute_envelope(ws.candidate_norm, Band::cells(query_env.window));
  const BoundResult ec = lb_keogh(cand_env, query_norm, ub, order);
  if (ec.total > ub) return CascadeTier::keogh_ec;
  ws.contrib_ec = ec.contributions;
  if (cfg.tighten_ub) {
    const auto& contrib = eq.total > ec.total ? ws.contrib_eq : ws.contrib_ec;
    ws.cumulative = cumulative_bound(contrib);
  }
  return CascadeTier::none;
}
[[nodiscard]] inline double tighten_threshold(const BestSoFar& bsf, std::span<const double> cb,
                                              std::size_t row, std::size_t window_cells) {
  if (cb.empty()) return bsf.distance_sq;  // search.cpp:109-115
  const std::size_t k = std::min(row + window_cells, cb.size());
  const double t = bsf.distance_sq - cb[k - 1];
  return t > 0.0 ? t : 0.0;
}

// io.hpp:33: seeded random walk, uniform steps in [-0.5, 0.5) (io.cpp:124-137)
[[nodiscard]] inline Series random_walk(std::size_t length, std::uint64_t seed) {
  if (length == 0) throw std::invalid_argument("random_walk: zero length");
  std::vector<double> v(length);
  detail::check(eapdtw_random_walk_uniform(length, seed, v.data()));
  return Series(std::move(v));
}

}  // namespace eapdtw_b200
