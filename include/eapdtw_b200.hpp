// eapdtw_b200.hpp -- the reference's public C++ API (proj/include/eapdtw/*.hpp)
// re-exposed on top of the B200 C ABI (eapdtw_b200.h).  Header-only; link with
// libeapdtw_b200.so.
//
// Same names, argument meaning and error behaviour as the reference, so a
// caller of the reference switches by changing the namespace:
//   eapdtw::ea_pruned_dtw_windowed (dtw.hpp:93-99)  -> eapdtw_b200::ea_pruned_dtw_windowed
//   eapdtw::ea_pruned_dtw          (dtw.hpp:85-87)  -> eapdtw_b200::ea_pruned_dtw
//   eapdtw::dtw_windowed           (dtw.hpp:72-74)  -> eapdtw_b200::dtw_windowed
//   eapdtw::dtw_left_prune(_windowed) (dtw.hpp:76-83) -> same names (identical results:
//        exact value iff <= ub, else PRUNED; the GPU kernel prunes from both sides)
//   eapdtw::similarity_search      (search.hpp:118-119) -> eapdtw_b200::similarity_search
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
  if (trace.capture_cells && cumulative_bound.empty())
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
  KernelTrace t;
  return ea_pruned_dtw_windowed(a, b, band, ub, cumulative_bound, t);
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
  if (trace.capture_cells) return detail::traced(EAPDTW_ALGO_FULL, a, b, band.window, PRUNED, trace);
  double out = PRUNED;
  uint64_t cells = 0;
  detail::check(eapdtw_dtw_windowed(detail::context(), a.data(), a.size(), b.data(), b.size(),
                                    band.window, &out, &cells));
  trace.cells_evaluated += cells;
  return out;
}
[[nodiscard]] inline double dtw_windowed(std::span<const double> a, std::span<const double> b,
                                         Band band) {
  KernelTrace t;
  return dtw_windowed(a, b, band, t);
}
[[nodiscard]] inline double dtw_full(std::span<const double> a, std::span<const double> b) {
  return dtw_windowed(a, b, Band::unbounded());
}
[[nodiscard]] inline double dtw_full(std::span<const double> a, std::span<const double> b,
                                     KernelTrace& trace) {
  return dtw_windowed(a, b, Band::unbounded(), trace);
}
// Left pruning has EAPrunedDTW's result contract (exact iff <= ub, else
// PRUNED); without capture it runs the pruned kernel.
[[nodiscard]] inline double dtw_left_prune_windowed(std::span<const double> a,
                                                    std::span<const double> b, Band band,
                                                    double ub, KernelTrace& trace) {
  if (trace.capture_cells)
    return detail::traced(EAPDTW_ALGO_LEFT_PRUNE, a, b, band.window, ub, trace);
  return ea_pruned_dtw_windowed(a, b, band, ub, {}, trace);
}
[[nodiscard]] inline double dtw_left_prune_windowed(std::span<const double> a,
                                                    std::span<const double> b, Band band,
                                                    double ub) {
  return ea_pruned_dtw_windowed(a, b, band, ub);
}
[[nodiscard]] inline double dtw_left_prune(std::span<const double> a, std::span<const double> b,
                                           double ub) {
  return ea_pruned_dtw_windowed(a, b, Band::unbounded(), ub);
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

// --- search (search.hpp:50-119)
struct BestSoFar {
  std::size_t location = 0;
  double distance_sq = PRUNED;
  bool found = false;
};
enum class Algo : std::uint8_t { full, left_prune, ea_pruned };
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

}  // namespace eapdtw_b200
