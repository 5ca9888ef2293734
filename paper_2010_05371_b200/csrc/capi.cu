// capi.cu -- host orchestration behind the C ABI (include/eapdtw_b200.h).
//
// Everything here is host C++: argument validation mirroring the reference's
// std::invalid_argument conditions, the exact host-side query preparation of
// similarity_search (search.cpp:131-149), device buffer management, the phase
// sequencing of a search (stats -> envelope -> probe -> sweep) and result
// read-back.  The compute itself is in kernels.cu.  There is no CPU fallback.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <numeric>
#include <random>
#include <string>
#include <atomic>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/eapdtw_b200.h"
#include "kernels.cuh"

using namespace eapdtw_b200;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(EAPDTW_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));     \
  } while (0)

constexpr double kInf = std::numeric_limits<double>::infinity();

// Engine options of a context (eapdtw_ctx_set_option).  The defaults are the
// measured best; the others exist so tests can pin that
// every variant returns the reference's answer.  Nothing is read from the
// environment: a search depends on its arguments and these options only.
enum Opt : int {
  kOptAdK = 0,        // exact-engine window: -1 auto (search: strip; pairwise/NN1: choose_ad_k), 0/1/3/5
  kOptScreenRows,     // phase-A lane screen depth (rows)
  kOptF32,            // FP32 screening engine ahead of the exact one
  kOptStreamed,       // host-pointer search streamed in two parts: -1 auto, 0, 1
  kOptStreamSplit,    // part 1's share of a streamed search, in eighths
  kOptRankStride,     // rank pass: every S-th candidate (0: off)
  kOptRankK,          // ... the ~K best by layered LB_Kim
  kOptRankWaves,      // ... in this many waves of growing rank
  kOptRankUb,         // ... upper-bound wave first (narrow-band DTW)
  kOptRankUbW,        // ... its band divisor
  kOptRankUbK,        // ... its list divisor
  kOptRankCascade,    // ... cascade over the ranked list
  kOptCoarseStride,   // coarse pass over every S-th candidate (0: off)
  kOptProbe,          // probe candidates
  kOptProbeForce,     // run the probe even when the upper-bound wave applies
  kOptTighten,        // tighten_ub honoured (0: ignored; results unchanged either way)
  kOptCbStrip,        // first strip using the cumulative-bound thresholds
  kOptWarps,          // warps per search block (0: occupancy-sized)
  kOptNn1Splits,      // NN1 blocks per query (0: auto)
  kOptNn1Warm,        // NN1 per-warp warm start
  kOptSeriesCache,    // device-resident series keep their last stats
  kOptProbeStrips,    // FP32 strip screen: strips probed in each direction before committing (0: forward only)
  kOptProducers,      // search sweep: SMSP-0 warps are LB producers until this queue backlog (0: off)
  kOptProbeWarm,      // the FP32 probe also in the warm-start passes (probe, rank)
  kOptPrepOverlap,    // envelope beside the stats chain on a side stream (0: after it)
  kOptWarmF32,        // FP32 screen in the warm-start cascade (upper-bound wave and ranked list)
  kOptCbEcStrip,      // first strip whose cumulative-bound thresholds also use the EC suffix
  kOptProbeExcess,    // FP32 probe: the dropped direction's frontier minimum tightens the other's bound
  kOptSpecStats,      // speculative prefix-sum statistics beside the exact chain: -1 auto, 0 (the chain first), 1
  kOptSpecEps,        // ... their assumed deviation from the chain's, in units of 1e-9
  kOptRankMin,        // rank pass: only on ranges of at least this many candidates
  kOptLbBlocks,       // Keogh visiting order by parts (first 256 positions, then the rest)
  kNumOpts
};
struct OptDef {
  const char* name;
  long long def, lo, hi;
};
constexpr OptDef kOpts[kNumOpts] = {
    {"ad_k", -1, -1, 5},          {"screen_rows", 2, 0, 64},    {"f32", 1, 0, 1},
    {"streamed", -1, -1, 1},      {"stream_split", 3, 1, 7},    {"rank_stride", 16, 0, 1 << 20},
    {"rank_k", 16384, 1, 1 << 24}, {"rank_waves", 1, 1, 4},     {"rank_ub", 1, 0, 1},
    {"rank_ub_w", 4, 1, 1 << 16}, {"rank_ub_k", 16, 1, 1 << 16}, {"rank_cascade", 1, 0, 1},
    {"coarse_stride", 0, 0, 1 << 20}, {"probe", 2048, 1, 1 << 24}, {"probe_force", 0, 0, 1},
    {"tighten", 1, 0, 1},         {"cb_strip", 1, 1, 1 << 16},  {"warps", 0, 0, 8},
    {"nn1_splits", 0, 0, 1 << 16}, {"nn1_warm", 1, 0, 1},       {"series_cache", 1, 0, 1},
    {"probe_strips", 1, 0, 8},    {"producers", 0, 0, 1 << 20}, {"probe_warm", 0, 0, 1},
    {"prep_overlap", 1, 0, 1},   {"warm_f32", 1, 0, 1},      {"cb_ec_strip", 2, 1, 1 << 16},
    {"probe_excess", 1, 0, 1},     {"spec_stats", -1, -1, 1},      {"spec_eps", 8000, 1, 1000000},
    {"rank_min", 32000000, 0, 1LL << 40}, {"lb_blocks", 1, 0, 1},
};

// Grow-only device buffer.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t n) {
    if (n <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, n);
    if (e == cudaSuccess) bytes = n;
    return e;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};

// RunningStats (search.hpp:16-42) on the host, same operation order.
struct HostStats {
  double sum = 0.0, sumsq = 0.0;
  size_t count = 0;
  static HostStats over(const double* x, size_t n) {
    HostStats s;
    for (size_t i = 0; i < n; ++i) {
      s.sum += x[i];
      s.sumsq += x[i] * x[i];
    }
    s.count = n;
    return s;
  }
  double mean() const { return sum / static_cast<double>(count); }
  double stddev() const {
    const double m = mean();
    const double v = sumsq / static_cast<double>(count) - m * m;
    return std::sqrt(v > 0.0 ? v : 0.0);
  }
};

// znormalize_into (search.cpp:37-46)
void host_znormalize(const double* src, size_t n, const HostStats& st, double* dst) {
  const double m = st.mean();
  const double s = st.stddev();
  if (s < kMinStddev) {
    std::fill(dst, dst + n, 0.0);
    return;
  }
  for (size_t i = 0; i < n; ++i) dst[i] = (src[i] - m) / s;
}

bool all_finite(const double* x, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(x[i])) return false;
  return true;
}

}  // namespace

struct PlanBuffers {
  DevBuf mean, sd, env, q, qul, qperm, order, best, key, work, counters, probe_counters, flag,
      queue, qtot, qctr, rank, rlist, scratch;
  // speculation: prefix-sum statistics, the completed candidates' list, and
  // {deviation bits, rule mismatches, list count}
  DevBuf mean_a, sd_a, vlist, spec;
  DevBuf qperm32;  // the visiting-order query envelope as outward-rounded floats
  void release() {
    for (DevBuf* b : {&mean, &sd, &env, &q, &qul, &qperm, &order, &best, &key, &work, &counters,
                      &probe_counters, &flag, &queue, &qtot, &qctr, &rank, &rlist, &scratch,
                      &mean_a, &sd_a, &vlist, &spec, &qperm32})
      b->release();
  }
};

// Kernel launches of one context, also added to a process-wide total (the
// concurrent grid's worker contexts are short-lived).
static std::atomic<uint64_t> g_total_launches{0};
static std::atomic<uint64_t> g_spec_fallbacks{0};  // speculative searches redone on the exact statistics
struct LaunchCounter {
  uint64_t n = 0;
  LaunchCounter& operator++() {
    ++n;
    g_total_launches.fetch_add(1, std::memory_order_relaxed);
    return *this;
  }
  LaunchCounter& operator+=(uint64_t k) {
    n += k;
    g_total_launches.fetch_add(k, std::memory_order_relaxed);
    return *this;
  }
  operator uint64_t() const { return n; }
};

struct eapdtw_ctx {
  int device = 0;
  long long opt[kNumOpts];
  eapdtw_ctx() {
    for (int k = 0; k < kNumOpts; ++k) opt[k] = kOpts[k].def;
  }
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  LaunchCounter launches;
  uint64_t last_cells_f32 = 0;  // FP32-screen share of the last nn1 call's cells
  // scratch for pairwise / nn1 host-pointer variants
  DevBuf a, b, ub, cb, out, cells, best, keys, counters, gscratch;
  DevBuf ref;  // host-pointer search copies the reference here
  PlanBuffers pb;  // scratch of the one-shot search API (grow-only, reused)
  cudaStream_t copy = nullptr;  // H2D stream of the streamed host-pointer search
  cudaEvent_t copied[2] = {nullptr, nullptr};
  cudaEvent_t fork = nullptr;  // orders the streamed copy after earlier work
  // side stream of the preparation: the envelope runs there beside the stats chain
  cudaStream_t aux = nullptr;
  cudaEvent_t aux_fork = nullptr, aux_join = nullptr;
  // speculation: the exact chain (then its verification) runs on this stream
  cudaStream_t aux2 = nullptr;
  cudaEvent_t spec_fork = nullptr, spec_fast = nullptr, spec_done = nullptr;
  int spec_cooldown = 0;      // searches left without speculation after a fallback (auto mode)
  double spec_dev = -1.0;     // last search: measured deviation (< 0: no speculation)
  uint64_t spec_listed = 0;   // ... candidates re-evaluated with the exact statistics
};

struct eapdtw_search_plan {
  eapdtw_ctx* ctx = nullptr;
  PlanBuffers own;
  PlanBuffers* buf = &own;            // the one-shot API borrows the context's buffers
  unsigned long long* key = nullptr;  // active threshold key (own or external)
  const double* ref = nullptr;        // device
  size_t n = 0, m = 0, w_cells = 0;
  int w_eff = 0;
  int env_r = 0;
  bool use_lb = true, have_env = false, tighten = true;
  int cb_strip = 1;
  int algo = EAPDTW_ALGO_EA_PRUNED;
  uint64_t offset = 0;
  size_t ncand = 0;
  cudaEvent_t ev[8] = {};
  bool prepared = false, ran = false;
  bool stats_ready = false;  // mean/sd already in the buffers (a series' cached stats)
  int blocks = 0, warps = 8, ad_k = 0, screen_rows = 2;  // screen depth: 2 measured best with the FP32 engine
  int use_f32 = 1;  // FP32 screening engine ahead of the exact one (EAPDTW_F32=0: off)
  int coarse_stride = 0;  // coarse pass (the rank pass replaced it; 0: off)
  // rank pass (warm start): the cascade over the ~rank_k candidates with the
  // smallest layered LB_Kim among every rank_stride-th (0: off)
  long long rank_stride = 16, rank_k = 16384;
  int rank_waves = 1;  // waves k/16^(n-1) .. k/16, k
  bool rank_ub = true;  // upper-bound wave first (narrow-band DTW of the k/16 best)
  int rank_ub_w = 4, rank_ub_k = 16;  // its band and list divisors
  bool rank_cascade = true;
  int probe = 2048;
  bool probe_force = false;
  size_t queue_slack = 0;  // spare survivor-queue slots (>= resident warps)
  bool gmem = false;       // per-warp buffers in global memory (queries too long for shared memory)
  double guard_rel = 1e-9, guard_abs = 1e-20;
  double qmax = 0.0;  // max |normalised query|
  std::chrono::steady_clock::time_point t0;
  // Speculative statistics (kernels.cu: fast_stats_kernel).  spec: allowed for
  // this plan; spec_active: this preparation runs on them (the exact chain is
  // in flight on the context's second side stream); spec_final: the exact
  // pass over the completed candidates is enqueued; runs: the candidate ranges
  // searched so far (replayed without speculation if the verification fails).
  bool lb_block_order = false;  // order[] by parts (plan_init)
  bool spec = false, spec_active = false, spec_final = false;
  double spec_eps = 0.0;
  long long vcap = 0;
  std::vector<std::pair<size_t, size_t>> runs;
};

extern "C" {

const char* eapdtw_last_error(void) { return g_err.c_str(); }
int eapdtw_version(void) { return 1; }

int eapdtw_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int eapdtw_ctx_create(eapdtw_ctx** out, int device) {
  if (!out) return fail(EAPDTW_EINVAL, "ctx_create: null out");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(EAPDTW_ECUDA, "no CUDA device: the B200 path has no CPU fallback");
  if (device < 0 || device >= n) return fail(EAPDTW_EINVAL, "ctx_create: bad device");
  CUDA_TRY(cudaSetDevice(device));
  auto* c = new eapdtw_ctx();
  c->device = device;

  e = cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    return fail(EAPDTW_ECUDA, cudaGetErrorString(e));
  }
  c->stream = c->own;
  *out = c;
  return EAPDTW_OK;
}

int eapdtw_ctx_destroy(eapdtw_ctx* c) {
  if (!c) return EAPDTW_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (DevBuf* b : {&c->a, &c->b, &c->ub, &c->cb, &c->out, &c->cells, &c->best, &c->keys,
                    &c->counters, &c->ref, &c->gscratch})
    b->release();
  c->pb.release();
  if (c->copy) {
    cudaStreamSynchronize(c->copy);
    cudaStreamDestroy(c->copy);
  }
  for (cudaEvent_t& ev : c->copied)
    if (ev) cudaEventDestroy(ev);
  if (c->fork) cudaEventDestroy(c->fork);
  if (c->aux) {
    cudaStreamSynchronize(c->aux);
    cudaStreamDestroy(c->aux);
  }
  if (c->aux_fork) cudaEventDestroy(c->aux_fork);
  if (c->aux_join) cudaEventDestroy(c->aux_join);
  if (c->aux2) {
    cudaStreamSynchronize(c->aux2);
    cudaStreamDestroy(c->aux2);
  }
  for (cudaEvent_t ev : {c->spec_fork, c->spec_fast, c->spec_done})
    if (ev) cudaEventDestroy(ev);
  if (c->own) cudaStreamDestroy(c->own);
  delete c;
  return EAPDTW_OK;
}

int eapdtw_ctx_set_stream(eapdtw_ctx* c, void* s) {
  if (!c) return fail(EAPDTW_EINVAL, "null ctx");
  c->stream = s ? static_cast<cudaStream_t>(s) : c->own;
  return EAPDTW_OK;
}

int eapdtw_ctx_set_option(eapdtw_ctx* c, const char* name, int64_t value) {
  if (!c || !name) return fail(EAPDTW_EINVAL, "null argument");
  for (int k = 0; k < kNumOpts; ++k) {
    if (std::strcmp(name, kOpts[k].name) != 0) continue;
    if (value < kOpts[k].lo || value > kOpts[k].hi)
      return fail(EAPDTW_EINVAL, std::string("option out of range: ") + name);
    if (k == kOptAdK && !(value == -1 || value == 0 || value == 1 || value == 3 || value == 5))
      return fail(EAPDTW_EINVAL, "option ad_k: -1, 0, 1, 3 or 5");
    c->opt[k] = value;
    if (k == kOptSpecStats) c->spec_cooldown = 0;
    return EAPDTW_OK;
  }
  return fail(EAPDTW_EINVAL, std::string("unknown option: ") + name);
}

int eapdtw_ctx_get_option(const eapdtw_ctx* c, const char* name, int64_t* value) {
  if (!c || !name || !value) return fail(EAPDTW_EINVAL, "null argument");
  for (int k = 0; k < kNumOpts; ++k)
    if (std::strcmp(name, kOpts[k].name) == 0) {
      *value = c->opt[k];
      return EAPDTW_OK;
    }
  return fail(EAPDTW_EINVAL, std::string("unknown option: ") + name);
}

int eapdtw_ctx_synchronize(eapdtw_ctx* c) {
  if (!c) return fail(EAPDTW_EINVAL, "null ctx");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (c->aux) CUDA_TRY(cudaStreamSynchronize(c->aux));
  if (c->aux2) CUDA_TRY(cudaStreamSynchronize(c->aux2));
  return EAPDTW_OK;
}

uint64_t eapdtw_ctx_launches(const eapdtw_ctx* c) { return c ? static_cast<uint64_t>(c->launches) : 0; }

uint64_t eapdtw_total_launches(void) { return g_total_launches.load(); }

// ---------------------------------------------------------------------------
// Pairwise
// ---------------------------------------------------------------------------
static int pairwise_impl(eapdtw_ctx* c, const double* rows_dev, const double* cols_dev,
                         size_t npairs, size_t lr, size_t lc, size_t window, const double* ub_dev,
                         const double* cb_dev, int prune, double* out_dev, uint64_t* cells) {
  // effective_window (dtw.cpp:57-62): caller guarantees lr >= lc.
  int w;
  if (window == EAPDTW_UNBOUNDED_WINDOW || window >= lc) w = static_cast<int>(lr);
  else w = static_cast<int>(window);
  CUDA_TRY(c->cells.ensure(sizeof(unsigned long long)));
  CUDA_TRY(cudaMemsetAsync(c->cells.p, 0, sizeof(unsigned long long), c->stream));
  PairParams p{};
  p.rows = rows_dev;
  p.cols = cols_dev;
  p.row_stride = static_cast<long long>(lr);
  p.col_stride = static_cast<long long>(lc);
  p.lr = static_cast<int>(lr);
  p.lc = static_cast<int>(lc);
  p.w = w;
  p.ub = ub_dev;
  p.cb = cb_dev;
  p.prune = prune;
  p.ad_k = c->opt[kOptAdK] >= 0 ? static_cast<int>(c->opt[kOptAdK]) : choose_ad_k(static_cast<int>(lr), w);
  p.out = out_dev;
  p.cells = c->cells.as<unsigned long long>();
  p.npairs = static_cast<long long>(npairs);
  if (const size_t g = pairwise_gscratch_doubles(p)) {  // series too long for shared memory
    CUDA_TRY(c->gscratch.ensure(g * 8));
    p.gscratch = c->gscratch.as<double>();
  }
  CUDA_TRY(launch_pairwise(p, c->stream));
  ++c->launches;
  if (cells) {
    unsigned long long h = 0;
    CUDA_TRY(cudaMemcpyAsync(&h, c->cells.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    *cells = h;
  }
  return EAPDTW_OK;
}

static int check_cb_host(const double* cb, size_t cb_len, size_t lr) {
  // check_cumulative_bound (dtw.cpp:64-75)
  if (cb_len == 0) return EAPDTW_OK;
  if (cb_len != lr)
    return fail(EAPDTW_EINVAL, "cumulative bound: length must match the longer series");
  for (size_t k = 0; k + 1 < cb_len; ++k)
    if (!(cb[k] >= cb[k + 1])) return fail(EAPDTW_EINVAL, "cumulative bound: must be non-increasing");
  if (cb[cb_len - 1] != 0.0) return fail(EAPDTW_EINVAL, "cumulative bound: final element must be 0");
  return EAPDTW_OK;
}

static int single_pair(eapdtw_ctx* c, const double* a, size_t la, const double* b, size_t lb,
                       size_t window, double ub, const double* cb, size_t cb_len, int prune,
                       double* out, uint64_t* cells) {
  if (!c) return fail(EAPDTW_EINVAL, "null ctx");
  if (la == 0 || lb == 0 || !a || !b || !out) return fail(EAPDTW_EINVAL, "dtw: empty series");
  // orient (dtw.cpp:48-52): longer series on rows, first argument wins ties
  const double* rows = a;
  const double* cols = b;
  size_t lr = la, lc = lb;
  if (la < lb) {
    rows = b;
    cols = a;
    lr = lb;
    lc = la;
  }
  if (prune == 1) {
    const int e = check_cb_host(cb, cb_len, lr);
    if (e) return e;
  }
  if (window != EAPDTW_UNBOUNDED_WINDOW && lr - lc > window) {  // no path fits the band
    *out = kInf;
    if (cells) *cells = 0;
    return EAPDTW_OK;
  }
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(c->a.ensure(lr * 8));
  CUDA_TRY(c->b.ensure(lc * 8));
  CUDA_TRY(c->ub.ensure(8));
  CUDA_TRY(c->out.ensure(8));
  CUDA_TRY(cudaMemcpyAsync(c->a.p, rows, lr * 8, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->b.p, cols, lc * 8, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->ub.p, &ub, 8, cudaMemcpyHostToDevice, c->stream));
  const double* cb_dev = nullptr;
  if (prune == 1 && cb_len) {
    CUDA_TRY(c->cb.ensure(cb_len * 8));
    CUDA_TRY(cudaMemcpyAsync(c->cb.p, cb, cb_len * 8, cudaMemcpyHostToDevice, c->stream));
    cb_dev = c->cb.as<double>();
  }
  uint64_t ncell = 0;
  const int e = pairwise_impl(c, c->a.as<double>(), c->b.as<double>(), 1, lr, lc, window,
                              c->ub.as<double>(), cb_dev, prune, c->out.as<double>(), &ncell);
  if (e) return e;
  CUDA_TRY(cudaMemcpyAsync(out, c->out.p, 8, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (cells) *cells = ncell;
  return EAPDTW_OK;
}

int eapdtw_ea_pruned_dtw_windowed(eapdtw_ctx* c, const double* a, size_t la, const double* b,
                                  size_t lb, size_t window, double ub, const double* cb,
                                  size_t cb_len, double* out, uint64_t* cells) {
  return single_pair(c, a, la, b, lb, window, ub, cb, cb_len, 1, out, cells);
}

int eapdtw_dtw_windowed(eapdtw_ctx* c, const double* a, size_t la, const double* b, size_t lb,
                        size_t window, double* out, uint64_t* cells) {
  return single_pair(c, a, la, b, lb, window, kInf, nullptr, 0, 0, out, cells);
}

int eapdtw_dtw_left_prune_windowed(eapdtw_ctx* c, const double* a, size_t la, const double* b,
                                   size_t lb, size_t window, double ub, double* out,
                                   uint64_t* cells) {
  return single_pair(c, a, la, b, lb, window, ub, nullptr, 0, 2, out, cells);
}

int eapdtw_trace(eapdtw_ctx* c, int algo, const double* a, size_t la, const double* b, size_t lb,
                 size_t window, double ub, eapdtw_trace_event* events, size_t cap,
                 size_t* n_events, uint64_t* cells, double* out) {
  if (!c || !n_events || !out) return fail(EAPDTW_EINVAL, "null argument");
  if (algo < 0 || algo > 2) return fail(EAPDTW_EINVAL, "trace: algo must be 0 (full), 1 (lp), 2 (eap)");
  if (la == 0 || lb == 0 || !a || !b) return fail(EAPDTW_EINVAL, "dtw: empty series");
  if (cap && !events) return fail(EAPDTW_EINVAL, "null argument");
  const double* rows = a;  // orient (dtw.cpp:48-52)
  const double* cols = b;
  size_t lr = la, lc = lb;
  if (la < lb) {
    rows = b;
    cols = a;
    lr = lb;
    lc = la;
  }
  *n_events = 0;
  if (cells) *cells = 0;
  // effective_window (dtw.cpp:57-62): no path fits -> PRUNED, nothing traced
  size_t w = lr;
  if (window != EAPDTW_UNBOUNDED_WINDOW) {
    if (lr - lc > window) {
      *out = kInf;
      return EAPDTW_OK;
    }
    if (window < lc) w = window;
  }
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(c->a.ensure(lr * 8));
  CUDA_TRY(c->b.ensure(lc * 8));
  CUDA_TRY(c->cb.ensure(2 * (lc + 1) * 8));
  CUDA_TRY(c->counters.ensure(3 * 8));
  CUDA_TRY(c->out.ensure((cap ? cap : 1) * sizeof(TraceEvent)));
  CUDA_TRY(c->ub.ensure(8));
  CUDA_TRY(cudaMemcpyAsync(c->a.p, rows, lr * 8, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->b.p, cols, lc * 8, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(launch_trace(algo, c->a.as<double>(), static_cast<long long>(lr), c->b.as<double>(),
                        static_cast<long long>(lc), static_cast<long long>(w), ub,
                        c->cb.as<double>(), c->out.as<TraceEvent>(), static_cast<long long>(cap),
                        c->counters.as<unsigned long long>(), c->ub.as<double>(), c->stream));
  ++c->launches;
  unsigned long long hdr[2] = {0, 0};
  CUDA_TRY(cudaMemcpyAsync(hdr, c->counters.p, 16, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaMemcpyAsync(out, c->ub.p, 8, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  const size_t stored = std::min<size_t>(cap, hdr[0]);
  if (stored)
    CUDA_TRY(cudaMemcpy(events, c->out.p, stored * sizeof(TraceEvent), cudaMemcpyDeviceToHost));
  *n_events = hdr[0];
  if (cells) *cells = hdr[1];
  return EAPDTW_OK;
}

int eapdtw_pairwise_dev(eapdtw_ctx* c, const double* a_dev, const double* b_dev, size_t npairs,
                        size_t len, size_t window, const double* ub_dev, int prune,
                        double* out_dev, uint64_t* cells) {
  if (!c) return fail(EAPDTW_EINVAL, "null ctx");
  if (len == 0) return fail(EAPDTW_EINVAL, "dtw: empty series");
  if (npairs == 0) return EAPDTW_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  return pairwise_impl(c, a_dev, b_dev, npairs, len, len, window, ub_dev, nullptr, prune, out_dev,
                       cells);
}

int eapdtw_pairwise(eapdtw_ctx* c, const double* a, const double* b, size_t npairs, size_t len,
                    size_t window, const double* ub, int prune, double* out, uint64_t* cells) {
  if (!c) return fail(EAPDTW_EINVAL, "null ctx");
  if (len == 0) return fail(EAPDTW_EINVAL, "dtw: empty series");
  if (npairs == 0) return EAPDTW_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  const size_t bytes = npairs * len * 8;
  CUDA_TRY(c->a.ensure(bytes));
  CUDA_TRY(c->b.ensure(bytes));
  CUDA_TRY(c->out.ensure(npairs * 8));
  CUDA_TRY(cudaMemcpyAsync(c->a.p, a, bytes, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->b.p, b, bytes, cudaMemcpyHostToDevice, c->stream));
  const double* ub_dev = nullptr;
  if (ub) {
    CUDA_TRY(c->ub.ensure(npairs * 8));
    CUDA_TRY(cudaMemcpyAsync(c->ub.p, ub, npairs * 8, cudaMemcpyHostToDevice, c->stream));
    ub_dev = c->ub.as<double>();
  }
  const int e = pairwise_impl(c, c->a.as<double>(), c->b.as<double>(), npairs, len, len, window,
                              ub_dev, nullptr, prune, c->out.as<double>(), cells);
  if (e) return e;
  CUDA_TRY(cudaMemcpyAsync(out, c->out.p, npairs * 8, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return EAPDTW_OK;
}

// ---------------------------------------------------------------------------
// Search plan
//
// A plan binds one (reference shard, query, config).  create() does the
// host-side query preparation of similarity_search (search.cpp:131-149) and
// allocates device buffers; every search then runs
//   reset()   -> best record / threshold / counters to their initial state
//   prepare() -> stats chain, raw envelope, probe candidates
//   run()     -> the persistent sweep over candidate ranges
//   result()  -> read back (location, distance, counters)
// ---------------------------------------------------------------------------
static int plan_init(eapdtw_search_plan* p, eapdtw_ctx* c, const double* ref_dev, size_t n,
                     const double* query, size_t qlen, const eapdtw_search_config* cfg,
                     uint64_t offset) {
  if (n == 0 || qlen == 0 || !query) return fail(EAPDTW_EINVAL, "Series: empty input");
  // similarity_search validation (search.cpp:121-127)
  const size_t m = cfg->query_length == 0 ? qlen : cfg->query_length;
  if (m == 0 || m > qlen) return fail(EAPDTW_EINVAL, "similarity_search: bad query length");
  if (m > n) return fail(EAPDTW_EINVAL, "similarity_search: query longer than reference");
  if (!all_finite(query, qlen)) return fail(EAPDTW_EINVAL, "Series: non-finite sample");
  if (offset % static_cast<uint64_t>(kStatsResetInterval) != 0)
    return fail(EAPDTW_EINVAL, "search plan: shard offset must be a multiple of 100000");
  if (m > (1u << 16)) return fail(EAPDTW_EINVAL, "search: query length above the GPU limit (65536)");
  if (cfg->algorithm < EAPDTW_ALGO_FULL || cfg->algorithm > EAPDTW_ALGO_EA_PRUNED)
    return fail(EAPDTW_EINVAL, "search: bad algorithm");
  CUDA_TRY(cudaSetDevice(c->device));

  p->t0 = std::chrono::steady_clock::now();
  p->ctx = c;
  p->ref = ref_dev;
  p->n = n;
  p->m = m;
  p->offset = offset;
  p->use_lb = cfg->use_lower_bounds != 0;
  // tighten_ub is consulted only with the cascade and EAPrunedDTW (search.cpp:101-105, 191)
  p->tighten = p->use_lb && cfg->tighten_ub != 0 && cfg->algorithm == EAPDTW_ALGO_EA_PRUNED;
  const long long* o = c->opt;
  p->tighten = p->tighten && o[kOptTighten] != 0;
  p->cb_strip = static_cast<int>(o[kOptCbStrip]);
  p->algo = cfg->algorithm;
  p->ncand = n - m + 1;
  // window_cells_for (search.cpp:18-21)
  const double wf = std::floor(cfg->window_ratio * static_cast<double>(m));
  p->w_cells = wf <= 0.0 ? 0 : static_cast<size_t>(wf);
  // effective_window for two length-m series (dtw.cpp:57-62)
  p->w_eff = p->w_cells >= m ? static_cast<int>(m) : static_cast<int>(p->w_cells);
  p->env_r = static_cast<int>(std::min(p->w_cells, m));  // compute_envelope clamp (lower_bounds.cpp:12)
  p->guard_rel = std::max(1e-9, 8.0 * static_cast<double>(m) * 0x1.0p-53);
  // Search DTW calls are mostly short (killed within a few strips), where the
  // strip engine's lower per-call setup wins; the anti-diagonal engine is
  // opt-in here (EAPDTW_AD_K) and the default for pairwise / NN1 batches.
  p->ad_k = o[kOptAdK] > 0 ? static_cast<int>(o[kOptAdK]) : 0;
  p->screen_rows = static_cast<int>(o[kOptScreenRows]);

  p->use_f32 = static_cast<int>(o[kOptF32]);
  p->coarse_stride = static_cast<int>(o[kOptCoarseStride]);
  p->probe = static_cast<int>(o[kOptProbe]);
  p->probe_force = o[kOptProbeForce] != 0;
  p->rank_ub = o[kOptRankUb] != 0;
  p->rank_stride = o[kOptRankStride];
  p->rank_k = o[kOptRankK];
  p->rank_waves = static_cast<int>(o[kOptRankWaves]);
  p->rank_ub_w = static_cast<int>(o[kOptRankUbW]);
  p->rank_ub_k = static_cast<int>(o[kOptRankUbK]);
  p->rank_cascade = o[kOptRankCascade] != 0;
  p->guard_abs = 1e-20;

  // Query preparation exactly as search.cpp:136-149.
  std::vector<double> qn(m), qu(m), ql(m), q1(m + 1, 0.0);
  host_znormalize(query, m, HostStats::over(query, m), qn.data());
  const size_t r = p->env_r;
  for (size_t j = 0; j < m; ++j) {  // compute_envelope (lower_bounds.cpp:9-49): exact max/min
    const size_t lo = j > r ? j - r : 0;
    const size_t hi = std::min(m - 1, j + r);
    double mx = qn[lo], mn = qn[lo];
    for (size_t k = lo + 1; k <= hi; ++k) {
      mx = std::max(mx, qn[k]);
      mn = std::min(mn, qn[k]);
    }
    qu[j] = mx;
    ql[j] = mn;
  }
  std::vector<int> order(m);
  std::iota(order.begin(), order.end(), 0);
  // Descending |q| (search.cpp:143-149); with option lb_blocks inside each of
  // two parts, the first kLbHead positions and the rest: any visiting order
  // gives the same sums, and a tier's leg then reads one part of the
  // reference stretch only (kernels.cu: EQ staging).
  const auto by_absq = [&](int a, int b) {
    const double fa = std::fabs(qn[a]), fb = std::fabs(qn[b]);
    return fa != fb ? fa > fb : a < b;
  };
  p->lb_block_order = o[kOptLbBlocks] != 0 && m > static_cast<size_t>(kLbHead);
  if (p->lb_block_order) {
    std::sort(order.begin(), order.begin() + kLbHead, by_absq);
    std::sort(order.begin() + kLbHead, order.end(), by_absq);
  } else {
    std::sort(order.begin(), order.end(), by_absq);
  }
  std::copy(qn.begin(), qn.end(), q1.begin() + 1);
  // (upper, lower) per position, and the same in visiting order.  (Outward-
  // rounded floats for the visiting-order copy, half its L1 footprint,
  // measured slower: cfg4 sweep +1.4 ms, the conversions and looser terms
  // cost more than the cache hits gained.)
  std::vector<double> qul(2 * m), qperm(2 * m);
  for (size_t j = 0; j < m; ++j) {
    qul[2 * j] = qu[j];
    qul[2 * j + 1] = ql[j];
    qperm[2 * j] = qu[order[j]];
    qperm[2 * j + 1] = ql[order[j]];
  }
  p->qmax = 0.0;
  for (const double v : qn) p->qmax = std::max(p->qmax, std::fabs(v));

  PlanBuffers& B = *p->buf;
  const size_t nc = p->ncand;
  CUDA_TRY(B.mean.ensure(nc * 8));
  CUDA_TRY(B.sd.ensure(nc * 8));
  CUDA_TRY(B.q.ensure((m + 1) * 8));
  CUDA_TRY(B.qul.ensure(m * 16));
  CUDA_TRY(B.qperm.ensure(m * 16));
  CUDA_TRY(B.qperm32.ensure(m * 8));
  CUDA_TRY(B.order.ensure(m * 4));
  CUDA_TRY(B.best.ensure(sizeof(BestRecord)));
  CUDA_TRY(B.key.ensure(8));
  CUDA_TRY(B.work.ensure(8));
  CUDA_TRY(B.qctr.ensure(24));
  CUDA_TRY(B.flag.ensure(8));
  CUDA_TRY(B.counters.ensure(kNumCountersExt * 8));
  CUDA_TRY(B.probe_counters.ensure(kNumCountersExt * 8));
  if (p->use_lb) {
    CUDA_TRY(B.env.ensure(n * 16));
  }
  p->key = B.key.as<unsigned long long>();
  for (auto& ev : p->ev) CUDA_TRY(cudaEventCreate(&ev));
  cudaStream_t s = c->stream;
  CUDA_TRY(cudaMemcpyAsync(B.q.p, q1.data(), (m + 1) * 8, cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(B.qul.p, qul.data(), m * 16, cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(B.qperm.p, qperm.data(), m * 16, cudaMemcpyHostToDevice, s));
  std::vector<float> qperm32(2 * m);
  for (size_t j = 0; j < m; ++j) {  // outward: the float envelope contains the double one
    float u = static_cast<float>(qperm[2 * j]), l = static_cast<float>(qperm[2 * j + 1]);
    if (static_cast<double>(u) < qperm[2 * j]) u = std::nextafter(u, std::numeric_limits<float>::infinity());
    if (static_cast<double>(l) > qperm[2 * j + 1]) l = std::nextafter(l, -std::numeric_limits<float>::infinity());
    qperm32[2 * j] = u;
    qperm32[2 * j + 1] = l;
  }
  CUDA_TRY(cudaMemcpyAsync(B.qperm32.p, qperm32.data(), m * 8, cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(B.order.p, order.data(), m * 4, cudaMemcpyHostToDevice, s));
  // the staging vectors are pageable locals: wait until the copies consumed them
  CUDA_TRY(cudaStreamSynchronize(s));

  // Occupancy-sized persistent grid: the largest number of resident warps
  // (blocks of `warps` warps, limited by shared memory and by the kernel's
  // register budget of 2 x 256-thread blocks per SM).
  int sms = 148, max_smem = 0, optin = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, c->device);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device);
  int best_warps = 0, best_w = 0, best_blocks = 0;
  for (int wpb = 8; wpb >= 1; --wpb) {
    const size_t smem = search_smem_bytes(static_cast<int>(m), wpb, p->ad_k);
    if (smem > static_cast<size_t>(optin)) continue;
    const int by_smem = static_cast<int>(max_smem / (smem + 1024));
    const int by_regs = (search_blocks_per_sm_by_regs() * 8) / wpb;  // register budget
    const int per_sm = std::min(by_smem, std::max(1, by_regs));
    if (per_sm * wpb > best_warps) {
      best_warps = per_sm * wpb;
      best_w = wpb;
      best_blocks = per_sm;
    }
  }
  p->gmem = best_warps == 0;
  if (p->gmem) {
    // Long queries: the per-warp buffers in global memory (the query and the
    // tier stacks stay in shared memory), one or two 8-warp blocks per SM.
    const size_t smem = search_smem_bytes(static_cast<int>(m), 8, p->ad_k, true);
    if (smem > static_cast<size_t>(optin))
      return fail(EAPDTW_EINVAL, "search: query length exceeds the GPU limit (shared memory)");
    best_w = 8;
    best_blocks = std::max(1, std::min(search_blocks_per_sm_by_regs(),
                                       static_cast<int>(max_smem / (smem + 1024))));
  }
  p->warps = best_w;
  p->blocks = sms * best_blocks;
  if (p->gmem)
    CUDA_TRY(B.scratch.ensure(static_cast<size_t>(p->blocks) * p->warps *
                              search_warp_buf_doubles(static_cast<int>(m), p->ad_k) * 8));
  if (o[kOptWarps] >= 1 && o[kOptWarps] < p->warps) p->warps = static_cast<int>(o[kOptWarps]);
  // One spare slot per resident warp: a consumer may hold a "future" slot past
  // the final tail, which must read as empty (-1) rather than stale data.
  p->queue_slack = static_cast<size_t>(p->blocks) * p->warps + 64;
  CUDA_TRY(B.queue.ensure((nc + p->queue_slack) * 8));
  CUDA_TRY(B.qtot.ensure((nc + p->queue_slack) * 8));
  // speculative statistics: pruned searches only (without a threshold every
  // candidate completes and would be evaluated twice)
  p->spec = p->algo == EAPDTW_ALGO_EA_PRUNED;
  return eapdtw_search_plan_reset(p);
}

int eapdtw_search_plan_create(eapdtw_ctx* c, const double* ref_dev, size_t n, const double* query,
                              size_t qlen, const eapdtw_search_config* cfg, uint64_t offset,
                              eapdtw_search_plan** out) {
  if (!c || !cfg || !out) return fail(EAPDTW_EINVAL, "search: null argument");
  auto* p = new eapdtw_search_plan();
  const int e = plan_init(p, c, ref_dev, n, query, qlen, cfg, offset);
  if (e) {
    const std::string msg = g_err;
    eapdtw_search_plan_destroy(p);
    g_err = msg;
    return e;
  }
  *out = p;
  return EAPDTW_OK;
}

int eapdtw_search_plan_reset(eapdtw_search_plan* p) {
  if (!p) return fail(EAPDTW_EINVAL, "null plan");
  eapdtw_ctx* c = p->ctx;
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  PlanBuffers& B = *p->buf;
  CUDA_TRY(cudaMemsetAsync(B.counters.p, 0, kNumCountersExt * 8, s));
  CUDA_TRY(cudaMemsetAsync(B.probe_counters.p, 0, kNumCountersExt * 8, s));
  CUDA_TRY(launch_init_best(B.best.as<BestRecord>(), p->key, 1, s));
  ++c->launches;
  p->prepared = false;
  p->ran = false;
  p->t0 = std::chrono::steady_clock::now();
  return EAPDTW_OK;
}

int eapdtw_search_plan_set_ub_key(eapdtw_search_plan* p, uint64_t* dev_key) {
  if (!p) return fail(EAPDTW_EINVAL, "null plan");
  p->key = dev_key ? reinterpret_cast<unsigned long long*>(dev_key)
                   : p->buf->key.as<unsigned long long>();
  return eapdtw_search_plan_reset(p);
}

size_t eapdtw_search_plan_candidates(const eapdtw_search_plan* p) { return p ? p->ncand : 0; }
uint64_t* eapdtw_search_plan_ub_key(eapdtw_search_plan* p) {
  return p ? reinterpret_cast<uint64_t*>(p->key) : nullptr;
}

// Zero the chunk counter and queue counters, fill the queue with -1 (empty).
static cudaError_t reset_work(eapdtw_search_plan* p, long long count, cudaStream_t s) {
  PlanBuffers& B = *p->buf;
  cudaError_t e = cudaMemsetAsync(B.work.p, 0, 8, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(B.qctr.p, 0, 24, s);
  if (e == cudaSuccess && count > 0)
    e = cudaMemsetAsync(B.queue.p, 0xff, static_cast<size_t>(count) * 8 + p->queue_slack * 8, s);
  return e;
}

static SearchParams base_params(eapdtw_search_plan* p) {
  PlanBuffers& B = *p->buf;
  SearchParams s{};
  s.ref = p->ref;
  s.mean = B.mean.as<double>();
  s.sd = B.sd.as<double>();
  s.env = p->have_env ? B.env.as<double2>() : nullptr;
  s.q = B.q.as<double>();
  s.qul = B.qul.as<double2>();
  s.qperm = B.qperm.as<double2>();
  s.qperm32 = B.qperm32.as<float2>();
  // a term's FP32 distance error: the value (|.| <= cmax or qmax) and the
  // difference (<= cmax + qmax) round once each, with margin
  s.lb_f32_e = 4.0 * 0x1.0p-24 * (std::sqrt(static_cast<double>(p->m)) + 1.0 + p->qmax);
  s.order = B.order.as<int>();
  s.lb_block_order = p->lb_block_order ? 1 : 0;
  s.ncand = static_cast<long long>(p->ncand);
  s.m = static_cast<int>(p->m);
  s.w = p->w_eff;
  s.use_lb = p->use_lb ? 1 : 0;
  s.tighten = p->tighten ? 1 : 0;
  s.cb_strip = p->cb_strip;
  s.cb_ec_strip = static_cast<int>(p->ctx->opt[kOptCbEcStrip]);
  s.probe_excess = static_cast<int>(p->ctx->opt[kOptProbeExcess]);
  // 0 full_scan, 1 EAPrunedDTW, 2 left_prune_scan (dtw.cpp:95-296)
  s.prune = p->algo == EAPDTW_ALGO_FULL ? 0 : (p->algo == EAPDTW_ALGO_LEFT_PRUNE ? 2 : 1);
  s.guard_rel = p->guard_rel;
  s.guard_abs = p->guard_abs;
  // 2 * 3u * sqrt(m) * cmax, cmax = sqrt(m) + 1 + qmax (z-normalised windows
  // and envelope values, the query), with margin
  s.guard_sqrt = 8.0 * 0x1.0p-53 * std::sqrt(static_cast<double>(p->m)) *
                 (std::sqrt(static_cast<double>(p->m)) + 1.0 + p->qmax);
  s.ub_key = p->key;
  s.best = B.best.as<BestRecord>();
  s.work = B.work.as<unsigned long long>();
  s.queue = B.queue.as<long long>();
  s.qtot = B.qtot.as<float2>();
  s.qmax = p->qmax;
  {
    const double R = p->qmax + std::sqrt(static_cast<double>(p->m)) + 1.0;
    s.kim_f32_guard = 72.0 * 0x1.0p-24 * R * R * 1.01;
  }
  s.qhead = B.qctr.as<unsigned long long>();
  s.qtail = B.qctr.as<unsigned long long>() + 1;
  s.chunks_done = B.qctr.as<unsigned long long>() + 2;
  s.direct_chunk = 4;
  s.stride = 1;
  s.chunk_span = 0;
  s.ad_k = p->ad_k;
  s.direct = 0;
  s.screen_rows = p->screen_rows;
  s.probe_strips = static_cast<int>(p->ctx->opt[kOptProbeStrips]);
  s.gscratch = p->gmem ? B.scratch.as<double>() : nullptr;
  s.producer_smsp = static_cast<int>(p->ctx->opt[kOptProducers]);
  {
    // z-normalised rows satisfy |c| <= sqrt(m - 1); the engine checks the
    // bound per strip (degenerate statistics fall back to the exact engine)
    const double cmax = std::sqrt(static_cast<double>(p->m)) + 1.0;
    const F32Guard g = make_f32_guard(static_cast<int>(p->m), static_cast<int>(p->m), cmax, p->qmax);
    s.use_f32 = p->use_f32;
    s.f32_a = g.a;
    s.f32_b = g.b;
    s.f32_ia = std::nextafter(static_cast<float>(1.0 / static_cast<double>(g.a)) , 0.0f);
    s.f32_cmax = static_cast<float>(cmax);
  }
  s.counters = B.counters.as<unsigned long long>();
  s.index_offset = static_cast<long long>(p->offset);
  if (p->spec_active && !p->spec_final) {
    // Speculative statistics: every normalised value is within
    // dc = eps (1 + |c|) <= eps (2 + sqrt(m)) of the chain's.  A lower bound or
    // a DTW over at most 2m cells then moves by at most dc sqrt(2m) in its
    // square root (Minkowski): the sqrt-term of lb_guard and its square; the
    // FP32 screen's guard takes dc through its value factor; cb_eps widens the
    // cumulative-bound guard (kernels.cu: cb_guard).
    const double sm = std::sqrt(static_cast<double>(p->m));
    const double dc = p->spec_eps * (2.0 + sm);
    const double dsq = dc * std::sqrt(2.0 * static_cast<double>(p->m));
    s.approx = 1;
    s.mean = B.mean_a.as<double>();
    s.sd = B.sd_a.as<double>();
    s.guard_sqrt += 2.5 * dsq;
    s.guard_abs += 1.5 * dsq * dsq;
    s.cb_eps = 2.5 * dc;
    s.vlist = B.vlist.as<long long>();
    s.vcount = B.spec.as<unsigned long long>() + 2;
    s.vcap = p->vcap;
    const double cmax = sm + 1.0;
    const double up = 0x1.0p-24 + 0x1.0p-49;
    const F32Guard g = make_f32_guard(static_cast<int>(p->m), static_cast<int>(p->m), cmax, p->qmax,
                                      1.0 + 1.5 * p->spec_eps * (2.0 + sm) / (up * cmax));
    s.f32_a = g.a;
    s.f32_b = g.b;
    s.f32_ia = std::nextafter(static_cast<float>(1.0 / static_cast<double>(g.a)), 0.0f);
  }
  return s;
}

// ---- preparation stages (each enqueued on the context stream) ----
// first: decides whether the EC tier exists (the envelope window fits a tile)
static int stage_env(eapdtw_search_plan* p, long long tile_b, long long tile_e, bool first,
                     cudaStream_t stream = nullptr) {
  PlanBuffers& B = *p->buf;
  if (!(p->use_lb && p->m >= 2)) return EAPDTW_OK;
  if (!first && !p->have_env) return EAPDTW_OK;
  const cudaError_t e = launch_envelope(p->ref, static_cast<long long>(p->n), p->env_r,
                                        B.env.as<double>(), stream ? stream : p->ctx->stream,
                                        tile_b, tile_e);
  if (e == cudaSuccess) {
    if (first) p->have_env = true;
    ++p->ctx->launches;
  } else if (e != cudaErrorInvalidValue) {
    return fail(EAPDTW_ECUDA, std::string("envelope: ") + cudaGetErrorString(e));
  } else {
    cudaGetLastError();  // window too wide for the tile: EC tier skipped
  }
  return EAPDTW_OK;
}

// Stats chain (segments [seg_b, seg_e)) on the context stream and, beside it
// on the side stream, the envelope (tiles [tile_b, tile_e)): the chain is
// latency-bound and holds one SM per 16 segments exclusively, so the envelope
// runs on the other SMs.  The context stream continues once both are done.  `stats` false: the
// statistics are already in the buffers (a series' cached stats).  `mid`:
// recorded on the context stream after the statistics (phase timings).
static int stage_stats_env(eapdtw_search_plan* p, long long seg_b, long long seg_e,
                           long long tile_b, long long tile_e, bool first, bool stats = true,
                           cudaEvent_t mid = nullptr) {
  eapdtw_ctx* c = p->ctx;
  PlanBuffers& B = *p->buf;
  cudaStream_t s = c->stream;
  const bool env = p->use_lb && p->m >= 2 && (first || p->have_env);
  const long long n = static_cast<long long>(p->n);
  if (!c->opt[kOptPrepOverlap]) {  // serial: chain, conversion, envelope
    if (stats) {
      CUDA_TRY(launch_stats(p->ref, n, static_cast<int>(p->m), B.mean.as<double>(), B.sd.as<double>(), s,
                            seg_b, seg_e));
      c->launches += kStatsLaunches;
    }
    if (mid) CUDA_TRY(cudaEventRecord(mid, s));
    return env ? stage_env(p, tile_b, tile_e, first) : EAPDTW_OK;
  }
  const int m = static_cast<int>(p->m);
  if (env) {
    if (!c->aux) {
      CUDA_TRY(cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking));
      CUDA_TRY(cudaEventCreateWithFlags(&c->aux_fork, cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&c->aux_join, cudaEventDisableTiming));
    }
    CUDA_TRY(cudaEventRecord(c->aux_fork, s));  // before the chain: the envelope must not wait for it
  }
  if (stats) {
    CUDA_TRY(launch_stats(p->ref, n, m, B.mean.as<double>(), B.sd.as<double>(), s, seg_b, seg_e));
    c->launches += kStatsLaunches;
  }
  if (env) {
    CUDA_TRY(cudaStreamWaitEvent(c->aux, c->aux_fork, 0));
    const int e = stage_env(p, tile_b, tile_e, first, c->aux);
    if (e) return e;
    CUDA_TRY(cudaEventRecord(c->aux_join, c->aux));
  }
  if (mid) CUDA_TRY(cudaEventRecord(mid, s));
  if (env) CUDA_TRY(cudaStreamWaitEvent(s, c->aux_join, 0));
  return EAPDTW_OK;
}

// Probe: evaluate evenly spaced candidates of [0, cand_end) first (no lower
// bounds, running threshold) so the sweep starts from a finite best-so-far.
// Probe hits are real candidates, so they legitimately enter the (d, index)
// record.
// The upper-bound wave pays off for wide bands only (cfg4: -0.7 ms; w/16 < 4
// makes the narrow band too loose a bound, cfg2 +0.1 ms).
static bool rank_ub_applies(const eapdtw_search_plan* p) { return p->rank_ub && p->w_eff >= 64; }

// The rank pass costs about a millisecond (its cascade ends in a tail of long
// DTWs) and pays through the sweep's better threshold, i.e. with the size of
// the search.  Measured on prefixes of cfg4 (m = 1024, tools/shard_emul.py):
// 5e7 candidates 27.0 ms with it / 28.8 without, 2.5e7 19.5 / 18.8, 1.25e7
// 13.3 / 11.8; cfg3 (1e7, m = 512) 2.6 / 2.15, cfg2 0.51 / 0.28 (device
// phases).  Option rank_min: the smallest range it runs on.
static bool rank_applies(const eapdtw_search_plan* p, size_t cb, size_t ce) {
  return p->rank_stride > 0 && p->use_lb && p->m >= 2 && p->algo != EAPDTW_ALGO_FULL &&
         static_cast<long long>(ce - cb) >= 64 * p->rank_stride &&
         static_cast<long long>(ce - cb) >= p->ctx->opt[kOptRankMin];
}

static int stage_probe(eapdtw_search_plan* p, size_t cand_end) {
  // the rank pass's upper-bound wave gives the first finite threshold
  if (rank_ub_applies(p) && rank_applies(p, 0, cand_end) && !p->probe_force) return EAPDTW_OK;
  PlanBuffers& B = *p->buf;
  cudaStream_t s = p->ctx->stream;
  const size_t nprobe =
      std::min<size_t>(static_cast<size_t>(p->probe), std::max<size_t>(1, cand_end / 64));
  SearchParams sp = base_params(p);
  if (!p->ctx->opt[kOptProbeWarm]) sp.probe_strips = 0;
  sp.use_lb = 0;
  sp.tighten = 0;
  sp.begin = 0;
  sp.stride = static_cast<long long>(std::max<size_t>(1, cand_end / nprobe));
  sp.end = std::min<long long>(static_cast<long long>(cand_end),
                               sp.stride * static_cast<long long>(nprobe));
  sp.counters = B.probe_counters.as<unsigned long long>();
  sp.direct_chunk = 1;
  sp.direct = 1;
  // (A probe in a band of w/4, thresholds only, measured slower on cfg4 shards:
  // probe 1.1 -> 0.5 ms, but the looser threshold costs the sweep 2 ms.)
  CUDA_TRY(reset_work(p, static_cast<long long>(nprobe), s));
  CUDA_TRY(launch_search(sp, p->blocks, p->warps, s));
  ++p->ctx->launches;
  return EAPDTW_OK;
}

// Coarse pass over [cb, ce): the full cascade over every coarse_stride-th
// candidate, so the sweep starts from a threshold close to the final one
// (neighbouring windows normalise to nearly the same series).  Its candidates
// are real, so their exact results enter the record; their work is counted
// with the probe's.
// Rank pass over [cb, ce) (kernels.cu: rank_kernel): the layered LB_Kim of
// every rank_stride-th candidate, then the full cascade over the ~rank_k with
// the smallest bound.  Real candidates: their exact results enter the record,
// their work counts with the probe's.
static int stage_rank(eapdtw_search_plan* p, size_t cb, size_t ce) {
  if (!rank_applies(p, cb, ce)) return EAPDTW_OK;
  const long long S = p->rank_stride;
  PlanBuffers& B = *p->buf;
  cudaStream_t s = p->ctx->stream;
  const long long cap = 4 * p->rank_k;
  CUDA_TRY(B.rank.ensure(rank_scratch_bytes(static_cast<long long>(ce - cb), S)));
  CUDA_TRY(B.rlist.ensure(static_cast<size_t>(cap) * 8 + 64));
  SearchParams rp = base_params(p);
  if (!p->ctx->opt[kOptProbeWarm]) rp.probe_strips = 0;
  if (!p->ctx->opt[kOptWarmF32]) rp.use_f32 = 0;
  rp.begin = static_cast<long long>(cb);
  rp.end = static_cast<long long>(ce);
  rp.counters = B.probe_counters.as<unsigned long long>();
  long long* list = B.rlist.as<long long>();
  unsigned long long* nlist = reinterpret_cast<unsigned long long*>(list + cap);
  CUDA_TRY(launch_rank(rp, S, B.rank.p, s));
  ++p->ctx->launches;
  rp.list = list;
  rp.nlist = nlist;
  rp.list_cap = cap;
  const long long nsamp = (static_cast<long long>(ce - cb) + S - 1) / S;
  // Upper-bound wave: the rank_k/16 best-ranked candidates' DTW in a band of
  // w/16 cells.  Fewer paths, so each value is >= that candidate's DTW (the
  // FP DP is monotone in its predecessor set): a valid threshold, computed
  // ~16x cheaper than the full-band DTW; it tightens the key only (ub_only).
  int wave = 0;
  if (rank_ub_applies(p)) {
    SearchParams up = rp;
    up.direct = 1;
    up.direct_chunk = 1;
    up.use_lb = 0;
    up.tighten = 0;
    up.ub_only = 1;
    // band w/4 measured best of w/16, w/8, w/4, w/2 (cfg4 -0.5 ms vs w/16)
    const int wdiv = p->rank_ub_w, kdiv = p->rank_ub_k;
    up.w = std::max(0, p->w_eff / wdiv);
    CUDA_TRY(launch_rank_select(up, S, wave, std::max<long long>(32, p->rank_k / kdiv), cap,
                                B.rank.p, list, nlist, s));
    p->ctx->launches += 2;
    CUDA_TRY(reset_work(p, 0, s));
    CUDA_TRY(launch_search(up, p->blocks, p->warps, s));
    ++p->ctx->launches;
    ++wave;
  }
  // then the cascade over the ranks past it (waves of growing rank, each
  // starting from the threshold the better-ranked candidates before it left)
  if (!p->rank_cascade) return EAPDTW_OK;
  for (long long k = std::max<long long>(32, p->rank_k >> (4 * (p->rank_waves - 1)));;
       k = std::min(p->rank_k, k << 4), ++wave) {
    CUDA_TRY(launch_rank_select(rp, S, wave, k, cap, B.rank.p, list, nlist, s));
    p->ctx->launches += 2;
    CUDA_TRY(reset_work(p, std::min(cap, nsamp), s));  // the queue holds ncand + slack slots
    CUDA_TRY(launch_search(rp, p->blocks, p->warps, s));
    ++p->ctx->launches;
    if (k >= p->rank_k || wave >= 14) break;
  }
  return EAPDTW_OK;
}

static int stage_coarse(eapdtw_search_plan* p, size_t cb, size_t ce) {
  const int stride = p->coarse_stride;
  if (stride <= 1 || ce - cb < 64 * static_cast<size_t>(stride)) return EAPDTW_OK;
  PlanBuffers& B = *p->buf;
  cudaStream_t s = p->ctx->stream;
  SearchParams cp = base_params(p);
  cp.begin = static_cast<long long>(cb);
  cp.end = static_cast<long long>(ce);
  cp.counters = B.probe_counters.as<unsigned long long>();
  cp.stride = stride;
  const long long count = (cp.end - cp.begin + cp.stride - 1) / cp.stride;
  CUDA_TRY(reset_work(p, count, s));
  CUDA_TRY(launch_search(cp, p->blocks, p->warps, s));
  ++p->ctx->launches;
  return EAPDTW_OK;
}

int eapdtw_search_plan_prepare(eapdtw_search_plan* p) {
  if (!p) return fail(EAPDTW_EINVAL, "null plan");
  eapdtw_ctx* c = p->ctx;
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  int e;
  CUDA_TRY(cudaEventRecord(p->ev[0], s));
  p->have_env = false;
  p->runs.clear();
  p->spec_final = false;
  // auto: where the chain's ~1.8 ms outweigh what the wider guards cost the
  // sweep (cfg2 2.37 -> 1.98 ms, cfg3 4.25 -> 3.10; at cfg4 the guards cost 7%
  // more DTW work, 45.7 -> 50.9 ms; the guards grow with m: a 1.25e7-candidate
  // shard of cfg4, m = 1024, breaks even, 13.5 ms either way)
  const long long spec_opt = c->opt[kOptSpecStats];
  p->spec_active = p->spec && !p->stats_ready &&
                   (spec_opt == 1 || (spec_opt < 0 && c->spec_cooldown == 0 && p->ncand <= 40000000 &&
                                      static_cast<double>(p->ncand) * static_cast<double>(p->m) <= 8e9)) &&
                   fast_stats_tile(static_cast<int>(p->m)) > 0 && p->ncand >= 1000;
  if (!p->spec_active && c->spec_cooldown > 0 && p->spec && !p->stats_ready) --c->spec_cooldown;
  if (p->spec_active) {
    // The exact chain first, on its own stream (its blocks take their SMs
    // before the search kernels fill the GPU), then the prefix-sum statistics
    // on the context stream; the verification follows the chain.
    PlanBuffers& B = *p->buf;
    const long long n = static_cast<long long>(p->n);
    const int m = static_cast<int>(p->m);
    p->spec_eps = static_cast<double>(c->opt[kOptSpecEps]) * 1e-9;
    p->vcap = static_cast<long long>(std::min<size_t>(p->ncand, size_t{1} << 20));
    CUDA_TRY(B.mean_a.ensure(p->ncand * 8));
    CUDA_TRY(B.sd_a.ensure(p->ncand * 8));
    CUDA_TRY(B.vlist.ensure(static_cast<size_t>(p->vcap) * 8));
    CUDA_TRY(B.spec.ensure(32));
    if (!c->aux2) {
      CUDA_TRY(cudaStreamCreateWithFlags(&c->aux2, cudaStreamNonBlocking));
      CUDA_TRY(cudaEventCreateWithFlags(&c->spec_fork, cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&c->spec_fast, cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&c->spec_done, cudaEventDisableTiming));
    }
    CUDA_TRY(cudaMemsetAsync(B.spec.p, 0, 32, s));
    CUDA_TRY(cudaEventRecord(c->spec_fork, s));
    CUDA_TRY(cudaStreamWaitEvent(c->aux2, c->spec_fork, 0));
    CUDA_TRY(launch_stats(p->ref, n, m, B.mean.as<double>(), B.sd.as<double>(), c->aux2, 0, -1));
    c->launches += kStatsLaunches;
    CUDA_TRY(launch_fast_stats(p->ref, n, m, B.mean_a.as<double>(), B.sd_a.as<double>(), s));
    ++c->launches;
    CUDA_TRY(cudaEventRecord(c->spec_fast, s));
    CUDA_TRY(cudaStreamWaitEvent(c->aux2, c->spec_fast, 0));
    CUDA_TRY(launch_stats_verify(B.mean.as<double>(), B.sd.as<double>(), B.mean_a.as<double>(),
                                 B.sd_a.as<double>(), static_cast<long long>(p->ncand),
                                 B.spec.as<unsigned long long>(), c->aux2));
    ++c->launches;
    CUDA_TRY(cudaEventRecord(c->spec_done, c->aux2));
  }
  if ((e = stage_stats_env(p, 0, -1, 0, -1, true, !p->stats_ready && !p->spec_active, p->ev[1])))
    return e;
  CUDA_TRY(cudaEventRecord(p->ev[2], s));
  if ((e = stage_probe(p, p->ncand))) return e;
  if ((e = stage_rank(p, 0, p->ncand))) return e;
  if ((e = stage_coarse(p, 0, p->ncand))) return e;
  CUDA_TRY(cudaEventRecord(p->ev[3], s));
  p->prepared = true;
  return EAPDTW_OK;
}

int eapdtw_search_plan_run(eapdtw_search_plan* p, size_t begin, size_t end) {
  if (!p) return fail(EAPDTW_EINVAL, "null plan");
  if (!p->prepared) {
    const int e = eapdtw_search_plan_prepare(p);
    if (e) return e;
  }
  end = std::min(end, p->ncand);
  if (begin >= end) return EAPDTW_OK;
  eapdtw_ctx* c = p->ctx;
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  SearchParams sp = base_params(p);
  sp.begin = static_cast<long long>(begin);
  sp.end = static_cast<long long>(end);
  sp.stride = 1;
  if (!p->ran) CUDA_TRY(cudaEventRecord(p->ev[4], s));
  if (p->spec_active) p->runs.emplace_back(begin, end);
  CUDA_TRY(reset_work(p, static_cast<long long>(end - begin), s));
  CUDA_TRY(launch_search(sp, p->blocks, p->warps, s));
  ++c->launches;
  CUDA_TRY(cudaEventRecord(p->ev[5], s));
  p->ran = true;
  return EAPDTW_OK;
}

int eapdtw_search_plan_result(eapdtw_search_plan* p, eapdtw_search_result* out) {
  if (!p || !out) return fail(EAPDTW_EINVAL, "null argument");
  eapdtw_ctx* c = p->ctx;
  PlanBuffers& B = *p->buf;
  CUDA_TRY(cudaSetDevice(c->device));
  unsigned long long spec_out[4] = {0, 0, 0, 0};
  if (p->spec_active) {
    if (!p->spec_final) {
      // The chain and its verification are done: the completed candidates
      // again, now with the exact statistics (every one a DTW task; the
      // threshold key holds a valid upper bound, the record takes the values).
      CUDA_TRY(cudaStreamWaitEvent(c->stream, c->spec_done, 0));
      p->spec_final = true;
      SearchParams xp = base_params(p);
      xp.direct = 1;
      xp.direct_chunk = 1;
      xp.use_lb = 0;
      xp.tighten = 0;
      xp.begin = 0;
      xp.end = static_cast<long long>(p->ncand);
      xp.list = B.vlist.as<long long>();
      xp.nlist = B.spec.as<unsigned long long>() + 2;
      xp.list_cap = p->vcap;
      // second evaluations: counted with the warm start's work, not as candidates
      xp.counters = B.probe_counters.as<unsigned long long>();
      CUDA_TRY(reset_work(p, 0, c->stream));
      CUDA_TRY(launch_search(xp, p->blocks, p->warps, c->stream));
      ++c->launches;
    }
    CUDA_TRY(cudaMemcpyAsync(spec_out, B.spec.p, 32, cudaMemcpyDeviceToHost, c->stream));
  }
  BestRecord rec{};
  unsigned long long cnt[kNumCountersExt], pc[kNumCountersExt];
  CUDA_TRY(cudaMemcpyAsync(&rec, B.best.p, sizeof(rec), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaMemcpyAsync(cnt, B.counters.p, sizeof(cnt), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaMemcpyAsync(pc, B.probe_counters.p, sizeof(pc), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  c->spec_dev = -1.0;
  if (p->spec_active) {
    double dev;
    std::memcpy(&dev, &spec_out[0], 8);
    c->spec_dev = dev;
    c->spec_listed = spec_out[2];
    if (!(dev <= p->spec_eps) || spec_out[1] != 0 ||
        spec_out[2] > static_cast<unsigned long long>(p->vcap)) {
      // The prefix-sum statistics were further from the chain's than assumed
      // (or disagreed on a constant window, or too many candidates completed):
      // nothing of the speculative pass is kept.  Search again on the exact
      // statistics, which are in the buffers now.
      const std::vector<std::pair<size_t, size_t>> runs = p->runs;
      p->spec = false;
      ++g_spec_fallbacks;
      // data like this would fail again: the context's next searches do not
      // speculate (one-shot searches build a new plan per call)
      c->spec_cooldown = 64;
      int e = eapdtw_search_plan_reset(p);
      p->stats_ready = true;
      if (!e) e = eapdtw_search_plan_prepare(p);
      p->stats_ready = false;
      for (const auto& r : runs)
        if (!e) e = eapdtw_search_plan_run(p, r.first, r.second);
      return e ? e : eapdtw_search_plan_result(p, out);
    }
  }
  std::memset(out, 0, sizeof(*out));
  out->found = rec.d != kInf ? 1 : 0;
  out->distance_sq = rec.d;
  out->location = out->found ? rec.idx : 0;
  out->candidates_total = cnt[kCntCandidates];
  out->pruned_kim = cnt[kCntKim];
  out->pruned_keogh_eq = cnt[kCntKeoghEq];
  out->pruned_keogh_ec = cnt[kCntKeoghEc];
  out->dtw_calls = cnt[kCntDtwCalls];
  out->dtw_abandoned = cnt[kCntDtwAbandoned];
  // dp_cells_evaluated: every DP cell the search's kernels evaluated, as the
  // reference counts its kernel's cells (dtw.cpp:28-33) -- the exact FP64
  // engines, the phase-A lane prefix, and the FP32 screening pass, which
  // evaluates the same cells at lower precision (its share is
  // screen_cells_evaluated).  Warm-start candidates are real candidates and
  // count like the sweep's.
  out->screen_cells_evaluated = cnt[kCntCellsF32] + pc[kCntCellsF32];
  out->dp_cells_evaluated = cnt[kCntCells] + pc[kCntCells] + out->screen_cells_evaluated;
  out->elapsed_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - p->t0).count();
#ifdef EAPDTW_PHASE_CLOCKS
  {
    unsigned long long dbg[16];
    debug_read_reset(dbg);
    std::fprintf(stderr, "strips/DTW bins [1,2,3-4,5-8,9-16,17+]: calls %llu %llu %llu %llu %llu %llu | steps %llu %llu %llu %llu %llu %llu\n",
                 dbg[2], dbg[3], dbg[4], dbg[5], dbg[6], dbg[7], dbg[8], dbg[9], dbg[10], dbg[11], dbg[12], dbg[13]);
    std::fprintf(stderr, "strip steps %llu strips %llu cells %llu (f32 %llu) -> lane eff %.3f\n", dbg[0], dbg[1],
                 cnt[kCntCells], cnt[kCntCellsF32], (cnt[kCntCells] + cnt[kCntCellsF32]) / (32.0 * dbg[0] + 1));
  }
  std::fprintf(stderr,
               "phase warp-Gcycles: total %.3f dtw %.3f eq %.3f ec %.3f screen %.3f kim %.3f wait %.3f | "
               "stage hit %llu miss %llu\n",
               cnt[kClkTotal] * 1e-9, cnt[kClkDtw] * 1e-9, cnt[kClkEq] * 1e-9, cnt[kClkEc] * 1e-9,
               cnt[kClkScreen] * 1e-9, cnt[kClkKim] * 1e-9, cnt[kClkWait] * 1e-9, cnt[kStageHit],
               cnt[kStageMiss]);
#endif
  return EAPDTW_OK;
}

int eapdtw_search_plan_counters(eapdtw_search_plan* p, uint64_t* out8) {  // 10 entries
  if (!p || !out8) return fail(EAPDTW_EINVAL, "null argument");
  CUDA_TRY(cudaSetDevice(p->ctx->device));
  unsigned long long cnt[kNumCounters];
  CUDA_TRY(cudaMemcpyAsync(cnt, p->buf->counters.p, sizeof(cnt), cudaMemcpyDeviceToHost,
                           p->ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(p->ctx->stream));
  for (int k = 0; k < 10; ++k) out8[k] = k < kNumCounters ? cnt[k] : 0;
  return EAPDTW_OK;
}

int eapdtw_search_plan_timings(eapdtw_search_plan* p, float* ms4) {
  if (!p || !ms4) return fail(EAPDTW_EINVAL, "null argument");
  CUDA_TRY(cudaSetDevice(p->ctx->device));
  CUDA_TRY(cudaEventSynchronize(p->ev[5]));
  CUDA_TRY(cudaEventElapsedTime(&ms4[0], p->ev[0], p->ev[1]));
  CUDA_TRY(cudaEventElapsedTime(&ms4[1], p->ev[1], p->ev[2]));
  CUDA_TRY(cudaEventElapsedTime(&ms4[2], p->ev[2], p->ev[3]));
  CUDA_TRY(cudaEventElapsedTime(&ms4[3], p->ev[4], p->ev[5]));
  return EAPDTW_OK;
}

int eapdtw_search_plan_destroy(eapdtw_search_plan* p) {
  if (!p) return EAPDTW_OK;
  if (p->ctx) {
    cudaSetDevice(p->ctx->device);
    cudaStreamSynchronize(p->ctx->stream);
    // a speculative preparation's chain may still be writing the plan's buffers
    if (p->ctx->aux2) cudaStreamSynchronize(p->ctx->aux2);
    if (p->ctx->aux) cudaStreamSynchronize(p->ctx->aux);
  }
  p->own.release();
  for (auto& ev : p->ev)
    if (ev) cudaEventDestroy(ev);
  delete p;
  return EAPDTW_OK;
}

// Cached sliding statistics of a device-resident series for one query length
// (the chain depends on the reference and m only, search.cpp:156-168): the
// grid's 5 window ratios per length share one stats pass.
// One cache per (series, context): a context's copies are ordered on its own
// stream, so contexts on other host threads searching the same series each
// keep their own entry.
struct SeriesStats {
  DevBuf mean, sd;
  size_t m = 0;  // 0: empty
};

static int one_shot(eapdtw_ctx* c, const double* ref_dev, size_t n, const double* query,
                    size_t qlen, const eapdtw_search_config* cfg, bool check_ref,
                    eapdtw_search_result* out, SeriesStats* cache = nullptr) {
  if (!c || !cfg || !out) return fail(EAPDTW_EINVAL, "null argument");
  eapdtw_search_plan p;
  p.buf = &c->pb;  // reuse the context's grow-only scratch
  int e = plan_init(&p, c, ref_dev, n, query, qlen, cfg, 0);
  bool fill_cache = false;
  if (cache) p.spec = false;  // a cached series wants the exact statistics on the context stream
  if (!e && cache) {
    const size_t bytes = p.ncand * 8;
    if (cache->m == p.m) {
      if (cudaMemcpyAsync(c->pb.mean.p, cache->mean.p, bytes, cudaMemcpyDeviceToDevice, c->stream) ||
          cudaMemcpyAsync(c->pb.sd.p, cache->sd.p, bytes, cudaMemcpyDeviceToDevice, c->stream))
        e = fail(EAPDTW_ECUDA, "series stats cache: copy failed");
      p.stats_ready = true;
    } else {
      fill_cache = true;
    }
  }
  if (!e && check_ref) {
    // Series validation (series.hpp:24-31) of the reference, on the device.
    CUDA_TRY(cudaMemsetAsync(c->pb.flag.p, 0, 8, c->stream));
    CUDA_TRY(launch_check_finite(ref_dev, static_cast<long long>(n),
                                 c->pb.flag.as<unsigned long long>(), c->stream));
    ++c->launches;
  }
  if (!e) e = eapdtw_search_plan_prepare(&p);
  if (!e && fill_cache) {
    const size_t bytes = p.ncand * 8;
    cache->m = 0;  // the cache is optional: on any failure it simply stays empty
    if (!cache->mean.ensure(bytes) && !cache->sd.ensure(bytes) &&
        !cudaMemcpyAsync(cache->mean.p, c->pb.mean.p, bytes, cudaMemcpyDeviceToDevice, c->stream) &&
        !cudaMemcpyAsync(cache->sd.p, c->pb.sd.p, bytes, cudaMemcpyDeviceToDevice, c->stream))
      cache->m = p.m;
    else
      cudaGetLastError();
  }
  if (!e) e = eapdtw_search_plan_run(&p, 0, p.ncand);
  if (!e) e = eapdtw_search_plan_result(&p, out);
  if (!e && check_ref) {
    unsigned long long bad = 0;
    CUDA_TRY(cudaMemcpy(&bad, c->pb.flag.p, 8, cudaMemcpyDeviceToHost));
    if (bad) e = fail(EAPDTW_EINVAL, "Series: non-finite sample in the reference");
  }
  for (auto& ev : p.ev)
    if (ev) cudaEventDestroy(ev);
  p.buf = &p.own;
  return e;
}

int eapdtw_similarity_search_dev(eapdtw_ctx* c, const double* ref_dev, size_t n,
                                 const double* query, size_t qlen,
                                 const eapdtw_search_config* cfg, eapdtw_search_result* out) {
  return one_shot(c, ref_dev, n, query, qlen, cfg, true, out);
}

// ---------------------------------------------------------------------------
// Device-resident series: one upload (and one Series validation,
// series.hpp:24-31) serves many searches -- the CLI's query-length x
// window-ratio grid (eapdtw_cli.cpp:110-142) and multi-query drivers.
// ---------------------------------------------------------------------------
struct eapdtw_series {
  int device = 0;
  DevBuf data;
  size_t n = 0;
  std::mutex mu;  // guards the map, not the entries (one host thread per context)
  std::map<const eapdtw_ctx*, std::unique_ptr<SeriesStats>> stats;  // last m's stats, per context
};

int eapdtw_series_upload(eapdtw_ctx* c, const double* host, size_t n, eapdtw_series** out) {
  if (!c || !host || !out) return fail(EAPDTW_EINVAL, "null argument");
  if (n == 0) return fail(EAPDTW_EINVAL, "Series: empty input");
  *out = nullptr;
  CUDA_TRY(cudaSetDevice(c->device));
  auto* s = new eapdtw_series;
  s->device = c->device;
  s->n = n;
  cudaError_t e = s->data.ensure(n * 8);
  if (e == cudaSuccess) e = cudaMemcpyAsync(s->data.p, host, n * 8, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = c->pb.flag.ensure(8);
  if (e == cudaSuccess) e = cudaMemsetAsync(c->pb.flag.p, 0, 8, c->stream);
  if (e == cudaSuccess) {
    e = launch_check_finite(s->data.as<double>(), static_cast<long long>(n),
                            c->pb.flag.as<unsigned long long>(), c->stream);
    ++c->launches;
  }
  unsigned long long bad = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&bad, c->pb.flag.p, 8, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess || bad) {
    s->data.release();
    delete s;
    if (e != cudaSuccess) return fail(EAPDTW_ECUDA, std::string("series_upload: ") + cudaGetErrorString(e));
    return fail(EAPDTW_EINVAL, "Series: non-finite sample in the reference");
  }
  *out = s;
  return EAPDTW_OK;
}

const double* eapdtw_series_device_ptr(const eapdtw_series* s) {
  return s ? s->data.as<const double>() : nullptr;
}

size_t eapdtw_series_length(const eapdtw_series* s) { return s ? s->n : 0; }

int eapdtw_series_free(eapdtw_series* s) {
  if (!s) return EAPDTW_OK;
  cudaSetDevice(s->device);
  cudaDeviceSynchronize();
  s->data.release();
  for (auto& kv : s->stats) {
    kv.second->mean.release();
    kv.second->sd.release();
  }
  delete s;
  return EAPDTW_OK;
}

int eapdtw_similarity_search_series(eapdtw_ctx* c, eapdtw_series* ref, const double* query,
                                    size_t qlen, const eapdtw_search_config* cfg,
                                    eapdtw_search_result* out) {
  if (!c || !ref) return fail(EAPDTW_EINVAL, "null argument");
  if (ref->device != c->device) return fail(EAPDTW_EINVAL, "series lives on another device");
  if (c->opt[kOptSeriesCache] == 0)
    return one_shot(c, ref->data.as<const double>(), ref->n, query, qlen, cfg, false, out);
  SeriesStats* cache = nullptr;
  {
    std::lock_guard<std::mutex> lock(ref->mu);
    auto& slot = ref->stats[c];
    if (!slot) slot = std::make_unique<SeriesStats>();
    cache = slot.get();
  }
  return one_shot(c, ref->data.as<const double>(), ref->n, query, qlen, cfg, false, out, cache);
}

// Host-pointer search of a long reference, streamed: the reference goes to the
// device in two parts on a copy stream, and the second part's copy runs under
// the first part's sweep.  Part 1 is the candidates of the first half of the
// 100000-candidate stats segments (plus the data their statistics and
// envelope need); its preparation (stats, envelope, probe over part 1,
// coarse pass over part 1) and sweep start as soon as part 1 has arrived.
// Part 2 then gets its stats, envelope, coarse pass and sweep.  The threshold
// and the (d, index) record carry over, so the result is the whole search's.
static int one_shot_streamed(eapdtw_ctx* c, const double* host_ref, size_t n,
                             const double* query, size_t qlen, const eapdtw_search_config* cfg,
                             eapdtw_search_result* out) {
  // The copies are issued first, so they overlap the host-side plan set-up
  // (query preparation, buffers): the split depends on n and m only.
  const size_t m = cfg->query_length == 0 ? qlen : cfg->query_length;
  const size_t ncand = n - m + 1;
  const long long nseg = static_cast<long long>((ncand + kStatsResetInterval - 1) / kStatsResetInterval);
  // Part 1 (3/8 of the candidates): everything waits for its copy, while
  // part 2's copy hides under part 1's stats, warm start and sweep.  Shares
  // of 1/8 .. 4/8 measured within noise (cfg4 e2e 61-64 ms; the second stats
  // chain and envelope, not the first copy, are what remains exposed).
  // Option stream_split = part 1's share in eighths.
  const long long eighths = c->opt[kOptStreamSplit];
  const long long seg1 = std::max<long long>(1, nseg * eighths / 8);
  const size_t c1 = static_cast<size_t>(seg1) * kStatsResetInterval;
  // data part 1 needs: its stats windows (< c1 + m - 1) and the envelope
  // tiles covering the positions its candidates' EC tier reads, each with
  // radius r <= m: within c1 + 2m + the largest tile (8192)
  const size_t d1 = std::min(n, c1 + 2 * m + 8192);
  double* dref = c->ref.as<double>();
  eapdtw_search_plan p;
  p.buf = &c->pb;
  // Every return after the copies are queued goes through finish(): an error
  // must not leave the copy stream reading the caller's host buffer.
  bool queued = false;
  auto finish = [&](int rc) {
    if (queued) cudaStreamSynchronize(c->copy);
    for (auto& ev : p.ev)
      if (ev) cudaEventDestroy(ev);
    p.buf = &p.own;
    return rc;
  };
#define CUDA_TRY_F(expr)                                                                   \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return finish(fail(EAPDTW_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_))); \
  } while (0)
  if (!c->copy) {
    CUDA_TRY_F(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
    for (cudaEvent_t& ev : c->copied)
      CUDA_TRY_F(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  if (!c->fork) CUDA_TRY_F(cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming));
  cudaStream_t s = c->stream;
  CUDA_TRY_F(cudaEventRecord(c->fork, s));  // the copy must not overtake earlier work on s
  CUDA_TRY_F(cudaStreamWaitEvent(c->copy, c->fork, 0));
  queued = true;
  CUDA_TRY_F(cudaMemcpyAsync(dref, host_ref, d1 * 8, cudaMemcpyHostToDevice, c->copy));
  CUDA_TRY_F(cudaEventRecord(c->copied[0], c->copy));
  CUDA_TRY_F(cudaMemcpyAsync(dref + d1, host_ref + d1, (n - d1) * 8, cudaMemcpyHostToDevice,
                             c->copy));
  CUDA_TRY_F(cudaEventRecord(c->copied[1], c->copy));

  int e = plan_init(&p, c, dref, n, query, qlen, cfg, 0);
  p.spec = false;  // the streamed parts run their stages themselves, on the exact chain
  if (e) return finish(e);
  long long te1 = 0;
  const int T = envelope_tile(p.env_r);
  if (p.use_lb && T >= 256) {
    // tiles [0, te1) read positions < te1*T + r <= c1 + 2m + T - 2 <= d1 (or n)
    te1 = static_cast<long long>((c1 + m - 1 + T - 1) / T);
  }
  CUDA_TRY_F(cudaEventRecord(p.ev[0], s));
  // ---- part 1
  CUDA_TRY_F(cudaStreamWaitEvent(s, c->copied[0], 0));
  CUDA_TRY_F(cudaMemsetAsync(c->pb.flag.p, 0, 8, s));
  CUDA_TRY_F(launch_check_finite(dref, static_cast<long long>(d1),
                                 c->pb.flag.as<unsigned long long>(), s));
  ++c->launches;
  p.have_env = false;
  if ((e = stage_stats_env(&p, 0, seg1, 0, te1, true))) return finish(e);
  if ((e = stage_probe(&p, c1))) return finish(e);
  if ((e = stage_rank(&p, 0, c1))) return finish(e);
  if ((e = stage_coarse(&p, 0, c1))) return finish(e);
  p.prepared = true;
  if ((e = eapdtw_search_plan_run(&p, 0, c1))) return finish(e);
  // ---- part 2
  CUDA_TRY_F(cudaStreamWaitEvent(s, c->copied[1], 0));
  if (n > d1) {
    CUDA_TRY_F(launch_check_finite(dref + d1, static_cast<long long>(n - d1),
                                   c->pb.flag.as<unsigned long long>(), s));
    ++c->launches;
  }
  if ((e = stage_stats_env(&p, seg1, -1, te1, -1, false))) return finish(e);
  if ((e = stage_coarse(&p, c1, ncand))) return finish(e);
  if ((e = eapdtw_search_plan_run(&p, c1, ncand))) return finish(e);
  if ((e = eapdtw_search_plan_result(&p, out))) return finish(e);
  unsigned long long bad = 0;
  CUDA_TRY_F(cudaMemcpy(&bad, c->pb.flag.p, 8, cudaMemcpyDeviceToHost));
  if (bad) return finish(fail(EAPDTW_EINVAL, "Series: non-finite sample in the reference"));
  return finish(EAPDTW_OK);
#undef CUDA_TRY_F
}

int eapdtw_similarity_search(eapdtw_ctx* c, const double* ref, size_t n, const double* query,
                             size_t qlen, const eapdtw_search_config* cfg,
                             eapdtw_search_result* out) {
  if (!c || !ref) return fail(EAPDTW_EINVAL, "null argument");
  if (n == 0) return fail(EAPDTW_EINVAL, "Series: empty input");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(c->ref.ensure(n * 8));
  // long references: overlap the second half's copy with the first half's
  // sweep (measured: cfg4 e2e +1.2%; below ~5e7 points the second stats
  // chain and coarse pass cost more than the hidden copy, e.g. cfg3 -30%)
  bool streamed = cfg && query && qlen > 0 && n >= 4 * static_cast<size_t>(kStatsResetInterval);
  if (c->opt[kOptStreamed] >= 0) streamed = streamed && c->opt[kOptStreamed] != 0;
  else streamed = streamed && n >= 50000000;
  if (streamed) {
    const size_t m = cfg->query_length == 0 ? qlen : cfg->query_length;
    streamed = m >= 1 && m <= qlen && m < n / 4;
  }
  if (streamed) return one_shot_streamed(c, ref, n, query, qlen, cfg, out);
  CUDA_TRY(cudaMemcpyAsync(c->ref.p, ref, n * 8, cudaMemcpyHostToDevice, c->stream));
  return one_shot(c, c->ref.as<double>(), n, query, qlen, cfg, true, out);
}

// ---------------------------------------------------------------------------
// NN1
// ---------------------------------------------------------------------------
// One NN1 launch over database rows db_dev[0, nd) against per-query threshold
// keys and (d, index) records already on the device (not re-initialised, so
// consecutive batches and shards carry them); recorded indices are the local
// row + index_offset.  counters: [FP64 cells, FP32 cells, dtw calls], added to.
static int nn1_launch(eapdtw_ctx* c, const double* q_dev, size_t nq, const double* db_dev,
                      size_t nd, size_t len, size_t window, unsigned long long* keys,
                      BestRecord* best, unsigned long long* counters, long long index_offset) {
  int w = (window == EAPDTW_UNBOUNDED_WINDOW || window >= len) ? static_cast<int>(len)
                                                              : static_cast<int>(window);
  Nn1Params p{};
  p.queries = q_dev;
  p.db = db_dev;
  p.nq = static_cast<long long>(nq);
  p.nd = static_cast<long long>(nd);
  p.len = static_cast<int>(len);
  p.w = w;
  // Many small blocks: a block's cost varies with its query, so with few
  // waves the last one leaves SMs idle (ncu: ALU-pipe use 58-95% across SMs
  // at 2 splits).  cfg5 (1000 queries) sweep of splits per query: 2 -> 187.8
  // ms, 4 -> 159.9, 6 -> 148.2, 10 -> 145.3, 16 -> 152.1 (the extra splits
  // re-warm more cutoffs).  ~64 blocks per SM, each block keeping at least 64
  // database rows.
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  const long long target = static_cast<long long>(sms) * 64;
  p.splits = static_cast<int>(std::max<long long>(1, std::min<long long>(
      static_cast<long long>(nd) / 64 + 1, (target + static_cast<long long>(nq) - 1) / static_cast<long long>(nq))));
  if (c->opt[kOptNn1Splits] > 0) p.splits = static_cast<int>(c->opt[kOptNn1Splits]);
  p.ad_k = c->opt[kOptAdK] >= 0 ? static_cast<int>(c->opt[kOptAdK]) : choose_ad_k(static_cast<int>(len), w);
  p.ub_keys = keys;
  p.best = best;
  p.cells = counters;
  p.dtw_calls = counters + 2;
  {
    // FP32 screen (dtw_f32.cuh) for z-normalised data: |values| <= sqrt(len)
    // + 1, checked per query (block) and per strip of database rows.
    const double cmax = std::sqrt(static_cast<double>(len)) + 1.0;
    const F32Guard g = make_f32_guard(static_cast<int>(len), static_cast<int>(len), cmax, cmax);
    p.use_f32 = static_cast<int>(c->opt[kOptF32]);
    p.f32_a = g.a;
    p.f32_b = g.b;
    p.f32_cmax = static_cast<float>(cmax);
  }
  p.guard_rel = std::max(1e-9, 8.0 * static_cast<double>(len) * 0x1.0p-53);
  p.guard_abs = 1e-20;
  p.warm = static_cast<int>(c->opt[kOptNn1Warm]);
  p.probe_strips = static_cast<int>(c->opt[kOptProbeStrips]);
  p.index_offset = index_offset;
  CUDA_TRY(launch_nn1(p, c->stream));
  ++c->launches;
  return EAPDTW_OK;
}

// Records -> (argmin, dist): a query with no row within its cutoff gets
// index 0 and +inf (the harness's strict < never fired).
static void nn1_unpack(const std::vector<BestRecord>& rec, uint64_t* argmin, double* dist) {
  for (size_t i = 0; i < rec.size(); ++i) {
    const bool none = rec[i].d == kInf;
    argmin[i] = none ? 0 : rec[i].idx;
    dist[i] = none ? kInf : rec[i].d;
  }
}

static int nn1_impl(eapdtw_ctx* c, const double* q_dev, size_t nq, const double* db_dev,
                    size_t nd, size_t len, size_t window, uint64_t* argmin, double* dist,
                    uint64_t* cells, const double* cutoff_dev = nullptr) {
  cudaStream_t s = c->stream;
  CUDA_TRY(c->best.ensure(nq * sizeof(BestRecord)));
  CUDA_TRY(c->keys.ensure(nq * 8));
  CUDA_TRY(c->counters.ensure(3 * 8));
  CUDA_TRY(cudaMemsetAsync(c->counters.p, 0, 24, s));
  CUDA_TRY(launch_init_best(c->best.as<BestRecord>(), c->keys.as<unsigned long long>(),
                            static_cast<long long>(nq), s));
  ++c->launches;
  // a starting cutoff per query: the threshold key is the bit pattern of a
  // non-negative double (order-preserving), so the cutoffs are copied in as is
  if (cutoff_dev)
    CUDA_TRY(cudaMemcpyAsync(c->keys.p, cutoff_dev, nq * 8, cudaMemcpyDeviceToDevice, s));
  int e = nn1_launch(c, q_dev, nq, db_dev, nd, len, window, c->keys.as<unsigned long long>(),
                     c->best.as<BestRecord>(), c->counters.as<unsigned long long>(), 0);
  if (e) return e;
  std::vector<BestRecord> rec(nq);
  unsigned long long cnt[3];
  CUDA_TRY(cudaMemcpyAsync(rec.data(), c->best.p, nq * sizeof(BestRecord), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaMemcpyAsync(cnt, c->counters.p, 24, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  nn1_unpack(rec, argmin, dist);
  if (cells) *cells = cnt[0] + cnt[1];  // both engines
  c->last_cells_f32 = cnt[1];
  return EAPDTW_OK;
}

uint64_t eapdtw_ctx_last_cells_f32(const eapdtw_ctx* c) { return c ? c->last_cells_f32 : 0; }
int eapdtw_ctx_spec_info(const eapdtw_ctx* c, double* deviation, uint64_t* listed,
                         uint64_t* fallbacks) {
  if (!c) return fail(EAPDTW_EINVAL, "null ctx");
  if (deviation) *deviation = c->spec_dev;
  if (listed) *listed = c->spec_listed;
  if (fallbacks) *fallbacks = g_spec_fallbacks.load();
  return EAPDTW_OK;
}

int eapdtw_nn1_dev(eapdtw_ctx* c, const double* q_dev, size_t nq, const double* db_dev, size_t nd,
                   size_t len, size_t window, uint64_t* argmin, double* dist, uint64_t* cells) {
  if (!c || !argmin || !dist) return fail(EAPDTW_EINVAL, "null argument");
  if (len == 0 || nd == 0) return fail(EAPDTW_EINVAL, "nn1: empty series");
  if (nq == 0) return EAPDTW_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  return nn1_impl(c, q_dev, nq, db_dev, nd, len, window, argmin, dist, cells);
}

int eapdtw_nn1_dev_cutoff(eapdtw_ctx* c, const double* q_dev, size_t nq, const double* db_dev,
                          size_t nd, size_t len, size_t window, const double* cutoff_dev,
                          uint64_t* argmin, double* dist, uint64_t* cells) {
  if (!c || !argmin || !dist || !cutoff_dev) return fail(EAPDTW_EINVAL, "null argument");
  if (len == 0 || nd == 0) return fail(EAPDTW_EINVAL, "nn1: empty series");
  if (nq == 0) return EAPDTW_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  return nn1_impl(c, q_dev, nq, db_dev, nd, len, window, argmin, dist, cells, cutoff_dev);
}

int eapdtw_nn1(eapdtw_ctx* c, const double* queries, size_t nq, const double* db, size_t nd,
               size_t len, size_t window, uint64_t* argmin, double* dist, uint64_t* cells) {
  if (!c || !queries || !db || !argmin || !dist) return fail(EAPDTW_EINVAL, "null argument");
  if (len == 0 || nd == 0) return fail(EAPDTW_EINVAL, "nn1: empty series");
  if (nq == 0) return EAPDTW_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(c->a.ensure(nq * len * 8));
  CUDA_TRY(c->b.ensure(nd * len * 8));
  CUDA_TRY(cudaMemcpyAsync(c->a.p, queries, nq * len * 8, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->b.p, db, nd * len * 8, cudaMemcpyHostToDevice, c->stream));
  return nn1_impl(c, c->a.as<double>(), nq, c->b.as<double>(), nd, len, window, argmin, dist, cells);
}

// ---------------------------------------------------------------------------
// The preparation kernels on their own (checking: tests compare them with the
// oracle element by element)
// ---------------------------------------------------------------------------
int eapdtw_sliding_stats(eapdtw_ctx* c, const double* ref, size_t n, size_t m, double* mean,
                         double* sd) {
  if (!c || !ref || !mean || !sd) return fail(EAPDTW_EINVAL, "null argument");
  if (n == 0 || m == 0 || m > n) return fail(EAPDTW_EINVAL, "sliding_stats: bad lengths");
  CUDA_TRY(cudaSetDevice(c->device));
  const size_t nc = n - m + 1;
  DevBuf dref, dmean, dsd;
  auto done = [&](int rc) {
    dref.release();
    dmean.release();
    dsd.release();
    return rc;
  };
  cudaError_t e = dref.ensure(n * 8);
  if (!e) e = dmean.ensure(nc * 8);
  if (!e) e = dsd.ensure(nc * 8);
  if (!e) e = cudaMemcpyAsync(dref.p, ref, n * 8, cudaMemcpyHostToDevice, c->stream);
  if (!e) e = launch_stats(dref.as<double>(), static_cast<long long>(n), static_cast<int>(m),
                           dmean.as<double>(), dsd.as<double>(), c->stream);
  if (!e) c->launches += kStatsLaunches;
  if (!e) e = cudaMemcpyAsync(mean, dmean.p, nc * 8, cudaMemcpyDeviceToHost, c->stream);
  if (!e) e = cudaMemcpyAsync(sd, dsd.p, nc * 8, cudaMemcpyDeviceToHost, c->stream);
  if (!e) e = cudaStreamSynchronize(c->stream);
  if (e) return done(fail(EAPDTW_ECUDA, std::string("sliding_stats: ") + cudaGetErrorString(e)));
  return done(EAPDTW_OK);
}

int eapdtw_sliding_envelope(eapdtw_ctx* c, const double* ref, size_t n, size_t r, double* upper,
                            double* lower) {
  if (!c || !ref || !upper || !lower) return fail(EAPDTW_EINVAL, "null argument");
  if (n == 0) return fail(EAPDTW_EINVAL, "sliding_envelope: empty series");
  if (envelope_tile(static_cast<int>(std::min<size_t>(r, 1u << 20))) < 256)
    return fail(EAPDTW_EINVAL, "sliding_envelope: radius too large for the envelope tile");
  CUDA_TRY(cudaSetDevice(c->device));
  DevBuf dref, denv;
  auto done = [&](int rc) {
    dref.release();
    denv.release();
    return rc;
  };
  std::vector<double> env(2 * n);
  cudaError_t e = dref.ensure(n * 8);
  if (!e) e = denv.ensure(2 * n * 8);
  if (!e) e = cudaMemcpyAsync(dref.p, ref, n * 8, cudaMemcpyHostToDevice, c->stream);
  if (!e) e = launch_envelope(dref.as<double>(), static_cast<long long>(n), static_cast<int>(r),
                              denv.as<double>(), c->stream);
  if (!e) ++c->launches;
  if (!e) e = cudaMemcpyAsync(env.data(), denv.p, 2 * n * 8, cudaMemcpyDeviceToHost, c->stream);
  if (!e) e = cudaStreamSynchronize(c->stream);
  if (e) return done(fail(EAPDTW_ECUDA, std::string("sliding_envelope: ") + cudaGetErrorString(e)));
  for (size_t k = 0; k < n; ++k) {
    upper[k] = env[2 * k];
    lower[k] = env[2 * k + 1];
  }
  return done(EAPDTW_OK);
}

// ---------------------------------------------------------------------------
// The reference's lower-bound API (lower_bounds.hpp:12-63) on the device
// ---------------------------------------------------------------------------
int eapdtw_compute_envelope(eapdtw_ctx* c, const double* series, size_t l, size_t window,
                            double* upper, double* lower) {
  if (!c || !upper || !lower) return fail(EAPDTW_EINVAL, "null argument");
  if (l == 0 || !series) return fail(EAPDTW_EINVAL, "compute_envelope: empty series");
  const size_t w = window == EAPDTW_UNBOUNDED_WINDOW ? l : std::min(window, l);
  CUDA_TRY(cudaSetDevice(c->device));
  const size_t scr = envelope_any_scratch_doubles(static_cast<long long>(l), static_cast<long long>(w));
  DevBuf dx, denv, dscr;
  auto done = [&](int rc) {
    dx.release();
    denv.release();
    dscr.release();
    return rc;
  };
  std::vector<double> env(2 * l);
  cudaError_t e = dx.ensure(l * 8);
  if (!e) e = denv.ensure(2 * l * 8);
  if (!e && scr) e = dscr.ensure(scr * 8);
  if (!e) e = cudaMemcpyAsync(dx.p, series, l * 8, cudaMemcpyHostToDevice, c->stream);
  if (!e) e = launch_envelope_any(dx.as<double>(), static_cast<long long>(l), static_cast<long long>(w),
                                  denv.as<double>(), dscr.as<double>(), c->stream);
  if (!e) ++c->launches;
  if (!e) e = cudaMemcpyAsync(env.data(), denv.p, 2 * l * 8, cudaMemcpyDeviceToHost, c->stream);
  if (!e) e = cudaStreamSynchronize(c->stream);
  if (e) return done(fail(EAPDTW_ECUDA, std::string("compute_envelope: ") + cudaGetErrorString(e)));
  for (size_t k = 0; k < l; ++k) {
    upper[k] = env[2 * k];
    lower[k] = env[2 * k + 1];
  }
  return done(EAPDTW_OK);
}

int eapdtw_lb_kim_fl(eapdtw_ctx* c, const double* q, const double* cs, size_t l, double* out) {
  if (!c || !out || !q || !cs) return fail(EAPDTW_EINVAL, "null argument");
  if (l < 2) return fail(EAPDTW_EINVAL, "lb_kim_fl: series must have length >= 2");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(c->a.ensure(l * 8));
  CUDA_TRY(c->b.ensure(l * 8));
  CUDA_TRY(c->out.ensure(8));
  CUDA_TRY(cudaMemcpyAsync(c->a.p, q, l * 8, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->b.p, cs, l * 8, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(launch_lb_kim_fl(c->a.as<double>(), c->b.as<double>(), static_cast<long long>(l),
                            c->out.as<double>(), c->stream));
  ++c->launches;
  CUDA_TRY(cudaMemcpyAsync(out, c->out.p, 8, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return EAPDTW_OK;
}

int eapdtw_lb_keogh(eapdtw_ctx* c, const double* upper, const double* lower, const double* series,
                    size_t l, double abandon_above, const size_t* order, double* total,
                    double* contributions, int* abandoned) {
  if (!c || !total || !abandoned) return fail(EAPDTW_EINVAL, "null argument");
  if (l > 0 && (!upper || !lower || !series)) return fail(EAPDTW_EINVAL, "null argument");
  if (order)
    for (size_t k = 0; k < l; ++k)
      if (order[k] >= l) return fail(EAPDTW_EINVAL, "lb_keogh: order index out of range");
  *total = 0.0;
  *abandoned = 0;
  if (contributions) std::fill(contributions, contributions + l, 0.0);
  if (l == 0) return EAPDTW_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  // a: upper | lower | series | contributions; b: order; out: total, abandoned
  CUDA_TRY(c->a.ensure(4 * l * 8));
  CUDA_TRY(c->b.ensure(l * 8));
  CUDA_TRY(c->out.ensure(16));
  double* d = c->a.as<double>();
  CUDA_TRY(cudaMemcpyAsync(d, upper, l * 8, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(d + l, lower, l * 8, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(d + 2 * l, series, l * 8, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemsetAsync(d + 3 * l, 0, l * 8, c->stream));
  const unsigned long long* dorder = nullptr;
  static_assert(sizeof(size_t) == sizeof(unsigned long long), "size_t is 64-bit");
  if (order) {
    CUDA_TRY(cudaMemcpyAsync(c->b.p, order, l * 8, cudaMemcpyHostToDevice, c->stream));
    dorder = c->b.as<unsigned long long>();
  }
  double* dout = c->out.as<double>();
  CUDA_TRY(launch_lb_keogh(d, d + l, d + 2 * l, static_cast<long long>(l), abandon_above, dorder,
                           dout, d + 3 * l, reinterpret_cast<int*>(dout + 1), c->stream));
  ++c->launches;
  double res[2];
  CUDA_TRY(cudaMemcpyAsync(res, dout, 16, cudaMemcpyDeviceToHost, c->stream));
  if (contributions)
    CUDA_TRY(cudaMemcpyAsync(contributions, d + 3 * l, l * 8, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  *total = res[0];
  int ab = 0;
  std::memcpy(&ab, &res[1], sizeof(int));
  *abandoned = ab;
  return EAPDTW_OK;
}

int eapdtw_cumulative_bound(eapdtw_ctx* c, const double* contributions, size_t l, double* cb) {
  if (!c || (l > 0 && (!contributions || !cb))) return fail(EAPDTW_EINVAL, "null argument");
  if (l == 0) return EAPDTW_OK;
  // lower_bounds.cpp:93-99: every contribution must be non-negative
  for (size_t k = 0; k < l; ++k)
    if (contributions[k] < 0.0) return fail(EAPDTW_EINVAL, "cumulative_bound: negative contribution");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(c->a.ensure(2 * l * 8));
  double* d = c->a.as<double>();
  CUDA_TRY(cudaMemcpyAsync(d, contributions, l * 8, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(launch_cumulative_bound(d, static_cast<long long>(l), d + l, c->stream));
  ++c->launches;
  CUDA_TRY(cudaMemcpyAsync(cb, d + l, l * 8, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return EAPDTW_OK;
}

// ---------------------------------------------------------------------------
// Host helpers
// ---------------------------------------------------------------------------
int eapdtw_running_stats_over(const double* x, size_t n, double* sum, double* sumsq) {
  if (!sum || !sumsq || (n > 0 && !x)) return fail(EAPDTW_EINVAL, "null argument");
  const HostStats st = HostStats::over(x, n);
  *sum = st.sum;
  *sumsq = st.sumsq;
  return EAPDTW_OK;
}

int eapdtw_znormalize_into(const double* src, size_t n, double sum, double sumsq, uint64_t count,
                           double* dst) {
  if (n > 0 && (!src || !dst)) return fail(EAPDTW_EINVAL, "null argument");
  HostStats st;
  st.sum = sum;
  st.sumsq = sumsq;
  st.count = static_cast<size_t>(count);
  host_znormalize(src, n, st, dst);
  return EAPDTW_OK;
}
int eapdtw_znormalize(const double* src, size_t n, double* dst) {
  if (!src || !dst || n == 0) return fail(EAPDTW_EINVAL, "znormalize: empty input");
  host_znormalize(src, n, HostStats::over(src, n), dst);
  return EAPDTW_OK;
}

int eapdtw_random_walk_uniform(size_t n, uint64_t seed, double* out) {
  if (n == 0 || !out) return fail(EAPDTW_EINVAL, "random_walk: zero length");
  std::mt19937_64 gen(seed);  // the standard fixes the mt19937_64 stream
  double x = 0.0;
  for (size_t i = 0; i < n; ++i) {
    const double u = static_cast<double>(gen() >> 11) * 0x1.0p-53;
    x += u - 0.5;
    out[i] = x;
  }
  return EAPDTW_OK;
}

int eapdtw_random_walk_normal(size_t n, uint64_t seed, double* out) {
  if (n == 0 || !out) return fail(EAPDTW_EINVAL, "random_walk: zero length");
  std::mt19937_64 gen(seed);
  auto u01 = [&]() { return (static_cast<double>(gen() >> 11) + 0.5) * 0x1.0p-53; };  // (0,1)
  double x = 0.0;
  out[0] = 0.0;
  size_t i = 1;
  while (i < n) {  // Box-Muller, both variates used
    const double u1 = u01(), u2 = u01();
    const double rad = std::sqrt(-2.0 * std::log(u1));
    const double th = 6.283185307179586 * u2;
    x += rad * std::cos(th);
    out[i++] = x;
    if (i < n) {
      x += rad * std::sin(th);
      out[i++] = x;
    }
  }
  return EAPDTW_OK;
}

static int fp_peak(eapdtw_ctx* c, int bits, double* ops) {
  if (!c || !ops) return fail(EAPDTW_EINVAL, "null argument");
  CUDA_TRY(cudaSetDevice(c->device));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  DevBuf sink;
  CUDA_TRY(sink.ensure(256 * 8));
  cudaEvent_t e0, e1;
  CUDA_TRY(cudaEventCreate(&e0));
  CUDA_TRY(cudaEventCreate(&e1));
  const int blocks = sms * 8, iters = 1 << 14;
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    CUDA_TRY(cudaEventRecord(e0, c->stream));
    if (bits == 64) CUDA_TRY(launch_fp64_probe(sink.as<double>(), blocks, iters, c->stream));
    else CUDA_TRY(launch_fp32_probe(sink.as<float>(), blocks, iters, c->stream));
    ++c->launches;
    CUDA_TRY(cudaEventRecord(e1, c->stream));
    CUDA_TRY(cudaEventSynchronize(e1));
    float ms = 0;
    CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
    best = std::min(best, ms);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  sink.release();
  *ops = static_cast<double>(blocks) * 256.0 * iters * 8.0 / (best * 1e-3);
  return EAPDTW_OK;
}

int eapdtw_fp64_peak(eapdtw_ctx* c, double* ops) { return fp_peak(c, 64, ops); }
int eapdtw_fp32_peak(eapdtw_ctx* c, double* ops) { return fp_peak(c, 32, ops); }

}  // extern "C"

// ---------------------------------------------------------------------------
// One host thread driving several devices: a context per
// device and an NCCL communicator over them (ncclCommInitAll).  NCCL is
// loaded at first use (dlopen), so the library has no hard dependency on it
// and shares the process's copy when a framework already loaded one.
// ---------------------------------------------------------------------------
#include <dlfcn.h>
#include <nccl.h>

namespace {
struct NcclApi {
  bool ok = false;
  std::string why;
  decltype(&ncclCommInitAll) commInitAll = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);  // already loaded?
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.why = std::string("NCCL not found: ") + dlerror();
      return;
    }
    api.commInitAll = reinterpret_cast<decltype(api.commInitAll)>(dlsym(h, "ncclCommInitAll"));
    api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.allReduce = reinterpret_cast<decltype(api.allReduce)>(dlsym(h, "ncclAllReduce"));
    api.groupStart = reinterpret_cast<decltype(api.groupStart)>(dlsym(h, "ncclGroupStart"));
    api.groupEnd = reinterpret_cast<decltype(api.groupEnd)>(dlsym(h, "ncclGroupEnd"));
    api.errorString = reinterpret_cast<decltype(api.errorString)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.commInitAll && api.commDestroy && api.allReduce && api.groupStart &&
             api.groupEnd && api.errorString;
    if (!api.ok) api.why = "NCCL: missing symbols";
  });
  return api;
}
}  // namespace

#define NCCL_TRY(expr)                                                                  \
  do {                                                                                  \
    const ncclResult_t r_ = (expr);                                                     \
    if (r_ != ncclSuccess)                                                              \
      return fail(EAPDTW_ENCCL, std::string(#expr) + ": " + nccl().errorString(r_));    \
  } while (0)

struct eapdtw_multi {
  std::vector<int> devs;
  std::vector<eapdtw_ctx*> ctx;
  std::vector<ncclComm_t> comm;
  std::vector<DevBuf> key;  // per device: a spare threshold key (empty shards) / NN1 keys
  std::vector<DevBuf> rec;  // per device: NN1 records
  std::vector<DevBuf> cnt;  // per device: NN1 counters
};

extern "C" {

int eapdtw_multi_create(eapdtw_multi** out, const int* devices, int n) {
  if (!out || !devices || n <= 0) return fail(EAPDTW_EINVAL, "multi_create: bad arguments");
  *out = nullptr;
  const NcclApi& api = nccl();
  if (!api.ok) return fail(EAPDTW_ENCCL, api.why);
  auto* mg = new eapdtw_multi;
  mg->devs.assign(devices, devices + n);
  for (int d = 0; d < n; ++d) {
    for (int e = 0; e < d; ++e)
      if (mg->devs[e] == mg->devs[d]) {
        eapdtw_multi_destroy(mg);
        return fail(EAPDTW_EINVAL, "multi_create: a device is listed twice");
      }
    eapdtw_ctx* c = nullptr;
    const int rc = eapdtw_ctx_create(&c, mg->devs[d]);
    if (rc) {
      const std::string msg = g_err;
      eapdtw_multi_destroy(mg);
      return fail(rc, msg);
    }
    mg->ctx.push_back(c);
  }
  mg->comm.assign(n, nullptr);
  mg->key.resize(n);
  mg->rec.resize(n);
  mg->cnt.resize(n);
  const ncclResult_t r = api.commInitAll(mg->comm.data(), n, mg->devs.data());
  if (r != ncclSuccess) {
    const std::string msg = std::string("ncclCommInitAll: ") + api.errorString(r);
    mg->comm.clear();
    eapdtw_multi_destroy(mg);
    return fail(EAPDTW_ENCCL, msg);
  }
  *out = mg;
  return EAPDTW_OK;
}

int eapdtw_multi_destroy(eapdtw_multi* mg) {
  if (!mg) return EAPDTW_OK;
  for (size_t d = 0; d < mg->comm.size(); ++d)
    if (mg->comm[d]) nccl().commDestroy(mg->comm[d]);
  for (size_t d = 0; d < mg->ctx.size(); ++d) {
    cudaSetDevice(mg->devs[d]);
    if (d < mg->key.size()) mg->key[d].release();
    if (d < mg->rec.size()) mg->rec[d].release();
    if (d < mg->cnt.size()) mg->cnt[d].release();
    eapdtw_ctx_destroy(mg->ctx[d]);
  }
  delete mg;
  return EAPDTW_OK;
}

int eapdtw_multi_device_count(const eapdtw_multi* mg) {
  return mg ? static_cast<int>(mg->devs.size()) : 0;
}

eapdtw_ctx* eapdtw_multi_context(eapdtw_multi* mg, int i) {
  return (mg && i >= 0 && i < static_cast<int>(mg->ctx.size())) ? mg->ctx[i] : nullptr;
}

// Candidate shard of device d: whole 100000-candidate segments, as even as
// possible, earlier devices taking the remainder (sharded.shard_bounds).
static void shard_bounds(size_t ncand, int world, int d, size_t& s0, size_t& s1) {
  const size_t seg = static_cast<size_t>(kStatsResetInterval);
  const size_t nseg = (ncand + seg - 1) / seg;
  const size_t base = nseg / world, extra = nseg % world;
  const size_t g0 = d * base + std::min<size_t>(d, extra);
  const size_t g1 = g0 + base + (static_cast<size_t>(d) < extra ? 1 : 0);
  s0 = std::min(ncand, g0 * seg);
  s1 = std::min(ncand, g1 * seg);
}

int eapdtw_multi_similarity_search(eapdtw_multi* mg, const double* reference, size_t n,
                                   const double* query, size_t qlen,
                                   const eapdtw_search_config* cfg, int batches,
                                   eapdtw_search_result* out) {
  if (!mg || !reference || !query || !cfg || !out) return fail(EAPDTW_EINVAL, "null argument");
  if (n == 0 || qlen == 0) return fail(EAPDTW_EINVAL, "Series: empty input");
  const size_t m = cfg->query_length == 0 ? qlen : cfg->query_length;
  if (m == 0 || m > qlen) return fail(EAPDTW_EINVAL, "similarity_search: bad query length");
  if (m > n) return fail(EAPDTW_EINVAL, "similarity_search: query longer than reference");
  const int G = static_cast<int>(mg->devs.size());
  batches = std::max(1, batches);
  const size_t ncand = n - m + 1;
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<eapdtw_search_plan*> plan(G, nullptr);
  std::vector<size_t> s0(G), s1(G);
  std::vector<uint64_t*> key(G, nullptr);
  auto cleanup = [&](int rc) {
    for (int d = 0; d < G; ++d)
      if (plan[d]) eapdtw_search_plan_destroy(plan[d]);
    return rc;
  };
  // shards: copy, validate (Series, series.hpp:24-31), plan
  for (int d = 0; d < G; ++d) {
    eapdtw_ctx* c = mg->ctx[d];
    shard_bounds(ncand, G, d, s0[d], s1[d]);
    CUDA_TRY(cudaSetDevice(mg->devs[d]));
    if (s1[d] <= s0[d]) {  // no candidates: a +inf key still joins the all-reduce
      CUDA_TRY(mg->key[d].ensure(8));
      const unsigned long long inf_key = 0x7ff0000000000000ull;
      CUDA_TRY(cudaMemcpyAsync(mg->key[d].p, &inf_key, 8, cudaMemcpyHostToDevice, c->stream));
      CUDA_TRY(cudaStreamSynchronize(c->stream));
      key[d] = mg->key[d].as<uint64_t>();
      continue;
    }
    const size_t npts = s1[d] - s0[d] + m - 1;
    CUDA_TRY(c->ref.ensure(npts * 8));
    CUDA_TRY(c->pb.flag.ensure(8));
    CUDA_TRY(cudaMemcpyAsync(c->ref.p, reference + s0[d], npts * 8, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(cudaMemsetAsync(c->pb.flag.p, 0, 8, c->stream));
    CUDA_TRY(launch_check_finite(c->ref.as<double>(), static_cast<long long>(npts),
                                 c->pb.flag.as<unsigned long long>(), c->stream));
    ++c->launches;
    const int rc = eapdtw_search_plan_create(c, c->ref.as<double>(), npts, query, qlen, cfg,
                                             s0[d], &plan[d]);
    if (rc) return cleanup(rc);
    key[d] = eapdtw_search_plan_ub_key(plan[d]);
  }
  auto allreduce_keys = [&]() -> int {
    NCCL_TRY(nccl().groupStart());
    for (int d = 0; d < G; ++d)
      NCCL_TRY(nccl().allReduce(key[d], key[d], 1, ncclUint64, ncclMin, mg->comm[d],
                                mg->ctx[d]->stream));
    NCCL_TRY(nccl().groupEnd());
    return EAPDTW_OK;
  };
  int rc;
  for (int d = 0; d < G; ++d)
    if (plan[d] && (rc = eapdtw_search_plan_prepare(plan[d]))) return cleanup(rc);
  if (G > 1 && (rc = allreduce_keys())) return cleanup(rc);  // the warm starts' best
  for (int b = 0; b < batches; ++b) {
    for (int d = 0; d < G; ++d) {
      if (!plan[d]) continue;
      const size_t nc = s1[d] - s0[d];
      const size_t b0 = nc * b / batches, b1 = nc * (b + 1) / batches;
      if ((rc = eapdtw_search_plan_run(plan[d], b0, b1))) return cleanup(rc);
    }
    if (G > 1 && (rc = allreduce_keys())) return cleanup(rc);
  }
  // (distance, lowest global index) over the shards; counters summed
  std::memset(out, 0, sizeof(*out));
  out->distance_sq = kInf;
  for (int d = 0; d < G; ++d) {
    if (!plan[d]) continue;
    eapdtw_search_result r{};
    if ((rc = eapdtw_search_plan_result(plan[d], &r))) return cleanup(rc);
    unsigned long long bad = 0;
    CUDA_TRY(cudaMemcpy(&bad, mg->ctx[d]->pb.flag.p, 8, cudaMemcpyDeviceToHost));
    if (bad) return cleanup(fail(EAPDTW_EINVAL, "Series: non-finite sample in the reference"));
    if (r.found && (!out->found || r.distance_sq < out->distance_sq ||
                    (r.distance_sq == out->distance_sq && r.location < out->location))) {
      out->found = 1;
      out->distance_sq = r.distance_sq;
      out->location = r.location;
    }
    out->candidates_total += r.candidates_total;
    out->pruned_kim += r.pruned_kim;
    out->pruned_keogh_eq += r.pruned_keogh_eq;
    out->pruned_keogh_ec += r.pruned_keogh_ec;
    out->dtw_calls += r.dtw_calls;
    out->dtw_abandoned += r.dtw_abandoned;
    out->dp_cells_evaluated += r.dp_cells_evaluated;
    out->screen_cells_evaluated += r.screen_cells_evaluated;
  }
  if (!out->found) out->location = 0;
  out->elapsed_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return cleanup(EAPDTW_OK);
}

int eapdtw_multi_nn1(eapdtw_multi* mg, const double* queries, size_t nq, const double* db,
                     size_t nd, size_t len, size_t window, int batches, uint64_t* argmin,
                     double* dist, uint64_t* cells) {
  if (!mg || !queries || !db || !argmin || !dist) return fail(EAPDTW_EINVAL, "null argument");
  if (len == 0 || nd == 0) return fail(EAPDTW_EINVAL, "nn1: empty series");
  if (nq == 0) return EAPDTW_OK;
  const int G = static_cast<int>(mg->devs.size());
  batches = std::max(1, batches);
  std::vector<size_t> d0(G), d1(G);
  for (int d = 0; d < G; ++d) {  // contiguous rows, earlier devices take the remainder
    const size_t base = nd / G, extra = nd % G;
    d0[d] = d * base + std::min<size_t>(d, extra);
    d1[d] = d0[d] + base + (static_cast<size_t>(d) < extra ? 1 : 0);
  }
  for (int d = 0; d < G; ++d) {
    eapdtw_ctx* c = mg->ctx[d];
    cudaStream_t s = c->stream;
    CUDA_TRY(cudaSetDevice(mg->devs[d]));
    CUDA_TRY(c->a.ensure(nq * len * 8));
    CUDA_TRY(c->b.ensure(std::max<size_t>(1, d1[d] - d0[d]) * len * 8));
    CUDA_TRY(mg->key[d].ensure(nq * 8));
    CUDA_TRY(mg->rec[d].ensure(nq * sizeof(BestRecord)));
    CUDA_TRY(mg->cnt[d].ensure(24));
    CUDA_TRY(cudaMemcpyAsync(c->a.p, queries, nq * len * 8, cudaMemcpyHostToDevice, s));
    if (d1[d] > d0[d])
      CUDA_TRY(cudaMemcpyAsync(c->b.p, db + d0[d] * len, (d1[d] - d0[d]) * len * 8,
                               cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemsetAsync(mg->cnt[d].p, 0, 24, s));
    CUDA_TRY(launch_init_best(mg->rec[d].as<BestRecord>(), mg->key[d].as<unsigned long long>(),
                              static_cast<long long>(nq), s));
    ++c->launches;
  }
  for (int b = 0; b < batches; ++b) {
    for (int d = 0; d < G; ++d) {
      const size_t rows = d1[d] - d0[d];
      const size_t b0 = rows * b / batches, b1 = rows * (b + 1) / batches;
      if (b1 <= b0) continue;
      CUDA_TRY(cudaSetDevice(mg->devs[d]));
      const int rc = nn1_launch(mg->ctx[d], mg->ctx[d]->a.as<double>(), nq,
                                mg->ctx[d]->b.as<double>() + b0 * len, b1 - b0, len, window,
                                mg->key[d].as<unsigned long long>(), mg->rec[d].as<BestRecord>(),
                                mg->cnt[d].as<unsigned long long>(),
                                static_cast<long long>(d0[d] + b0));
      if (rc) return rc;
    }
    if (G > 1) {  // every device continues from the per-query minimum cutoff
      NCCL_TRY(nccl().groupStart());
      for (int d = 0; d < G; ++d)
        NCCL_TRY(nccl().allReduce(mg->key[d].p, mg->key[d].p, nq, ncclUint64, ncclMin,
                                  mg->comm[d], mg->ctx[d]->stream));
      NCCL_TRY(nccl().groupEnd());
    }
  }
  // per query: (distance, lowest global index) over the devices' records
  std::vector<BestRecord> best(nq, BestRecord{kInf, ~0ull}), rec(nq);
  uint64_t total_cells = 0;
  for (int d = 0; d < G; ++d) {
    unsigned long long cnt[3];
    CUDA_TRY(cudaSetDevice(mg->devs[d]));
    CUDA_TRY(cudaMemcpyAsync(rec.data(), mg->rec[d].p, nq * sizeof(BestRecord),
                             cudaMemcpyDeviceToHost, mg->ctx[d]->stream));
    CUDA_TRY(cudaMemcpyAsync(cnt, mg->cnt[d].p, 24, cudaMemcpyDeviceToHost, mg->ctx[d]->stream));
    CUDA_TRY(cudaStreamSynchronize(mg->ctx[d]->stream));
    total_cells += cnt[0] + cnt[1];
    for (size_t i = 0; i < nq; ++i)
      if (rec[i].d < best[i].d || (rec[i].d == best[i].d && rec[i].idx < best[i].idx))
        best[i] = rec[i];
  }
  nn1_unpack(best, argmin, dist);
  if (cells) *cells = total_cells;
  return EAPDTW_OK;
}

}  // extern "C"
