/*
 * eapdtw_b200.h -- C ABI of the B200 (sm_100a) EAPrunedDTW subsequence-search
 * hot path.  Plain pointers and sizes only; no exceptions, no torch types.
 *
 * Each entry point replaces one reference interface (paths relative to
 * /root/reference/proj).  The reference C++ signatures are re-exposed on top
 * of this ABI by include/eapdtw_b200.hpp; INTEGRATION.md shows the binding.
 *
 * Conventions:
 *   - status codes: EAPDTW_OK, EAPDTW_EINVAL for exactly the conditions where
 *     the reference throws std::invalid_argument, EAPDTW_ECUDA for a CUDA
 *     failure (message via eapdtw_last_error(), thread-local);
 *   - abandonment returns +inf, the reference's PRUNED (series.hpp:16);
 *   - EAPDTW_UNBOUNDED_WINDOW == Band::unbounded_window (dtw.hpp:17);
 *   - host pointers are copied; *_dev variants take device pointers;
 *   - one host thread per context; calls on a context are serialised on its
 *     stream.  There is no CPU fallback: without a GPU every compute call
 *     returns EAPDTW_ECUDA.
 */
#ifndef EAPDTW_B200_H
#define EAPDTW_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EAPDTW_OK 0
#define EAPDTW_EINVAL 1
#define EAPDTW_ECUDA 2
#define EAPDTW_ENOMEM 3
#define EAPDTW_ENCCL 4
#define EAPDTW_UNBOUNDED_WINDOW ((size_t)-1)

/* Algo (search.hpp:56) */
#define EAPDTW_ALGO_FULL 0
#define EAPDTW_ALGO_LEFT_PRUNE 1
#define EAPDTW_ALGO_EA_PRUNED 2

typedef struct eapdtw_ctx eapdtw_ctx;
typedef struct eapdtw_search_plan eapdtw_search_plan;

/* SearchConfig (search.hpp:60-66) */
typedef struct {
  size_t query_length; /* 0: the query's full length */
  double window_ratio; /* window_cells = floor(window_ratio * m) (search.cpp:18-21) */
  int32_t algorithm;   /* EAPDTW_ALGO_* */
  int32_t use_lower_bounds;
  int32_t tighten_ub;  /* per-row cumulative-bound thresholds (search.cpp:101-113); results unchanged */
  int32_t reserved_;
} eapdtw_search_config;

/* SearchResult = BestSoFar + SearchReport (search.hpp:50-82), flattened. */
typedef struct {
  uint64_t location;
  double distance_sq;
  int32_t found;
  int32_t pad_;
  uint64_t candidates_total, pruned_kim, pruned_keogh_eq, pruned_keogh_ec, dtw_calls,
      dtw_abandoned, dp_cells_evaluated; /* DP cells evaluated by every engine (dtw.cpp:28-33) */
  double elapsed_seconds;
  uint64_t screen_cells_evaluated; /* ... of which the FP32 screening pass (the exact DP: the rest) */
} eapdtw_search_result;

/* --- errors / context ---------------------------------------------------- */
const char* eapdtw_last_error(void);
int eapdtw_version(void);
int eapdtw_device_count(void);
int eapdtw_ctx_create(eapdtw_ctx** out, int device);
int eapdtw_ctx_destroy(eapdtw_ctx* ctx);
/* Run on an external stream (e.g. torch.cuda.current_stream().cuda_stream).
 * NULL: the context's own (non-blocking) stream.  The legacy default stream
 * (torch's default stream reports handle 0) must be passed as
 * EAPDTW_STREAM_LEGACY (cudaStreamLegacy), not NULL. */
#define EAPDTW_STREAM_LEGACY ((void*)0x1)
int eapdtw_ctx_set_stream(eapdtw_ctx* ctx, void* cuda_stream);
/* Engine options (no environment variables are read).  Names and defaults:
 *   ad_k -1 (exact-engine window: -1 auto, 0 strip, 1/3/5 anti-diagonal 64K),
 *   screen_rows 2, f32 1 (FP32 screening engine), streamed -1 (auto/0/1),
 *   stream_split 3, rank_stride 16, rank_k 16384, rank_waves 1, rank_ub 1,
 *   rank_ub_w 4, rank_ub_k 16, rank_cascade 1, coarse_stride 0, probe 2048,
 *   probe_force 0, tighten 1, cb_strip 1, warps 0, nn1_splits 0, nn1_warm 1,
 *   series_cache 1, probe_strips 1 (FP32 screen: strips probed in each direction),
 *   producers 0, probe_warm 0, prep_overlap 1 (envelope beside the stats chain),
 *   warm_f32 1, cb_ec_strip 2 (first strip whose row thresholds use the EC suffix),
 *   probe_excess 1 (the dropped probe's frontier minimum joins the other's bound),
 *   spec_stats -1 (speculative prefix-sum statistics beside the exact chain of
 *   search.cpp:156-168: -1 auto, 0, 1), spec_eps 8000 (their assumed deviation,
 *   in 1e-9), rank_min 32000000 (smallest candidate range the rank pass runs on),
 *   lb_blocks 1 (Keogh visiting order by parts: the first 256 positions, then the rest).
 * Every value returns the reference's answer; the defaults are the fastest
 * measured.  EAPDTW_EINVAL for an unknown name or out-of-range value. */
int eapdtw_ctx_set_option(eapdtw_ctx* ctx, const char* name, int64_t value);
int eapdtw_ctx_get_option(const eapdtw_ctx* ctx, const char* name, int64_t* value);
int eapdtw_ctx_synchronize(eapdtw_ctx* ctx);
/* Number of kernels this context has launched (gpu_launches accounting). */
uint64_t eapdtw_ctx_launches(const eapdtw_ctx* ctx);
/* Kernels launched by every context of this process so far. */
uint64_t eapdtw_total_launches(void);
/* Cells of the last eapdtw_nn1(_dev) call evaluated by the FP32 screening
 * engine (included in that call's *cells total). */
uint64_t eapdtw_ctx_last_cells_f32(const eapdtw_ctx* ctx);
/* Speculative statistics (option spec_stats; search.cpp:156-168 is the exact
 * chain they run beside): the last search's measured deviation of the
 * prefix-sum statistics from the chain's (max |delta| / stddev; < 0: the last
 * search did not speculate), the candidates it re-evaluated exactly, and the
 * number of searches this process redid on the exact statistics because the
 * deviation exceeded option spec_eps. */
int eapdtw_ctx_spec_info(const eapdtw_ctx* ctx, double* deviation, uint64_t* listed,
                         uint64_t* fallbacks);

/* --- DTW kernels, one pair (dtw.hpp:69-99) ------------------------------- *
 * ea_pruned_dtw_windowed(a, b, Band{window}, ub, cumulative_bound)  dtw.hpp:93-99
 * dtw_windowed(a, b, Band{window})                                  dtw.hpp:72-74
 * ea_pruned_dtw(a, b, ub)      == window EAPDTW_UNBOUNDED_WINDOW    dtw.hpp:85-87
 * cb may be NULL (cb_len 0).  cells (nullable) receives the evaluated cells. */
int eapdtw_ea_pruned_dtw_windowed(eapdtw_ctx* ctx, const double* a, size_t la, const double* b,
                                  size_t lb, size_t window, double ub, const double* cb,
                                  size_t cb_len, double* out, uint64_t* cells);
int eapdtw_dtw_windowed(eapdtw_ctx* ctx, const double* a, size_t la, const double* b, size_t lb,
                        size_t window, double* out, uint64_t* cells);
/* dtw_left_prune_windowed(a, b, Band{window}, ub)                 dtw.hpp:76-83
 * (left_prune_scan, dtw.cpp:130-182: pruning from the left only) */
int eapdtw_dtw_left_prune_windowed(eapdtw_ctx* ctx, const double* a, size_t la, const double* b,
                                   size_t lb, size_t window, double ub, double* out,
                                   uint64_t* cells);

/* --- per-cell trace of one DTW (KernelTrace, dtw.hpp:42-57) ---------------- *
 * algo 0 dtw_full / dtw_windowed, 1 dtw_left_prune(_windowed), 2 ea_pruned_dtw
 * (dtw.hpp:69-99, no cumulative bound), computed on the device by one thread
 * in the reference's event order: kind 0 cell (row, col, value), 1 discard
 * point, 2 pruning point, 3 abandon (at the last evaluated cell).  Rows and
 * columns are 1-based matrix coordinates (row 0 / col 0 are the borders).
 * At most cap events are stored; *n_events is the full count (retry with a
 * larger buffer if it exceeds cap).  A debugging path (the CLI's `trace`),
 * not a throughput path. */
typedef struct {
  uint32_t kind;
  uint32_t pad_;
  uint64_t row, col;
  double value;
} eapdtw_trace_event;
int eapdtw_trace(eapdtw_ctx* ctx, int algo, const double* a, size_t la, const double* b,
                 size_t lb, size_t window, double ub, eapdtw_trace_event* events, size_t cap,
                 size_t* n_events, uint64_t* cells, double* out);

/* --- batched pairwise (cfg1): npairs pairs of equal length len --------------
 * out[p] = ea_pruned_dtw_windowed(a_p, b_p, Band{window}, ub[p]); ub NULL = +inf.
 * prune 0 gives dtw_windowed (no abandoning). */
int eapdtw_pairwise(eapdtw_ctx* ctx, const double* a, const double* b, size_t npairs, size_t len,
                    size_t window, const double* ub, int prune, double* out, uint64_t* cells);
int eapdtw_pairwise_dev(eapdtw_ctx* ctx, const double* a_dev, const double* b_dev, size_t npairs,
                        size_t len, size_t window, const double* ub_dev, int prune,
                        double* out_dev, uint64_t* cells);

/* --- subsequence search (similarity_search, search.hpp:118-119) ------------ */
int eapdtw_similarity_search(eapdtw_ctx* ctx, const double* reference, size_t n,
                             const double* query, size_t qlen, const eapdtw_search_config* cfg,
                             eapdtw_search_result* out);
int eapdtw_similarity_search_dev(eapdtw_ctx* ctx, const double* reference_dev, size_t n,
                                 const double* query, size_t qlen,
                                 const eapdtw_search_config* cfg, eapdtw_search_result* out);

/* Device-resident reference: one upload + one Series validation
 * (series.hpp:24-31) shared by many searches -- the reference CLI's
 * query-length x window-ratio grid (run_bench, eapdtw_cli.cpp:110-142, which
 * calls similarity_search once per grid point on the same reference) and
 * multi-query drivers.  The handle owns its HBM copy until series_free, and
 * caches the sliding statistics (mean, sd) of the last query length searched:
 * they depend on the reference and m only (search.cpp:156-168), so searches
 * that differ in window, algorithm or query content reuse them.  Several
 * contexts (one per host thread) may search one series concurrently; each
 * keeps its own cache entry. */
typedef struct eapdtw_series eapdtw_series;
int eapdtw_series_upload(eapdtw_ctx* ctx, const double* host, size_t n, eapdtw_series** out);
const double* eapdtw_series_device_ptr(const eapdtw_series* s);
size_t eapdtw_series_length(const eapdtw_series* s);
int eapdtw_series_free(eapdtw_series* s);
int eapdtw_similarity_search_series(eapdtw_ctx* ctx, eapdtw_series* reference,
                                    const double* query, size_t qlen,
                                    const eapdtw_search_config* cfg, eapdtw_search_result* out);

/* Stepped search over one shard, for multi-GPU drivers.  The shard holds
 * reference[global_offset : global_offset + n) (candidates plus an (m-1)-point
 * halo); global_offset must be a multiple of 100000 (the stats reset
 * interval, search.cpp:16) so the shard reproduces the unsharded chain.
 * run() may be called for consecutive candidate ranges; between calls a
 * driver may lower the threshold key (all-reduce MIN across ranks) through
 * the device pointer returned by ub_key(). */
int eapdtw_search_plan_create(eapdtw_ctx* ctx, const double* reference_dev, size_t n,
                              const double* query, size_t qlen, const eapdtw_search_config* cfg,
                              uint64_t global_offset, eapdtw_search_plan** out);
/* Restart the search on the same inputs (best record, threshold, counters). */
int eapdtw_search_plan_reset(eapdtw_search_plan* plan);
/* Use a caller-owned 8-byte device threshold key (e.g. a torch int64 tensor
 * that is all-reduced with MIN across ranks); NULL restores the plan's own.
 * Implies reset(). */
int eapdtw_search_plan_set_ub_key(eapdtw_search_plan* plan, uint64_t* dev_key);
int eapdtw_search_plan_prepare(eapdtw_search_plan* plan); /* stats, envelope, probe */
size_t eapdtw_search_plan_candidates(const eapdtw_search_plan* plan);
int eapdtw_search_plan_run(eapdtw_search_plan* plan, size_t begin, size_t end);
uint64_t* eapdtw_search_plan_ub_key(eapdtw_search_plan* plan);
/* Synchronises; location is global (offset added). */
int eapdtw_search_plan_result(eapdtw_search_plan* plan, eapdtw_search_result* out);
/* Device time in ms of the last prepare/run, per phase: [stats, envelope, probe, sweep]. */
int eapdtw_search_plan_timings(eapdtw_search_plan* plan, float* ms4);
/* Raw device counters of the last sweep (10 entries): [kim, keogh_eq, keogh_ec,
 * dtw_calls, dtw_abandoned, cells (exact FP64 engine), candidates,
 * engine_overflows, screened, cells_f32 (FP32 screening engine)]. */
int eapdtw_search_plan_counters(eapdtw_search_plan* plan, uint64_t* out10);
int eapdtw_search_plan_destroy(eapdtw_search_plan* plan);

/* --- batched NN1 (cfg5): per query, argmin over the database ------------- *
 * Each query keeps a running cutoff: d_k = ea_pruned_dtw_windowed(db_k, q,
 * Band{window}, bsf); strict < keeps the lowest index. */
int eapdtw_nn1(eapdtw_ctx* ctx, const double* queries, size_t nq, const double* db, size_t nd,
               size_t len, size_t window, uint64_t* argmin, double* dist, uint64_t* cells);
int eapdtw_nn1_dev(eapdtw_ctx* ctx, const double* queries_dev, size_t nq, const double* db_dev,
                   size_t nd, size_t len, size_t window, uint64_t* argmin, double* dist,
                   uint64_t* cells);

/* One shard / batch of a multi-GPU NN1: the same search
 * starting from a per-query cutoff (cutoff_dev: nq non-negative doubles on the
 * device, +inf = none), e.g. the all-reduced MIN of every rank's best so far.
 * A database row is reported iff its distance is <= the cutoff (ties with the
 * cutoff are kept, so a lexicographic (distance, global index) merge across
 * shards keeps the lowest index); a query with no such row gets argmin 0 and
 * dist +inf.  argmin is local to db_dev. */
int eapdtw_nn1_dev_cutoff(eapdtw_ctx* ctx, const double* queries_dev, size_t nq,
                          const double* db_dev, size_t nd, size_t len, size_t window,
                          const double* cutoff_dev, uint64_t* argmin, double* dist,
                          uint64_t* cells);

/* --- one host thread, several devices -------------------------
 * A context per device and an NCCL communicator over them (ncclCommInitAll;
 * NCCL is loaded at first use).  EAPDTW_ENCCL for an NCCL failure.
 *   multi_similarity_search: the reference split into 100000-aligned
 *     candidate shards (the stats reset interval, search.cpp:16), each with its
 *     (m-1)-point halo, one per device; the threshold keys all-reduced (MIN)
 *     after the warm start and after each of `batches` candidate batches; the
 *     result the (distance, lowest global index) minimum, counters summed.
 *   multi_nn1: the database split into contiguous row ranges, the queries on
 *     every device; per-query cutoff keys all-reduced (MIN) after each of
 *     `batches` batches; per query the (distance, lowest global index) min. */
typedef struct eapdtw_multi eapdtw_multi;
int eapdtw_multi_create(eapdtw_multi** out, const int* devices, int n);
int eapdtw_multi_destroy(eapdtw_multi* mg);
int eapdtw_multi_device_count(const eapdtw_multi* mg);
/* The context of the i-th device (options, streams); owned by mg. */
eapdtw_ctx* eapdtw_multi_context(eapdtw_multi* mg, int i);
int eapdtw_multi_similarity_search(eapdtw_multi* mg, const double* reference, size_t n,
                                   const double* query, size_t qlen,
                                   const eapdtw_search_config* cfg, int batches,
                                   eapdtw_search_result* out);
int eapdtw_multi_nn1(eapdtw_multi* mg, const double* queries, size_t nq, const double* db,
                     size_t nd, size_t len, size_t window, int batches, uint64_t* argmin,
                     double* dist, uint64_t* cells);

/* --- the search's preparation kernels, exposed for checking -------------------
 * Sliding statistics of every length-m window of ref (the RunningStats chain of
 * similarity_search, search.cpp:156-168, reset every 100000 slides): mean[s]
 * and sd[s] for s in [0, n-m+1), computed by the search's own stats kernel.
 * Raw sliding envelope of radius r (compute_envelope's window,
 * lower_bounds.cpp:9-49, clamped to [0, n)): upper[p] = max(ref[p-r .. p+r]),
 * lower[p] = min(...), computed by the search's envelope kernel.  Host
 * pointers in and out; EAPDTW_EINVAL when the envelope tile cannot hold 2r+1. */
int eapdtw_sliding_stats(eapdtw_ctx* ctx, const double* ref, size_t n, size_t m, double* mean,
                         double* sd);
int eapdtw_sliding_envelope(eapdtw_ctx* ctx, const double* ref, size_t n, size_t r, double* upper,
                            double* lower);

/* --- the reference's lower-bound API (lower_bounds.hpp:12-63), computed on the
 * device with the reference's arithmetic and order (bit-identical results).
 * Host pointers.  EAPDTW_EINVAL exactly where the reference throws.
 *   compute_envelope(series, Band{window})        lower_bounds.hpp:25 / .cpp:9-49
 *     window EAPDTW_UNBOUNDED_WINDOW = the whole series
 *   lb_kim_fl(q, c)                               lower_bounds.hpp:33 / .cpp:51-55
 *   lb_keogh(env, series, abandon_above, order)   lower_bounds.hpp:52-54 / .cpp:57-88
 *     order may be NULL (natural order); contributions (nullable) receives l
 *     values in natural index order, 0 where not visited
 *   cumulative_bound(contributions)               lower_bounds.hpp:63 / .cpp:90-103 */
int eapdtw_compute_envelope(eapdtw_ctx* ctx, const double* series, size_t l, size_t window,
                            double* upper, double* lower);
int eapdtw_lb_kim_fl(eapdtw_ctx* ctx, const double* q, const double* c, size_t l, double* out);
int eapdtw_lb_keogh(eapdtw_ctx* ctx, const double* upper, const double* lower, const double* series,
                    size_t l, double abandon_above, const size_t* order, double* total,
                    double* contributions, int* abandoned);
int eapdtw_cumulative_bound(eapdtw_ctx* ctx, const double* contributions, size_t l, double* cb);

/* --- host-side helpers (bit-identical to the reference) -------------------- */
/* RunningStats::over (search.cpp:25-33): sum and sum of squares of x[0, n) */
int eapdtw_running_stats_over(const double* x, size_t n, double* sum, double* sumsq);
/* znormalize_into (search.cpp:37-46) with given RunningStats (sum, sumsq, count) */
int eapdtw_znormalize_into(const double* src, size_t n, double sum, double sumsq, uint64_t count,
                           double* dst);
/* RunningStats::over + znormalize_into (search.cpp:25-46) */
int eapdtw_znormalize(const double* src, size_t n, double* dst);
/* random_walk (io.cpp:124-137): mt19937_64, uniform steps in [-0.5, 0.5) */
int eapdtw_random_walk_uniform(size_t n, uint64_t seed, double* out);
/* Benchmark data: x0 = 0, x[i+1] = x[i] + N(0,1) (mt19937_64 + Box-Muller) */
int eapdtw_random_walk_normal(size_t n, uint64_t seed, double* out);

/* --- measurement ------------------------------------------------------------ */
/* Measured FP64 (DADD) issue rate of this device in ops/s (the DTW roofline). */
int eapdtw_fp64_peak(eapdtw_ctx* ctx, double* ops_per_s);
/* Measured FP32 add issue rate (ops/s): the roofline of the FP32 screening engine. */
int eapdtw_fp32_peak(eapdtw_ctx* ctx, double* ops_per_s);

#ifdef __cplusplus
}
#endif
#endif /* EAPDTW_B200_H */
