// kernels.cuh -- launch interface of the sm_100a kernels (host side of kernels.cu).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "dtw_warp.cuh"
#include "dtw_f32.cuh"

namespace eapdtw_b200 {

constexpr long long kStatsResetInterval = 100000;  // search.cpp:16
constexpr double kMinStddev = 1e-12;               // search.cpp:13
constexpr int kScreenSlots = 24;                   // phase-A window (band offsets)
constexpr int kStack = 64;                         // per-warp tier stack capacity
#ifndef EAPDTW_LB_GROUP
#define EAPDTW_LB_GROUP 8
#endif
constexpr int kLbGroup = EAPDTW_LB_GROUP;          // Keogh positions per abandon vote
#ifndef EAPDTW_KIM_LAYERS
#define EAPDTW_KIM_LAYERS 3
#endif
constexpr int kKimLayers = EAPDTW_KIM_LAYERS;     // LB_Kim points per end (short queries)
constexpr int kKimLayersLong = 8;                  // ... for m >= kKimLongFrom
constexpr int kKimLongFrom = 768;
#ifndef EAPDTW_SUPER_CHUNK
#define EAPDTW_SUPER_CHUNK 4
#endif
constexpr int kSuperChunk = EAPDTW_SUPER_CHUNK;    // LB chunks (of 32 candidates) per claim
constexpr int kStageExtra = 48;                    // extra doubles per warp buffer: EQ staging span (>= 2 super-chunks... 128 candidates + 2)
constexpr int kLbHead = 256;                       // first leg of the Keogh tiers (positions of order[])
// A, A2, B, B2, C indices; B, B2 EQ totals; C (EQ, EC) totals; A2, B2 partial sums
// + the FP32 screen's probe state (two F32Strip, two cumulative-bound prefixes)
constexpr int kProbeStateBytes = 128;
constexpr int kStackBytesPerWarp = kStack * (5 * 4 + 2 * 4 + 8 + 2 * 8) + kProbeStateBytes;

// Tier counters accumulated on the device (SearchReport, search.hpp:68-77).
enum Counter : int {
  kCntKim = 0,
  kCntKeoghEq,
  kCntKeoghEc,
  kCntDtwCalls,
  kCntDtwAbandoned,
  kCntCells,
  kCntCandidates,
  kCntOverflows,
  kCntScreened,
  kCntCellsF32,  // cells evaluated by the FP32 screening engine
  kNumCounters,
  // phase clocks (builds with -DEAPDTW_PHASE_CLOCKS only): warp-cycles per phase
  kClkDtw = kNumCounters,
  kClkEq,
  kClkEc,
  kClkScreen,
  kClkKim,
  kClkWait,
  kStageHit,
  kStageMiss,
  kClkTotal,
  kNumCountersExt
};

struct SearchParams {
  const double* ref;     // shard reference, n points
  const double* mean;    // per candidate (ncand)
  const double* sd;      // per candidate (ncand)
  const double2* env;    // raw sliding (max, min) of ref, radius env_r (nullptr: no EC tier)
  const double* q;       // normalised query, 1-based: q[1..m] (q[0] unused)
  const double2* qul;    // query envelope (upper, lower) per position, 0-based
  const double2* qperm;  // the same in visiting order: qperm[k] = qul[order[k]]
  const float2* qperm32; // ... as floats rounded outward (upper up, lower down), for FP32 Keogh terms
  double lb_f32_e;       // FP32 Keogh terms: bound on a term's distance error (kernels.cu: lb_f32_excess)
  const int* order;      // Keogh visiting order (search.cpp:143-149)
  int lb_block_order;    // order[] lists the first kLbHead positions first (partial EQ staging)
  long long ncand;
  long long begin, end, stride;  // candidates begin, begin+stride, ... < end
  long long chunk_span;          // cascade: chunk c starts at begin + c*chunk_span (0: 32*stride)
  int m, w;                      // query length, effective half window
  int use_lb;                    // Kim -> Keogh EQ -> Keogh EC cascade
  int tighten;                   // per-row thresholds from the Keogh cumulative bound (search.cpp:101-105)
  int cb_strip;                  // first strip (1-based) that uses them
  int probe_excess;              // the dropped probe's frontier minimum joins the continuing pass's bound
  int cb_ec_strip;               // first strip whose thresholds also use the EC suffix (before: EQ alone)
  int prune;                     // 0: Algo::full (no pruning), 1: pruned DTW
  double guard_rel, guard_abs;   // LB soundness guard
  double guard_sqrt;             // ... and its reciprocal-normalisation term (lb_guard)
  double qmax;                   // max |q| (cumulative-bound guard)
  double kim_f32_guard;          // FP32 LB_Kim layers: what their rounding can add (kernels.cu)
  unsigned long long* ub_key;    // running threshold key (order-preserving bits)
  BestRecord* best;              // exact (d, lowest index) record
  unsigned long long* work;      // chunk counter (zeroed before launch)
  long long* queue;              // survivor queue, -1 filled before launch
  float2* qtot;                  // per queue slot: LB_Keogh EQ / EC totals (rounded down)
  unsigned long long* qhead;     // next slot to consume (zeroed before launch)
  unsigned long long* qtail;     // next slot to fill (zeroed before launch)
  unsigned long long* chunks_done;  // LB chunks published (zeroed before launch)
  long long direct_chunk;        // candidates per claim without the cascade
  int ad_k;                      // anti-diagonal engine window 64*ad_k (0: strip engine only)
  int direct;                    // 1: every candidate is a DTW task (the probe)
  int screen_rows;               // phase-A lane screen depth (0: off)
  int probe_strips;              // FP32 strip screen: strips probed in each direction (0: forward only)
  int producer_smsp;             // > 0: SMSP-0 warps run the LB tiers, taking DTW tasks only past this backlog
  int use_f32;                   // FP32 screening engine ahead of the exact FP64 one
  float f32_a, f32_b, f32_cmax;  // its threshold guard (dtw_f32.cuh) and row-value bound
  float f32_ia;                  // <= 1 / f32_a (the guard's inverse without a division)
  unsigned long long* counters;  // kNumCounters
  long long index_offset;        // shard start in the global reference
  // list mode (rank pass): chunk c covers list[32c .. 32c+31] (candidate
  // indices in [begin, end)); the count is read on the device
  const long long* list;
  const unsigned long long* nlist;
  long long list_cap;            // entries past it were not written
  int ub_only;                   // results tighten the threshold only (no record update)
  // speculative statistics (capi.cu): mean / sd are the prefix-sum ones, the
  // guards are widened, completed candidates are listed for the exact pass
  int approx;
  double cb_eps;                 // extra cumulative-bound guard per sqrt(m T) (0 unless approx)
  long long* vlist;              // completed candidates (plan-relative indices)
  unsigned long long* vcount;    // entries claimed (may exceed vcap: overflow)
  long long vcap;
  double* gscratch;              // non-null: the per-warp buffers live here (global memory),
                                 // warp_buf_doubles(m, ad_k) each, for queries whose buffers
                                 // exceed shared memory
};
// Resident 8-warp search blocks per SM the kernel's register budget allows.
int search_blocks_per_sm_by_regs();

struct PairParams {
  const double* rows;  // npairs x lr (row-major, pair p at p*row_stride)
  const double* cols;  // npairs x lc
  long long row_stride, col_stride;
  int lr, lc, w;
  const double* ub;  // per pair (nullptr: +inf)
  const double* cb;  // per pair cumulative bound, lr each (nullptr: none)
  int prune;         // 0: full DP (dtw_windowed), 1: pruned
  int ad_k;          // anti-diagonal engine window 64*ad_k (0: strip engine only)
  double* out;
  unsigned long long* cells;  // one counter
  long long npairs;
  double* gscratch;  // non-null: each warp's (cols, row) buffers in global memory (long series)
};
// Global scratch doubles launch_pairwise needs for p (0: shared memory suffices).
size_t pairwise_gscratch_doubles(const PairParams& p);

struct Nn1Params {
  const double* queries;  // nq x len
  const double* db;       // nd x len
  long long nq, nd;
  int len, w;
  int splits;                     // blocks per query
  int ad_k;                       // anti-diagonal engine window 64*ad_k (0: strip engine only)
  unsigned long long* ub_keys;    // nq
  BestRecord* best;               // nq
  unsigned long long* cells;      // two counters: exact FP64 engine, FP32 screen
  unsigned long long* dtw_calls;  // one counter
  int use_f32;                    // FP32 screen for queries with max |q| <= f32_cmax
  float f32_a, f32_b, f32_cmax;   // guard built with qmax = cmax (dtw_f32.cuh)
  double guard_rel, guard_abs;    // layered LB_Kim guard (summation order)
  int warm;                       // per-warp warm start (best layered-Kim row first)
  int probe_strips;               // FP32 screen: strips probed in each direction (0: forward only)
  long long index_offset;         // recorded index = local row + index_offset (database shards)
};

// Each launcher enqueues on `stream` and returns the launch error (no sync).
// Segments [seg_begin, seg_end) of kStatsResetInterval candidates (-1: all).
constexpr int kStatsLaunches = 1;
cudaError_t launch_stats(const double* ref, long long n, int m, double* mean, double* sd,
                         cudaStream_t stream, long long seg_begin = 0, long long seg_end = -1);
// env: 2n doubles, (max, min) interleaved; output tiles [tile_begin, tile_end)
// of envelope_tile(r) positions (-1: all).  Tile t reads ref[tT - r, (t+1)T + r).
// Speculative statistics: per-tile prefix sums, and their measured deviation
// from the chain's (out[0]: max relative deviation as bits, out[1]: candidates
// on different sides of the constant-window rule).
int fast_stats_tile(int m);  // 0: window too long
cudaError_t launch_fast_stats(const double* ref, long long n, int m, double* mean, double* sd,
                              cudaStream_t stream);
cudaError_t launch_stats_verify(const double* mean, const double* sd, const double* mean_a,
                                const double* sd_a, long long ncand, unsigned long long* out,
                                cudaStream_t stream);
int envelope_tile(int r);
cudaError_t launch_envelope(const double* ref, long long n, int r, double* env,
                            cudaStream_t stream, long long tile_begin = 0, long long tile_end = -1);
// gmem: the per-warp buffers are in SearchParams::gscratch, not shared memory.
size_t search_smem_bytes(int m, int warps, int ad_k, bool gmem = false);
size_t search_warp_buf_doubles(int m, int ad_k);
// Window parameter of the anti-diagonal engine for a band of half width w
// over series of length n: the smallest of 1/3/5 whose window 64K covers
// the band, else 5 (odd K keeps shared-memory reads conflict-free).
int choose_ad_k(int n, int w);
cudaError_t launch_search(const SearchParams& p, int blocks, int warps, cudaStream_t stream);
// Rank pass (the threshold's warm start): the layered LB_Kim of every S-th
// candidate of [p.begin, p.end), then the candidates whose bound is among the
// ~k smallest (a 2^16-bin histogram of the float bits) into list (<= cap,
// count in *nlist).  scratch: 4 * ceil((end-begin)/S) + 4 * 65536 + 8 bytes.
size_t rank_scratch_bytes(long long ncand, long long S);
cudaError_t launch_rank(const SearchParams& p, long long S, void* scratch, cudaStream_t stream);
// Wave w selects the candidates ranked in [k_{w-1}, k_w) (disjoint waves).
cudaError_t launch_rank_select(const SearchParams& p, long long S, int wave, long long k,
                               long long cap, void* scratch, long long* list,
                               unsigned long long* nlist, cudaStream_t stream);
cudaError_t launch_pairwise(const PairParams& p, cudaStream_t stream);
// bounds.cu: the reference's single-pair lower-bound helpers on the device
cudaError_t launch_lb_kim_fl(const double* q, const double* c, long long l, double* out,
                             cudaStream_t s);
cudaError_t launch_lb_keogh(const double* up, const double* lo, const double* x, long long l,
                            double abandon_above, const unsigned long long* order, double* total,
                            double* contrib, int* abandoned, cudaStream_t s);
cudaError_t launch_cumulative_bound(const double* c, long long l, double* cb, cudaStream_t s);
// Sliding (max, min) interleaved in env (2n) for any radius r; scratch holds
// envelope_any_scratch_doubles(n, r) doubles (0 when the tiled kernel fits).
size_t envelope_any_scratch_doubles(long long n, long long r);
cudaError_t launch_envelope_any(const double* x, long long n, long long r, double* env,
                                double* scratch, cudaStream_t s);
cudaError_t launch_nn1(const Nn1Params& p, cudaStream_t stream);
cudaError_t launch_init_best(BestRecord* rec, unsigned long long* keys, long long count,
                             cudaStream_t stream);
cudaError_t launch_check_finite(const double* x, long long n, unsigned long long* flag,
                                cudaStream_t stream);
#ifdef EAPDTW_PHASE_CLOCKS
void debug_read_reset(unsigned long long* out16);
#endif
cudaError_t launch_fp64_probe(double* sink, int blocks, int iters, cudaStream_t stream);
cudaError_t launch_fp32_probe(float* sink, int blocks, int iters, cudaStream_t stream);

// Per-cell event log of one DTW (trace.cu); layout = eapdtw_trace_event.
enum : unsigned { kTraceCell = 0, kTraceDiscard = 1, kTracePruningPoint = 2, kTraceAbandon = 3 };
struct TraceEvent {
  unsigned kind, pad_;
  unsigned long long row, col;
  double value;
};
// algo 0 full_scan, 1 left_prune_scan, 2 ea_pruned_scan over rows (the longer
// series) x cols with effective half-window w; buf: 2 (lc + 1) doubles;
// hdr[0] = events (may exceed cap: only cap are stored), hdr[1] = cells.
cudaError_t launch_trace(int algo, const double* rows, long long lr, const double* cols,
                         long long lc, long long w, double ub, double* buf, TraceEvent* ev,
                         long long cap, unsigned long long* hdr, double* result,
                         cudaStream_t stream);

}  // namespace eapdtw_b200
