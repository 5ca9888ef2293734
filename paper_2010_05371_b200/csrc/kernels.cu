// kernels.cu -- sm_100a kernels of the subsequence-search hot path.
//
//   stats_chain_kernel   RunningStats chain, bit-identical to search.cpp:156-168
//   envelope_gw_kernel   global sliding max/min (two-level van Herk/Gil-Werman)
//   search_kernel        persistent: LB_Kim -> LB_Keogh EQ -> LB_Keogh EC -> pruned DTW
//   pairwise_kernel      warp per pair (cfg1, and the single-pair drop-in calls)
//   nn1_kernel           block per (query, database split) with a per-query cutoff (cfg5)
//
// All FP64 arithmetic that must match the CPU oracle bit-for-bit uses explicitly
// rounded intrinsics, and the library is built with -fmad=false as a second
// line of defence.
#include <cfloat>
#include <climits>
#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

#include "dtw_ad.cuh"
#include "screen.cuh"
#include "kernels.cuh"

namespace eapdtw_b200 {

// Raise a kernel's dynamic shared-memory limit, never lower it: the attribute
// is per function (and device), so with several contexts launching the same
// kernel from different host threads a smaller request must not undercut a
// concurrent larger launch.  Thread-safe; one real call per new maximum.
#ifndef EAPDTW_NN1_STEP_BLOCK
#define EAPDTW_NN1_STEP_BLOCK 8  // FP32 engine steps per finish-bookkeeping block in NN1 (dtw_f32.cuh)
#endif
constexpr int kNn1StepBlock = EAPDTW_NN1_STEP_BLOCK;
#ifndef EAPDTW_SEARCH_STEP_BLOCK
#define EAPDTW_SEARCH_STEP_BLOCK 8  // the same in the search kernel (4 -> 8: cfg4 -2%, cfg3-nolb -3%)
#endif
constexpr int kSearchStepBlock = EAPDTW_SEARCH_STEP_BLOCK;

static cudaError_t ensure_dyn_smem(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> granted;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  size_t& cur = granted[{dev, func}];
  if (bytes <= cur) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
  if (e == cudaSuccess) cur = bytes;
  return e;
}

// ---------------------------------------------------------------------------
// Sliding z-normalisation statistics.
//
// The reference keeps one running (sum, sum of squares) chain over the start
// positions and rebuilds it from scratch every 100000 slides
// (search.cpp:156-168).  Its bits depend on that exact sequence of roundings,
// and SURVEY.md A.1 shows any re-association (e.g. prefix sums) misses the
// 1e-9 distance tolerance.  The chain is therefore reproduced step-for-step:
// the 100000-slide segments are independent chains.
//
// A chain is a serial dependency (2 DADD of latency per slide), so the pass
// is latency-bound and needs few SMs.  stats_chain_kernel: one block per
// kChainLanes segments, eight warps (warp w runs on SMSP w % 4):
//   * warp 0, the chains (lane = segment).  An FP64 warp instruction costs
//     the same with 1 or 32 active lanes, so the chains of a block run at the
//     speed of one.  They read their (in, out) values from shared memory as
//     16-byte pairs two batches of 8 slides ahead, with the squares of the
//     next batch computed during this one (the warp issues in order, so no
//     instruction may wait on a load), and write (sum, sumsq) pairs.
//   * warp 4 keeps the ring of kChainDepth tiles of every chain's `in` and
//     `out` rows filled with 16-byte cp.async (rows start 16-byte aligned, one
//     element early if needed): a few issue slots beside the chains on SMSP 0
//     (measured faster than giving the loads to a converter warp).
//   * warps 1-3 and 5-7 turn the previous tile's (sum, sumsq) into mean and
//     stddev with correctly rounded div/sqrt (RunningStats::mean/variance/
//     stddev, search.hpp:34-41, search.cpp:35) and store them as 16-byte
//     pairs.  They run on SMSPs 1..3, so their FP64 work never delays the
//     chains' pipe; two per SMSP hide the dependent div/sqrt latencies.
// The warps hand tiles over through mbarriers (ring slot full / empty,
// accumulator full / empty; the loads arrive through cp.async.mbarrier.arrive),
// so no warp waits on a block-wide barrier: the chains stall only on data.
// The block claims enough shared memory that no other kernel's block shares
// its SM; the envelope runs beside it on the remaining SMs, on another stream.
// (Measured on the way here: per-element cp.async staging 72 cycles/slide at
// 32 chains, per-lane bulk copies 130, a separate conversion kernel 0.5 ms at
// cfg4: the copy loops and the extra pass, not the chains, set the pace.)
// ---------------------------------------------------------------------------
#ifndef EAPDTW_CHAIN_LANES
#define EAPDTW_CHAIN_LANES 16
#endif
#ifndef EAPDTW_CHAIN_DEPTH
#define EAPDTW_CHAIN_DEPTH 3
#endif
constexpr int kChainLanes = EAPDTW_CHAIN_LANES;  // segments (chains) per block
#ifndef EAPDTW_CHAIN_TILE
#define EAPDTW_CHAIN_TILE 128
#endif
constexpr int kChainTile = EAPDTW_CHAIN_TILE;    // slides per tile
constexpr int kChainDepth = EAPDTW_CHAIN_DEPTH;  // input ring slots
// rows of kChainTile + 2 doubles: 16-byte multiples whose 4-word bank offset
// keeps the chain lanes' 16-byte accesses conflict-free
constexpr int kChainRow = kChainTile + 2;
constexpr int kChainThreads = 256;  // warp 0: chains; warp 4: loads; warps 1-3, 5-7: conversion
constexpr int kChainConverters = 6;
constexpr size_t kChainRingDoubles = static_cast<size_t>(kChainDepth) * 2 * kChainLanes * kChainRow;
constexpr size_t kChainAccDoubles = 2ull * 2 * kChainLanes * kChainRow;
// mbarriers: full / empty per ring slot, full / empty per accumulator buffer
constexpr size_t kChainSmemUsed = (kChainRingDoubles + kChainAccDoubles) * 8 + (2 * kChainDepth + 4) * 8;
constexpr size_t kChainSmem = kChainSmemUsed > 150 * 1024 ? kChainSmemUsed : 150 * 1024;

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem_src) : "memory");
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// arrives once this thread's earlier cp.async copies have landed
__device__ __forceinline__ void mbar_arrive_cp_async(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// RunningStats::mean / stddev from (sum, sumsq); a power-of-two m divides
// exactly by multiplying with 1/m.
template <bool POW2>
__device__ __forceinline__ void stats_of(double sum, double sq, double dm, double inv_m, double& mu,
                                         double& sd) {
  mu = POW2 ? __dmul_rn(sum, inv_m) : __ddiv_rn(sum, dm);
  const double var = __dsub_rn(POW2 ? __dmul_rn(sq, inv_m) : __ddiv_rn(sq, dm), __dmul_rn(mu, mu));
  sd = __dsqrt_rn(var > 0.0 ? var : 0.0);
}

// OFF_IN / OFF_OUT: position of a tile's first `in` / `out` value in its row.
template <int OFF_IN, int OFF_OUT, bool POW2>
__global__ void __launch_bounds__(kChainThreads, 1) stats_chain_kernel(
    const double* __restrict__ ref, long long n, int m, double* __restrict__ mean_out,
    double* __restrict__ sd_out, long long seg_begin, long long seg_end) {
  extern __shared__ __align__(16) double csm[];
  double* ring = csm;                     // [depth][in, out][lanes][row]
  double* acc = csm + kChainRingDoubles;  // [2][sum, sumsq][lanes][row]
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(acc + kChainAccDoubles);
  unsigned long long* slot_full = bars;                  // loads landed (32 loader lanes)
  unsigned long long* slot_empty = bars + kChainDepth;   // chains done reading (1)
  unsigned long long* acc_full = bars + 2 * kChainDepth; // chains wrote (sum, sumsq) (1)
  unsigned long long* acc_empty = acc_full + 2;          // converters done (kChainConverters)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long ncand = n - m + 1;
  const long long seg0 = seg_begin + static_cast<long long>(blockIdx.x) * kChainLanes;
  const int nch = static_cast<int>(min(static_cast<long long>(kChainLanes), seg_end - seg0));
  // only the reference's last segment is short
  auto seg_len = [&](int c) -> int {
    return static_cast<int>(
        min(static_cast<long long>(kStatsResetInterval), ncand - (seg0 + c) * kStatsResetInterval));
  };
  const int ntiles = (seg_len(0) + kChainTile - 1) / kChainTile;
  const int last_len = seg_len(nch - 1);
  const long long s00 = seg0 * kStatsResetInterval;
  const double dm = static_cast<double>(m), inv_m = 1.0 / dm;

  // warp 4: tile t's `in` row of chain c starts at s0 + t*T + m - 1 - OFF_IN,
  // its `out` row at s0 + t*T - 1 - OFF_OUT (16-byte aligned).  All rows of a
  // tile lie inside [0, n) except in the reference's first and last tiles;
  // those rows are filled element by element.
  const long long last_row = (seg0 + nch - 1) * kStatsResetInterval;
  auto produce = [&](int t) {
    const int slot = t % kChainDepth;
    const long long t0 = static_cast<long long>(t) * kChainTile;
    const long long a_in = s00 + t0 + m - 1 - OFF_IN, a_out = s00 + t0 - 1 - OFF_OUT;
    double* rin = ring + (slot * 2 + 0) * kChainLanes * kChainRow;
    double* rout = ring + (slot * 2 + 1) * kChainLanes * kChainRow;
    if (a_out >= 0 && last_row + t0 + m - 1 - OFF_IN + kChainRow <= n) {
      const double* gi = ref + a_in + 2 * lane;
      const double* go = ref + a_out + 2 * lane;
#pragma unroll 4
      for (int c = 0; c < nch; ++c) {
#pragma unroll
        for (int k = 2 * lane; k < kChainRow; k += 64) {
          cp_async16(rin + c * kChainRow + k, gi + k - 2 * lane);
          cp_async16(rout + c * kChainRow + k, go + k - 2 * lane);
        }
        gi += kStatsResetInterval;
        go += kStatsResetInterval;
      }
      mbar_arrive_cp_async(&slot_full[slot]);
    } else {
      for (int c = 0; c < nch; ++c) {
        const long long ai = a_in + c * kStatsResetInterval, ao = a_out + c * kStatsResetInterval;
        for (int k = lane; k < kChainRow; k += 32) {
          rin[c * kChainRow + k] = (ai + k >= 0 && ai + k < n) ? ref[ai + k] : 0.0;
          rout[c * kChainRow + k] = (ao + k >= 0 && ao + k < n) ? ref[ao + k] : 0.0;
        }
      }
      mbar_arrive(&slot_full[slot]);
    }
  };
  // converter warps: (sum, sumsq) of tile t -> (mean, stddev), 16-byte pairs
  // (segments and tiles start at even indices; mean / sd are 16-byte aligned)
  auto convert = [&](int t) {
    const int b = t & 1;
    const long long t0 = static_cast<long long>(t) * kChainTile;
    const double* as = acc + (b * 2 + 0) * kChainLanes * kChainRow;
    const double* aq = acc + (b * 2 + 1) * kChainLanes * kChainRow;
    const int full_cnt = static_cast<int>(min(static_cast<long long>(kChainTile), kStatsResetInterval - t0));
    const int last_cnt = static_cast<int>(max(0LL, min(static_cast<long long>(kChainTile), last_len - t0)));
    const int rank = warp < 4 ? warp - 1 : warp - 2;
    for (int i = rank * 32 + lane; i < nch * (kChainTile / 2); i += kChainConverters * 32) {
      const int c = i / (kChainTile / 2), k = 2 * (i % (kChainTile / 2));
      const int cnt = c == nch - 1 ? last_cnt : full_cnt;
      if (k >= cnt) continue;
      const double2 v = *reinterpret_cast<const double2*>(as + c * kChainRow + k);
      const double2 w = *reinterpret_cast<const double2*>(aq + c * kChainRow + k);
      const long long s = s00 + c * kStatsResetInterval + t0 + k;
      double m0, d0, m1, d1;
      stats_of<POW2>(v.x, w.x, dm, inv_m, m0, d0);
      if (k + 1 < cnt) {
        stats_of<POW2>(v.y, w.y, dm, inv_m, m1, d1);
        *reinterpret_cast<double2*>(mean_out + s) = make_double2(m0, m1);
        *reinterpret_cast<double2*>(sd_out + s) = make_double2(d0, d1);
      } else {
        mean_out[s] = m0;
        sd_out[s] = d0;
      }
    }
  };

  if (threadIdx.x == 0) {
    for (int d = 0; d < kChainDepth; ++d) {
      mbar_init(&slot_full[d], 32);
      mbar_init(&slot_empty[d], 1);
    }
    for (int d = 0; d < 2; ++d) {
      mbar_init(&acc_full[d], 1);
      mbar_init(&acc_empty[d], kChainConverters);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // No block-wide barrier after this point: every hand-over is an mbarrier
  // phase (use u of a slot or buffer completes phase u, parity u & 1).
  if (warp == 4) {  // loads run ahead as far as the ring allows
    for (int t = 0; t < ntiles; ++t) {
      if (t >= kChainDepth) mbar_wait(&slot_empty[t % kChainDepth], ((t / kChainDepth) - 1) & 1);
      produce(t);
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    return;
  }
  if (warp >= 1) {  // converters
    for (int t = 0; t < ntiles; ++t) {
      mbar_wait(&acc_full[t & 1], (t >> 1) & 1);
      convert(t);
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[t & 1]);
    }
    return;
  }
  // warp 0: the chains
  double sum = 0.0, sq = 0.0;
  if (lane < nch) {  // RunningStats::over(ref[s0 : s0+m]) (search.cpp:25-33)
    const long long s0 = (seg0 + lane) * kStatsResetInterval;
#pragma unroll 16
    for (int k = 0; k < m; ++k) {
      const double x = ref[s0 + k];
      sum = __dadd_rn(sum, x);
      sq = __dadd_rn(sq, __dmul_rn(x, x));
    }
  }
  for (int t = 0; t < ntiles; ++t) {
    const int slot = t % kChainDepth;
    mbar_wait(&slot_full[slot], (t / kChainDepth) & 1);
    if (t >= 2) mbar_wait(&acc_empty[t & 1], ((t >> 1) - 1) & 1);
    if (lane < kChainLanes) {
      const double* rin = ring + ((slot * 2 + 0) * kChainLanes + lane) * kChainRow;
      const double* rout = ring + ((slot * 2 + 1) * kChainLanes + lane) * kChainRow;
      double* as = acc + (((t & 1) * 2 + 0) * kChainLanes + lane) * kChainRow;
      double* aq = acc + (((t & 1) * 2 + 1) * kChainLanes + lane) * kChainRow;
      // stats.add(in); stats.remove(out) (search.hpp:23-32).  A batch is 8
      // slides: its (in, out) values and their squares are in registers
      // before it starts.  Lanes past their segment's end (the short last
      // one) compute on filler values that are never stored.
      struct Batch {
        double in[8], out[8], qi[8], qo[8];
      };
      auto load = [&](int k, Batch& b) {
        double vi[10], vo[10];
#pragma unroll
        for (int u = 0; u < 5; ++u) {
          const double2 a = *reinterpret_cast<const double2*>(rin + k + 2 * u);
          const double2 c = *reinterpret_cast<const double2*>(rout + k + 2 * u);
          vi[2 * u] = a.x;
          vi[2 * u + 1] = a.y;
          vo[2 * u] = c.x;
          vo[2 * u + 1] = c.y;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          b.in[u] = vi[u + OFF_IN];
          b.out[u] = vo[u + OFF_OUT];
        }
      };
      auto squares = [&](Batch& b) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          b.qi[u] = __dmul_rn(b.in[u], b.in[u]);
          b.qo[u] = __dmul_rn(b.out[u], b.out[u]);
        }
      };
      auto run = [&](int k, const Batch& b) {
        double ps[8], pq[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (u == 0 && t == 0 && k == 0) {  // the segment's first position: the over() result
            ps[0] = sum;
            pq[0] = sq;
            continue;
          }
          sum = __dsub_rn(__dadd_rn(sum, b.in[u]), b.out[u]);
          sq = __dsub_rn(__dadd_rn(sq, b.qi[u]), b.qo[u]);
          ps[u] = sum;
          pq[u] = sq;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          *reinterpret_cast<double2*>(as + k + 2 * u) = make_double2(ps[2 * u], ps[2 * u + 1]);
          *reinterpret_cast<double2*>(aq + k + 2 * u) = make_double2(pq[2 * u], pq[2 * u + 1]);
        }
      };
      Batch b0, b1;
      load(0, b0);
      squares(b0);
#pragma unroll 1
      for (int k = 0; k < kChainTile; k += 16) {
        load(k + 8, b1);
        squares(b1);
        run(k, b0);
        if (k + 16 < kChainTile) {
          load(k + 16, b0);
          squares(b0);
        }
        run(k + 8, b1);
      }
    }
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&slot_empty[slot]);
      mbar_arrive(&acc_full[t & 1]);
    }
  }
}

cudaError_t launch_stats(const double* ref, long long n, int m, double* mean, double* sd,
                         cudaStream_t stream, long long seg_begin, long long seg_end) {
  const long long ncand = n - m + 1;
  const long long nseg = (ncand + kStatsResetInterval - 1) / kStatsResetInterval;
  if (seg_end < 0 || seg_end > nseg) seg_end = nseg;
  if (seg_begin >= seg_end) return cudaSuccess;
  // 16-byte pair stores (segments start at even indices)
  if ((reinterpret_cast<uintptr_t>(mean) | reinterpret_cast<uintptr_t>(sd)) & 15) return cudaErrorInvalidValue;
  // row starts s0 + t*T + m - 1 - OFF_IN and s0 + t*T - 1 - OFF_OUT must be
  // 16-byte aligned; s0 + t*T is even
  const unsigned par = static_cast<unsigned>((reinterpret_cast<uintptr_t>(ref) >> 3) & 1);
  const int off_in = static_cast<int>((par + static_cast<unsigned>(m - 1)) & 1);
  const int off_out = static_cast<int>((par + 1u) & 1);
  const bool pow2 = (m & (m - 1)) == 0;
  using Fn = void (*)(const double*, long long, int, double*, double*, long long, long long);
  static const Fn fns[2][2][2] = {
      {{stats_chain_kernel<0, 0, false>, stats_chain_kernel<0, 0, true>},
       {stats_chain_kernel<0, 1, false>, stats_chain_kernel<0, 1, true>}},
      {{stats_chain_kernel<1, 0, false>, stats_chain_kernel<1, 0, true>},
       {stats_chain_kernel<1, 1, false>, stats_chain_kernel<1, 1, true>}}};
  const Fn fn = fns[off_in][off_out][pow2 ? 1 : 0];
  const cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(fn), kChainSmem);
  if (e != cudaSuccess) return e;
  const long long blocks = (seg_end - seg_begin + kChainLanes - 1) / kChainLanes;
  fn<<<static_cast<unsigned>(blocks), kChainThreads, kChainSmem, stream>>>(ref, n, m, mean, sd, seg_begin,
                                                                           seg_end);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Speculative statistics (north_star (1): running mean / stddev via prefix
// sums).  The exact chain above is a serial dependency of 100000 slides per
// segment (~1.5 ms whatever the size of the search); everything that only has
// to be SOUND, not bit-exact -- the lower-bound tiers, the FP32 screen, the
// warm start's thresholds -- can run on statistics from per-tile prefix sums
// instead, with its guards widened for an assumed deviation eps, while the
// chain runs beside it on a few SMs.  Once the chain is done,
// stats_verify_kernel measures the actual deviation of the prefix statistics
// from the chain's; only candidates whose evaluation completed are then
// re-evaluated with the exact statistics (capi.cu: speculation).
//
// fast_stats_kernel: a tile of T candidates per block; the T + m - 1 points
// are staged in shared memory, each thread runs an inclusive prefix over its
// contiguous chunk (sum and sum of squares), the chunk totals are scanned
// across the block, and a window's sums are prefix differences.  Same
// mean / variance formulas as RunningStats (search.hpp:34-41).
// ---------------------------------------------------------------------------
constexpr int kFastThreads = 256;
int fast_stats_tile(int m) {
  // (T + m) * 16 bytes of shared memory within ~96 KB (2 blocks per SM)
  const long long cap = (96 * 1024) / 16;
  long long T = cap - m;
  if (T > 4096) T = 4096;
  return T >= 256 ? static_cast<int>(T) : 0;  // 0: the window is too long for a tile
}

template <bool POW2>
__global__ void __launch_bounds__(kFastThreads) fast_stats_kernel(const double* __restrict__ ref,
                                                                  long long n, int m, int T,
                                                                  double* __restrict__ mean,
                                                                  double* __restrict__ sd) {
  extern __shared__ double fsm[];
  const long long ncand = n - m + 1;
  const long long s0 = static_cast<long long>(blockIdx.x) * T;
  const int cnt = static_cast<int>(min(static_cast<long long>(T), ncand - s0));
  const int L = cnt + m - 1;
  double* P1 = fsm;              // P1[i + 1]: inclusive prefix of x over the tile, P1[0] = 0
  double* P2 = fsm + (T + m);    // the same of x^2
  __shared__ double tot1[kFastThreads], tot2[kFastThreads];
  const int t = threadIdx.x;
  for (int i = t; i < L; i += kFastThreads) P1[i + 1] = ref[s0 + i];
  if (t == 0) {
    P1[0] = 0.0;
    P2[0] = 0.0;
  }
  __syncthreads();
  // odd chunk length: the threads' strided accesses fall in different banks
  const int c = ((L + kFastThreads - 1) / kFastThreads) | 1;
  const int b = min(L, t * c), e = min(L, b + c);
  double a1 = 0.0, a2 = 0.0;
  for (int i = b; i < e; ++i) {
    const double x = P1[i + 1];
    a1 += x;
    a2 += x * x;
    P1[i + 1] = a1;
    P2[i + 1] = a2;
  }
  tot1[t] = a1;
  tot2[t] = a2;
  __syncthreads();
  // exclusive scan of the chunk totals (256 values: one warp, 8 per lane)
  if (t < 32) {
    double r1[8], r2[8], l1 = 0.0, l2 = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      r1[k] = l1;
      r2[k] = l2;
      l1 += tot1[8 * t + k];
      l2 += tot2[8 * t + k];
    }
    double i1 = l1, i2 = l2;
    for (int off = 1; off < 32; off <<= 1) {
      const double y1 = __shfl_up_sync(0xffffffffu, i1, off), y2 = __shfl_up_sync(0xffffffffu, i2, off);
      if (t >= off) {
        i1 += y1;
        i2 += y2;
      }
    }
    const double e1 = i1 - l1, e2 = i2 - l2;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      tot1[8 * t + k] = e1 + r1[k];
      tot2[8 * t + k] = e2 + r2[k];
    }
  }
  __syncthreads();
  const double o1 = tot1[t], o2 = tot2[t];
  for (int i = b; i < e; ++i) {
    P1[i + 1] += o1;
    P2[i + 1] += o2;
  }
  __syncthreads();
  const double dm = static_cast<double>(m), inv_m = 1.0 / dm;
  for (int k = t; k < cnt; k += kFastThreads) {
    double mu, sg;
    stats_of<POW2>(P1[k + m] - P1[k], P2[k + m] - P2[k], dm, inv_m, mu, sg);
    mean[s0 + k] = mu;
    sd[s0 + k] = sg;
  }
}

cudaError_t launch_fast_stats(const double* ref, long long n, int m, double* mean, double* sd,
                              cudaStream_t stream) {
  const int T = fast_stats_tile(m);
  if (T <= 0) return cudaErrorInvalidValue;
  const long long ncand = n - m + 1;
  const size_t smem = static_cast<size_t>(T + m) * 16;
  const bool pow2 = (m & (m - 1)) == 0;
  const void* fn = pow2 ? reinterpret_cast<const void*>(fast_stats_kernel<true>)
                        : reinterpret_cast<const void*>(fast_stats_kernel<false>);
  const cudaError_t e = ensure_dyn_smem(fn, smem);
  if (e != cudaSuccess) return e;
  const unsigned grid = static_cast<unsigned>((ncand + T - 1) / T);
  if (pow2) fast_stats_kernel<true><<<grid, kFastThreads, smem, stream>>>(ref, n, m, T, mean, sd);
  else fast_stats_kernel<false><<<grid, kFastThreads, smem, stream>>>(ref, n, m, T, mean, sd);
  return cudaGetLastError();
}

// out[0]: max over the candidates of max(|mean_a - mean|, |sd_a - sd|) / sd as
// order-preserving bits (a deviation of the normalised value c of at most
// out[0] * (1 + |c|)); out[1]: candidates on different sides of kMinStddev
// (the constant-window rule, search.cpp:37-46) or with non-finite statistics.
__global__ void __launch_bounds__(256) stats_verify_kernel(const double* __restrict__ mean,
                                                           const double* __restrict__ sd,
                                                           const double* __restrict__ mean_a,
                                                           const double* __restrict__ sd_a,
                                                           long long ncand,
                                                           unsigned long long* __restrict__ out) {
  double worst = 0.0;
  unsigned long long bad = 0;
  for (long long k = blockIdx.x * 256LL + threadIdx.x; k < ncand; k += 256LL * gridDim.x) {
    const double mu = mean[k], sg = sd[k], ma = mean_a[k], sa = sd_a[k];
    const bool c0 = sg < kMinStddev, c1 = sa < kMinStddev;
    if (c0 != c1 || !(fabs(ma) <= DBL_MAX) || !(sa <= DBL_MAX) || !(sg <= DBL_MAX)) {
      ++bad;
    } else if (!c0) {
      const double r = 1.0 / sg;
      worst = fmax(worst, fmax(fabs(ma - mu), fabs(sa - sg)) * r);
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, off));
    bad += __shfl_xor_sync(0xffffffffu, bad, off);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(worst)));
    if (bad) atomicAdd(out + 1, bad);
  }
}

cudaError_t launch_stats_verify(const double* mean, const double* sd, const double* mean_a,
                                const double* sd_a, long long ncand, unsigned long long* out,
                                cudaStream_t stream) {
  const long long blocks = std::min<long long>((ncand + 255) / 256, 148LL * 8);
  stats_verify_kernel<<<static_cast<unsigned>(std::max<long long>(1, blocks)), 256, 0, stream>>>(
      mean, sd, mean_a, sd_a, ncand, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Global raw envelope for the LB_Keogh EC tier.
//
// The reference builds, per surviving candidate, the envelope of the
// normalised candidate with a deque sweep (lower_bounds.cpp:9-49, called from
// search.cpp:97).  Normalisation x -> (x-mean)/sd is monotone, so the
// normalised envelope equals the normalised raw envelope.  Here the raw
// envelope is built ONCE for the whole reference with radius r; at the two
// candidate edges (j < r or j > m-1-r) the global window is a superset of the
// candidate's clamped window, which only loosens the bound (still sound).
//
// Window K = 2r+1 >= 8: two-level van Herk / Gil-Werman per tile.  Level 1:
// blocks of 8 positions, one per thread, prefix and suffix max/min in
// registers -> shared memory (g, h).  Level 2: the block maxima/minima,
// doubled k times (k = floor(log2(q-1)), q = floor((K-1)/8)) so that one
// lookup pair covers any run of q-1 or q whole blocks.  The window [s, s+K-1]
// is then h[s] (rest of s's block), g[s+K-1] (the last block up to s+K-1) and
// the whole blocks strictly between: ~12 shared-memory accesses per position
// for both envelopes instead of the ~50 of plain doubling, so the kernel runs
// at HBM speed (reads 8 B, writes 16 B per position).
// K < 8 (or a tile too large for shared memory): sparse-table doubling.
// ---------------------------------------------------------------------------
constexpr int kEnvThreads = 256;
struct EnvGeom {
  int gw;      // 1: Gil-Werman kernel, 0: doubling kernel
  int len, T;  // loaded positions, outputs per tile
  int nb, k;   // Gil-Werman: blocks of 8 per tile, doubling passes over them
  size_t smem;
};
__host__ __device__ inline int env_pad(int i) { return i + (i >> 3); }  // 9-double lane stride

static EnvGeom env_geom(int r) {
  EnvGeom g{};
  const long long K = 2LL * r + 1;
  if (K >= 8) {
    const long long len = std::max<long long>(2048, (2LL * r + 1 + 1024 + 63) / 64 * 64);
    const long long nb = len / 8;
    const long long q = (K - 1) / 8;
    int k = 0;
    while ((2LL << k) <= q - 1) ++k;
    const size_t smem = 4 * static_cast<size_t>(env_pad(static_cast<int>(std::min(len, 1LL << 24)))) * 8 +
                        4 * static_cast<size_t>(nb) * 8;
    if (len < (1LL << 24) && smem <= 200 * 1024) {
      g.gw = 1;
      g.len = static_cast<int>(len);
      g.T = static_cast<int>(len - 2 * r - 1);
      g.nb = static_cast<int>(nb);
      g.k = k;
      g.smem = smem;
      return g;
    }
  }
  // two ping-pong arrays of (T + 2r) doubles within 64 KB (3 blocks per SM)
  const long long cap = (64 * 1024) / (2 * 8);
  long long T = cap - 2LL * r;
  if (T > 8192) T = 8192;
  g.gw = 0;
  g.T = static_cast<int>(std::max<long long>(T, -1));
  g.len = static_cast<int>(std::max<long long>(T + 2LL * r, 0));
  g.smem = 2 * static_cast<size_t>(std::max(g.len, 0)) * sizeof(double);
  return g;
}

__global__ void __launch_bounds__(kEnvThreads) envelope_gw_kernel(
    const double* __restrict__ ref, long long n, int r, int T, int len, int nb, int k,
    double2* __restrict__ env, long long tile_begin) {
  extern __shared__ double esm[];
  const int plen = env_pad(len);
  double* gmax = esm;
  double* gmin = esm + plen;
  double* hmax = esm + 2 * plen;
  double* hmin = esm + 3 * plen;
  double* st = esm + 4 * plen;  // [2 ping-pong][max, min][nb]
  const long long P0 = (tile_begin + blockIdx.x) * static_cast<long long>(T);  // first output
  // first loaded position, even-aligned in memory so blocks load as 16-byte pairs
  const long long Ar = P0 - r;
  const int d = static_cast<int>(((reinterpret_cast<uintptr_t>(ref) >> 3) + static_cast<uintptr_t>(Ar)) & 1);
  const long long A = Ar - d;
  // level 1: prefix / suffix max and min of each 8-position block
  for (int b = threadIdx.x; b < nb; b += kEnvThreads) {
    const long long p = A + 8LL * b;
    double vx[8], vn[8];
    if (p >= 0 && p + 8 <= n) {
      const double2* src = reinterpret_cast<const double2*>(ref + p);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double2 t = __ldg(src + u);
        vx[2 * u] = vn[2 * u] = t.x;
        vx[2 * u + 1] = vn[2 * u + 1] = t.y;
      }
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const bool in = p + u >= 0 && p + u < n;
        const double x = in ? ref[p + u] : 0.0;
        vx[u] = in ? x : -d_inf();
        vn[u] = in ? x : d_inf();
      }
    }
    const int o = env_pad(8 * b);
    double ax = vx[0], an = vn[0];
    gmax[o] = ax;
    gmin[o] = an;
#pragma unroll
    for (int u = 1; u < 8; ++u) {
      ax = fmax(ax, vx[u]);
      an = fmin(an, vn[u]);
      gmax[o + u] = ax;
      gmin[o + u] = an;
    }
    st[b] = ax;       // block maximum
    st[nb + b] = an;  // block minimum
    ax = vx[7];
    an = vn[7];
    hmax[o + 7] = ax;
    hmin[o + 7] = an;
#pragma unroll
    for (int u = 6; u >= 0; --u) {
      ax = fmax(ax, vx[u]);
      an = fmin(an, vn[u]);
      hmax[o + u] = ax;
      hmin[o + u] = an;
    }
  }
  __syncthreads();
  // level 2: block extrema over runs of 2^k blocks
  for (int j = 0; j < k; ++j) {
    const double* sx = st + (j & 1) * 2 * nb;
    double* dx = st + ((j + 1) & 1) * 2 * nb;
    const int valid = nb - (2 << j) + 1;
    for (int b = threadIdx.x; b < valid; b += kEnvThreads) {
      dx[b] = fmax(sx[b], sx[b + (1 << j)]);
      dx[nb + b] = fmin(sx[nb + b], sx[nb + b + (1 << j)]);
    }
    __syncthreads();
  }
  const double* sk = st + (k & 1) * 2 * nb;
  const int K = 2 * r + 1;
  for (int t = threadIdx.x; t < T; t += kEnvThreads) {
    const long long P = P0 + t;
    if (P >= n) break;
    const int s = t + d, e = s + K - 1;
    double mx = fmax(hmax[env_pad(s)], gmax[env_pad(e)]);
    double mn = fmin(hmin[env_pad(s)], gmin[env_pad(e)]);
    const int a = s >> 3, z = e >> 3;
    if (z - a >= 2) {  // whole blocks a+1 .. z-1: two overlapping runs of 2^k
      const int lo = a + 1, hi = z - (1 << k);
      mx = fmax(mx, fmax(sk[lo], sk[hi]));
      mn = fmin(mn, fmin(sk[nb + lo], sk[nb + hi]));
    }
    env[P] = make_double2(mx, mn);
  }
}

template <bool MAX>
__device__ __forceinline__ double pick(double a, double b) {
  return MAX ? (a > b ? a : b) : (a < b ? a : b);
}

template <bool MAX>
__device__ void envelope_doubling(const double* __restrict__ ref, long long n, long long A, int len,
                                  int r, int T, long long P0, double* buf0, double* buf1,
                                  double* __restrict__ out) {
  const double ident = MAX ? -d_inf() : d_inf();
  for (int k = threadIdx.x; k < len; k += blockDim.x) {
    const long long p = A + k;
    buf0[k] = (p >= 0 && p < n) ? ref[p] : ident;
  }
  __syncthreads();
  const int K = 2 * r + 1;
  int P = 1;
  while (2 * P <= K) P *= 2;
  double* src = buf0;
  double* dst = buf1;
  for (int s = 1; s < P; s *= 2) {  // M_{2s}[i] = max(M_s[i], M_s[i+s])
    const int valid = len - 2 * s + 1;
    for (int k = threadIdx.x; k < valid; k += blockDim.x) dst[k] = pick<MAX>(src[k], src[k + s]);
    __syncthreads();
    double* t = src;
    src = dst;
    dst = t;
  }
  for (int t = threadIdx.x; t < T; t += blockDim.x) {  // interleaved (max, min)
    if (P0 + t < n) out[2 * (P0 + t) + (MAX ? 0 : 1)] = pick<MAX>(src[t], src[t + K - P]);
  }
  __syncthreads();
}

__global__ void __launch_bounds__(512) envelope_kernel(const double* __restrict__ ref, long long n,
                                                       int r, int T, double* __restrict__ env,
                                                       long long tile_begin) {
  extern __shared__ double smem[];
  const int len = T + 2 * r;
  const long long P0 = (tile_begin + blockIdx.x) * T;  // first output
  const long long A = P0 - r;                                   // first input
  envelope_doubling<true>(ref, n, A, len, r, T, P0, smem, smem + len, env);
  envelope_doubling<false>(ref, n, A, len, r, T, P0, smem, smem + len, env);
}

int envelope_tile(int r) { return env_geom(r).T; }

cudaError_t launch_envelope(const double* ref, long long n, int r, double* env,
                            cudaStream_t stream, long long tile_begin, long long tile_end) {
  const EnvGeom g = env_geom(r);
  if (g.T < 256) return cudaErrorInvalidValue;  // caller disables the EC tier
  const void* fn = g.gw ? reinterpret_cast<const void*>(envelope_gw_kernel)
                        : reinterpret_cast<const void*>(envelope_kernel);
  cudaError_t e = ensure_dyn_smem(fn, g.smem);
  if (e != cudaSuccess) return e;
  const long long ntiles = (n + g.T - 1) / g.T;
  if (tile_end < 0 || tile_end > ntiles) tile_end = ntiles;
  if (tile_begin >= tile_end) return cudaSuccess;
  const unsigned grid = static_cast<unsigned>(tile_end - tile_begin);
  if (g.gw)
    envelope_gw_kernel<<<grid, kEnvThreads, g.smem, stream>>>(ref, n, r, g.T, g.len, g.nb, g.k,
                                                              reinterpret_cast<double2*>(env), tile_begin);
  else
    envelope_kernel<<<grid, 512, g.smem, stream>>>(ref, n, r, g.T, env, tile_begin);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Fused persistent search kernel (the cascade_decision + kernel dispatch of
// search.cpp:160-204, re-organised for a GPU).
//
// Two kinds of work share one persistent grid:
//   * LB chunks: a warp claims 32 consecutive candidates (atomic chunk
//     counter, so the sweep advances through the reference in order like the
//     CPU's sequential best-so-far) and runs the lower-bound tiers
//     lane-per-candidate over coalesced 256-byte rows of the reference, each
//     tier pruning against the CURRENT global threshold.  Survivors are
//     appended to a global queue.
//   * DTW tasks: a warp pops one survivor and evaluates it with warp_dtw,
//     re-reading the threshold at every 32-row strip.
// A warp always drains the queue before claiming a new chunk, so a chunk's
// survivors are spread over the whole GPU instead of serialising on one warp.
//
// Soundness: LB_Kim is computed with the DTW's own IEEE divisions and is
// bit-for-bit <= the DTW value; the Keogh tiers normalise by
// reciprocal multiplication and prune only when lb > ub*(1+guard_rel) +
// guard_abs.  Survivors are evaluated exactly, and the record
// keeps the lowest index among equal distances, so the result is the
// reference's (first strict minimum, search.cpp:199).
// ---------------------------------------------------------------------------
// Shared-memory padding of the query / per-warp buffers: enough for the strip
// engine (kPadL/kPadR) and for the anti-diagonal engine with K = ad_k.
static __host__ __device__ inline int smem_pad(int ad_k) {
  const int p = ad_k > 0 ? ad_pad(ad_k) : 0;
  return p > kPadR ? p : kPadR;
}
static __host__ __device__ inline size_t padded_len(int m, int ad_k) {
  return static_cast<size_t>(m) + 2 + 2 * static_cast<size_t>(smem_pad(ad_k));
}

// Per-warp buffer: the exact engine's row (or the EQ staging tile), which
// the FP32 screen's two float rows (forward and reversed pass) alias.
static __host__ __device__ inline size_t warp_buf_doubles(int m, int ad_k) {
  return padded_len(m, ad_k) + kStageExtra;
}
// The query as float (FP32 screen), padded like the FP64 copy.
static __host__ __device__ inline size_t q32_len(int m) {
  return static_cast<size_t>(m) + 2 + 2 * static_cast<size_t>(kPadR);
}

size_t search_warp_buf_doubles(int m, int ad_k) { return warp_buf_doubles(m, ad_k); }

size_t search_smem_bytes(int m, int warps, int ad_k, bool gmem) {
  return padded_len(m, ad_k) * 8                        // q (padded, 1-based)
         + (gmem ? 0 : static_cast<size_t>(warps) * warp_buf_doubles(m, ad_k) * 8)  // per-warp buffers
         + static_cast<size_t>(warps) * kStackBytesPerWarp  // per-warp tier stacks
         + (q32_len(m) * 4 + 7) / 8 * 8                       // q as float (FP32 screens)
         + 64;
}

int choose_ad_k(int n, int w) {
  // The anti-diagonal engine wins (1.25-1.45x per cell, scratch/engine
  // measurements in DESIGN.md) only when its window holds the whole band, so
  // it can never overflow; wider bands use the strip engine.
  const long long band = std::min(2LL * w + 1, 2LL * n - 1);
  if (band <= 64) return 1;
  if (band <= 192) return 3;
  return 0;
}

// One exact pruned DTW with the whole warp: the anti-diagonal engine with
// window 64*ad_k first, the strip engine when the live region overflows it
// (or ad_k == 0).  Both share `buf` (their DP scratch).
template <bool KILL, bool LEFT = false, class RawFn, class NormFn, class UbFn, class RowThrFn>
__device__ double dtw_dispatch(int ad_k, const RawFn& rowraw, const NormFn& rownorm, int lr,
                               const double* qsp, int lc, int w, UbFn&& get_ub, RowThrFn&& rowthr,
                               double* buf, unsigned long long& cells,
                               unsigned long long& overflows) {
  if (!KILL && !LEFT && ad_k > 0) {
    double r = d_inf();
    int st = kAdOverflow;
    // odd K: lanes read shared memory at an odd 8-byte stride, i.e. without
    // bank conflicts (2 wavefronts per 64-bit access, the minimum)
    if (ad_k == 1) st = warp_dtw_ad<1>(rowraw, rownorm, lr, qsp, lc, w, get_ub, buf, r, cells);
    else if (ad_k == 3) st = warp_dtw_ad<3>(rowraw, rownorm, lr, qsp, lc, w, get_ub, buf, r, cells);
    else st = warp_dtw_ad<5>(rowraw, rownorm, lr, qsp, lc, w, get_ub, buf, r, cells);
    if (st == kAdOk) return r;
    ++overflows;
    __syncwarp();
  }
  return warp_dtw<KILL, LEFT>(rowraw, rownorm, lr, qsp, lc, w, get_ub, rowthr, buf, cells);
}

// Pruning threshold of the guarded lower bounds (Kim layers, Keogh EQ/EC):
// a bound prunes iff it exceeds ub (1 + g_rel) + g_abs + g_sqrt sqrt(ub).
// g_rel covers a summation order other than the DTW's; g_sqrt the
// reciprocal normalisation (each normalised value is within 3 ulp of the
// reference's division, so by Minkowski the bound moves by at most
// 2 sqrt(lb) * 3u sqrt(m) cmax); g_abs the square of that term.
__device__ __forceinline__ double lb_guard(const SearchParams& p, double ub) {
  return ub * (1.0 + p.guard_rel) + p.guard_abs + p.guard_sqrt * __dsqrt_ru(ub);
}

#ifndef EAPDTW_CB_F32
#define EAPDTW_CB_F32 1  // cumulative-bound prefixes (row thresholds) in FP32, rounded up: cfg4 sweep 34.6 -> 33.5 ms
#endif
#ifndef EAPDTW_LB_F32
#define EAPDTW_LB_F32 1  // LB_Keogh terms in FP32 (guarded): cfg4 sweep 36.7 -> 34.9 ms, cfg3 1.78 -> 1.64
#endif
// FP32 Keogh terms: an upper bound of (float sum) - (true sum T).  A term's
// distance dd moves by at most e = lb_f32_e (its FP32 value and difference
// round once each; the envelope is rounded outward, which only lowers dd), so
// the sum of squares moves by at most 2 e sum(dd) + m e^2 <= 2 e sqrt(m T) +
// m e^2, and the float products / group sums by a relative 12 u.
__device__ __forceinline__ double lb_f32_excess(const SearchParams& p, double T) {
  if (!(T < DBL_MAX)) return 0.0;
  const double dm = static_cast<double>(p.m);
  return __dadd_ru(__dadd_ru(__dmul_ru(12.0 * 0x1.0p-24, T),
                             __dmul_ru(2.0 * p.lb_f32_e, __dsqrt_ru(__dmul_ru(dm, T)))),
                   __dmul_ru(dm, __dmul_ru(p.lb_f32_e, p.lb_f32_e)));
}
__device__ __forceinline__ float fmax3f(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

__device__ __forceinline__ long long vload(const long long* p) {
  return *reinterpret_cast<const volatile long long*>(p);
}
__device__ __forceinline__ unsigned long long vload(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}

#ifdef EAPDTW_PHASE_CLOCKS
#define PHASE_BEGIN() const long long _t0 = clock64()
#define PHASE_END(idx) \
  if (lane == 0) atomicAdd(&p.counters[idx], static_cast<unsigned long long>(clock64() - _t0))
#else
#define PHASE_BEGIN() (void)0
#define PHASE_END(idx) (void)0
#endif

#ifdef EAPDTW_PHASE_CLOCKS
void debug_read_reset(unsigned long long* out8) {
  cudaMemcpyFromSymbol(out8, g_dbg, 16 * sizeof(unsigned long long));
  unsigned long long z[16] = {};
  cudaMemcpyToSymbol(g_dbg, z, sizeof(z));
}
#endif

#ifndef EAPDTW_KIM_PREFETCH
#define EAPDTW_KIM_PREFETCH 1  // 1: prefetch the next LB chunk to L1, 2: to L2
#endif
#ifndef EAPDTW_KIM_CORNER_RSD
#define EAPDTW_KIM_CORNER_RSD 1  // corner LB_Kim by reciprocal too (guarded)
#endif
#ifndef EAPDTW_KIM_F32
#define EAPDTW_KIM_F32 1  // LB_Kim layers in FP32 (guarded): cfg4 sweep 39.2 -> 36.6 ms, total -1.9 ms
#endif
#ifndef EAPDTW_KIM_RSD
#define EAPDTW_KIM_RSD 1  // Kim layers normalised by reciprocal multiplication
#endif
#ifndef EAPDTW_SEARCH_THREADS
#define EAPDTW_SEARCH_THREADS 256
#endif
#ifndef EAPDTW_SEARCH_MIN_BLOCKS
#define EAPDTW_SEARCH_MIN_BLOCKS 2
#endif
constexpr int kSearchMinBlocks = EAPDTW_SEARCH_MIN_BLOCKS;

// AD_K: the exact engine's anti-diagonal window compiled into this
// instantiation (0: strip engine only -- the default search path).
// LP: Algo::left_prune searches (p.prune == 2): every DTW call runs the
// exact left-pruning schedule (no FP32 screen).  GMEM: queries whose per-warp
// buffers exceed shared memory (p.gscratch).  Separate instantiations, so the
// default kernel's code is untouched by either.
template <int AD_K, bool LP = false, bool GMEM = false>
__global__ void __launch_bounds__(EAPDTW_SEARCH_THREADS, kSearchMinBlocks) search_kernel(SearchParams p) {
  extern __shared__ double smem[];
  const int m = p.m;
  const int pad = smem_pad(p.ad_k);
  const size_t plen = padded_len(m, p.ad_k);
  double* qsp = smem + pad;                        // qsp[-pad .. m+1+pad]
  // The Keogh envelope and visiting order stay in global memory: every lane
  // reads the same element (broadcast through L1), which frees shared memory
  // for more resident warps.
  const double2* __restrict__ qul = p.qul;
  const double2* __restrict__ qperm = p.qperm;
  const int* __restrict__ order = p.order;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // per-warp buffer: the DTW row buffer, or the LB_Keogh EQ staging tile
  const size_t wlen = warp_buf_doubles(m, p.ad_k);
  constexpr bool gmem = GMEM;  // long queries: the per-warp buffers in global memory
  double* rowbuf =
      (gmem ? p.gscratch + (static_cast<size_t>(blockIdx.x) * (blockDim.x >> 5) + warp) * wlen
            : smem + plen + static_cast<size_t>(warp) * wlen) + pad;
  int* stacks = reinterpret_cast<int*>(smem + plen +
                                       (gmem ? 0 : static_cast<size_t>(blockDim.x >> 5) * wlen));
  // the query as float (FP32 screens), after the stacks
  float* q32base = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(stacks) +
                                            static_cast<size_t>(blockDim.x >> 5) * kStackBytesPerWarp);
  const float* qsp32 = q32base + kPadR;
  const int q32n = static_cast<int>(q32_len(m));
  // this warp's FP32 probe state: two F32Strip, then two cumulative-bound prefixes
  unsigned char* pstate = reinterpret_cast<unsigned char*>(stacks) + warp * kStackBytesPerWarp +
                          (kStackBytesPerWarp - kProbeStateBytes);
  F32Strip* probe_st = reinterpret_cast<F32Strip*>(pstate);
  // The FP32 engine's row buffer aliases the warp's FP64 one (both engines
  // initialise [0, lc+1] on entry and never depend on the padding contents:
  // out-of-band cells are +inf by the band test).
  float* rowbuf32 = reinterpret_cast<float*>(rowbuf);
  // the FP32 probe's second (reversed-pass) row follows the first
  const int rowbuf32_len = m + 2 + kPadL + kPadR + 8;

  const double INF = d_inf();
  for (int k = threadIdx.x; k < static_cast<int>(plen); k += blockDim.x) {
    const int j = k - pad;
    smem[k] = (j >= 1 && j <= m) ? p.q[j] : INF;
  }
  for (int k = threadIdx.x; k < q32n; k += blockDim.x) {
    const int j = k - kPadR;
    q32base[k] = (j >= 1 && j <= m) ? __double2float_rn(p.q[j]) : f_inf();
  }
  for (int k = lane; k < static_cast<int>(plen); k += 32) rowbuf[k - pad] = INF;
  __syncthreads();

#ifdef EAPDTW_PHASE_CLOCKS
  const long long t_kernel0 = clock64();
#endif
  unsigned long long c_kim = 0, c_eq = 0, c_ec = 0, c_calls = 0, c_aband = 0, c_cells = 0,
                     c_cand = 0, c_ovf = 0, c_scr = 0, c_cells_lane = 0, c_cells32 = 0;
  const double* __restrict__ ref = p.ref;
  const bool prune = p.prune != 0;

  // One exact pruned DTW of candidate `cand` with the whole warp.  teq / tec:
  // the candidate's LB_Keogh EQ / EC totals from the cascade (rounded down),
  // when have_tot.
  auto run_dtw = [&](long long cand, bool have_tot, double teq, double tec) {
    const double cm = p.mean[cand];
    const double cs = p.sd[cand];
    const bool cconst = cs < kMinStddev;
    const double* crow = ref + cand;
    auto rowraw = [&](int r) -> double { return crow[r]; };
    auto rownorm = [&](double x) -> double {
      return cconst ? 0.0 : __ddiv_rn(__dsub_rn(x, cm), cs);
    };
    auto get_ub = [&]() -> double { return prune ? load_ub(p.ub_key) : INF; };
    // tighten_ub (search.cpp:101-113, dtw.cpp:81-86): row i's threshold is
    // ub - cb(k), k = min(i+w, m) - 1, cb(k) a lower bound on the cost of the
    // positions past k that every path still has to visit.  Here cb is the
    // larger of the EQ (per row) and EC (per column) Keogh suffix sums, each
    // total - prefix(k): the totals come with the candidate from the
    // cascade, and each strip extends the prefix by the 32 positions its
    // rows need (one coalesced load per lane, one warp scan).  The terms are
    // the cascade's (reciprocal normalisation); cb is lowered by guard_rel *
    // total for the summation order and by 8 ulp * (T + qmax sqrt(m T)) for
    // the normalisation (each term is off by < 2 dd (|dd| + qmax) * 3 ulp).
    // guard_rel also covers the rounding of the rest of the path.  Liveness
    // only (the strip engine never kills values): the result is still the
    // exact DTW value whenever that is <= ub.
    const bool tight = p.tighten != 0 && have_tot;
    const double rsd = cconst ? 0.0 : __drcp_rn(cs);
    const bool have_ec = p.env != nullptr;
    // EQ / EC contribution of position k (0 past the end)
    auto contrib_eq = [&](int k) -> double {
      if (k >= m) return 0.0;
      const double c = __dmul_rn(__dsub_rn(crow[k], cm), rsd);
      const double2 b = qul[k];
      const double e1 = __dsub_rn(c, b.x), e2 = __dsub_rn(b.y, c);
      const double d1 = e1 > 0.0 ? e1 : (e2 > 0.0 ? e2 : 0.0);
      return __dmul_rn(d1, d1);
    };
    auto contrib_ec = [&](int k) -> double {
      if (k >= m || !have_ec) return 0.0;
      const double2 e = p.env[cand + k];
      const double U = __dmul_rn(__dsub_rn(e.x, cm), rsd);
      const double L = __dmul_rn(__dsub_rn(e.y, cm), rsd);
      const double qk = qsp[k + 1];
      const double f1 = __dsub_rn(qk, U), f2 = __dsub_rn(L, qk);
      const double d2 = f1 > 0.0 ? f1 : (f2 > 0.0 ? f2 : 0.0);
      return __dmul_rn(d2, d2);
    };
    const double tmax = fmax(teq, tec);
    // (p.cb_eps: speculative statistics move each normalised value by up to
    // eps (1 + |c|), hence the sum of the terms by 2 eps (1 + cmax) sqrt(m T))
    const double sq_mt = __dsqrt_rn(static_cast<double>(m) * tmax);
    const double cb_guard =
        p.guard_rel * tmax + 8.0 * 0x1.0p-52 * (tmax + p.qmax * sq_mt) + p.cb_eps * sq_mt;
    // Row i's remaining cost: every path still visits every later row
    // (0-based positions >= i: EQ terms are per candidate position = row),
    // and every column past i+w (0-based >= i+w: EC terms are per query
    // position = column).  So the EQ suffix starts w positions earlier than
    // the reference's single k = min(i+w, m) - 1 (which must also serve EC);
    // the bound is tighter and still sound.  Each strip extends both
    // prefixes by 32 positions (one lane each, one warp scan each).
    // A pass over the REVERSED pair (the FP32 screen's probe, dtw_f32.cuh)
    // sees position k of the pass at the candidate's / query's position
    // m-1-k, so its prefixes run over the positions from the end: the same
    // bound for the mirrored problem.
#if EAPDTW_CB_F32
    // The prefixes as floats: every contribution rounded UP (envelope rounded
    // inward, the distance raised by the FP32 term error lb_f32_e, products and
    // sums rounded up), so total - prefix stays a lower bound of the suffix.
    using cb_t = float;
    const float cb_ef = __double2float_ru(p.lb_f32_e);
    auto cb_add = [](float x, float y) { return __fadd_ru(x, y); };
    auto contrib_eq_c = [&](int k) -> float {
      if (k >= m) return 0.0f;
      const float c = __double2float_rn(__dmul_rn(__dsub_rn(crow[k], cm), rsd));
      const double2 b = qul[k];
      const float U = __double2float_rd(b.x), L = __double2float_ru(b.y);
      const float dd = __fadd_ru(fmax3f(__fsub_ru(c, U), __fsub_ru(L, c), 0.0f), cb_ef);
      return __fmul_ru(dd, dd);
    };
    auto contrib_ec_c = [&](int k) -> float {
      if (k >= m || !have_ec) return 0.0f;
      const double2 e = p.env[cand + k];
      const float U = __double2float_rd(__dmul_rn(__dsub_rn(e.x, cm), rsd));
      const float L = __double2float_ru(__dmul_rn(__dsub_rn(e.y, cm), rsd));
      const float qk = qsp32[k + 1];
      const float dd = __fadd_ru(fmax3f(__fsub_ru(qk, U), __fsub_ru(L, qk), 0.0f), cb_ef);
      return __fmul_ru(dd, dd);
    };
#else
    using cb_t = double;
    auto cb_add = [](double x, double y) { return __dadd_rn(x, y); };
    auto& contrib_eq_c = contrib_eq;
    auto& contrib_ec_c = contrib_ec;
#endif
    struct CbPrefix {
      cb_t eq, ec;
      int end_eq, end_ec;  // the prefixes cover pass positions [0, end) once started (-1: not yet)
    };
    static_assert(2 * sizeof(F32Strip) + 2 * sizeof(CbPrefix) <= kProbeStateBytes, "probe state");
    // (both directions' prefix states in the warp's shared probe state:
    // memory, not registers -- the kernel is at its register budget)
    CbPrefix* cbp = reinterpret_cast<CbPrefix*>(pstate + 2 * sizeof(F32Strip));
    if (lane == 0) cbp[0] = cbp[1] = CbPrefix{cb_t(0), cb_t(0), -1, -1};
    __syncwarp();
    // Both probes' evidence in one bound.  Once the FP32 screen has probed P
    // rows from each end and picked a direction, the dropped probe's frontier
    // row still says something: any path's cells in the P rows that probe
    // covered cost at least the minimum R of that row (its DP runs from the
    // corner to that row; as an FP32 value, at least f32_lower(R) in exact
    // terms, dtw_f32.cuh).  The continuing direction's EQ suffix counts those
    // P rows with their Keogh terms only (their sum is the dropped probe's EQ
    // prefix), so for the rows before them the suffix grows by
    // x = f32_lower(R) - prefix (when positive): every path still pays the
    // Keogh terms of the rows in between plus R.  on_pick (below) subtracts x
    // from the continuing pass's EQ prefix, which adds it to every later
    // suffix at no cost per row; the bound does not hold inside the last P
    // rows, so the screen then stops before them (undecided: the exact
    // engine runs).  Design study (tools/live_study.c): 14% fewer live cells
    // than the probe alone.
    auto rowthr_dir = [&](auto rev_tag, CbPrefix& st, double u, int i, int i0) -> double {
      constexpr bool REV = decltype(rev_tag)::value;
      if (!tight || i0 < 1 + 32 * (p.cb_strip - 1)) return u;
      auto pos = [&](int k) { return REV ? m - 1 - k : k; };
      const int k_eq = i0 - 1, k_ec = i0 + p.w - 1;  // lane 0's positions
      // The EC prefix starts with strip p.cb_ec_strip (default 2): its first
      // use sums the w + 32 positions before the strip's rows (L2 gathers of
      // the candidate's envelope), which the many tasks that die in their
      // first strip then never pay; until then cb is the EQ suffix alone.
      const bool use_ec = have_ec && i0 >= 1 + 32 * (p.cb_ec_strip - 1);
      if (st.end_eq < 0) {  // positions before this strip's first ones
        st.end_eq = min(m, k_eq);
        cb_t eq = 0;
        for (int k = lane; k < st.end_eq; k += 32) eq = cb_add(eq, contrib_eq_c(pos(k)));
        for (int off = 16; off > 0; off >>= 1) eq = cb_add(eq, __shfl_xor_sync(kFull, eq, off));
        st.eq = eq;
      }
      if (use_ec && st.end_ec < 0) {
        st.end_ec = min(m, k_ec);
        cb_t ec = 0;
        // (4 positions per lane in flight: the envelope loads are L2 latency)
        for (int k0 = lane; k0 < st.end_ec; k0 += 128) {
          cb_t t4[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int k = k0 + 32 * u;
            t4[u] = k < st.end_ec ? contrib_ec_c(pos(k)) : cb_t(0);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) ec = cb_add(ec, t4[u]);
        }
        for (int off = 16; off > 0; off >>= 1) ec = cb_add(ec, __shfl_xor_sync(kFull, ec, off));
        st.ec = ec;
      }
      // this strip's rows need prefixes through k_eq + lane and k_ec + lane
      const int ke = k_eq + lane, kc = k_ec + lane;
      cb_t a = 0, b = 0;
      if (ke >= st.end_eq && ke < m) a = contrib_eq_c(pos(ke));
      if (use_ec && kc >= st.end_ec && kc < m) b = contrib_ec_c(pos(kc));
      for (int off = 1; off < 32; off <<= 1) {  // inclusive prefix scans
        const cb_t x = __shfl_up_sync(kFull, a, off);
        const cb_t y = __shfl_up_sync(kFull, b, off);
        if (lane >= off) {
          a = cb_add(a, x);
          b = cb_add(b, y);
        }
      }
      const cb_t peq = cb_add(st.eq, a), pec = cb_add(st.ec, b);
      // the next strip starts where this one's rows end
      const int nxe = min(m, k_eq + 32), nxc = min(m, k_ec + 32);
      if (nxe > st.end_eq) {
        st.eq = __shfl_sync(kFull, peq, min(31, nxe - 1 - k_eq));
        st.end_eq = nxe;
      }
      if (use_ec && nxc > st.end_ec) {
        st.ec = __shfl_sync(kFull, pec, min(31, nxc - 1 - k_ec));
        st.end_ec = nxc;
      }
      if (i >= m) return u;  // the last row: nothing left
      const double ceq = __dsub_rn(teq, static_cast<double>(peq));
      const double cec = use_ec && kc < m - 1 ? __dsub_rn(tec, static_cast<double>(pec)) : 0.0;
      const double cbv = __dsub_rn(fmax(ceq, cec), cb_guard);
      if (!(cbv > 0.0)) return u;
      const double t = __dsub_rn(__dmul_rn(u, 1.0 + p.guard_rel), cbv);
      return t > 0.0 ? t : 0.0;
    };
    auto rowthr = [&](double u, int i, int i0) -> double {
      return rowthr_dir(std::false_type{}, cbp[0], u, i, i0);
    };
    // FP32 screen first (dtw_f32.cuh) once a finite threshold exists: it
    // abandons with a sound, error-inflated threshold; whatever it cannot
    // abandon is evaluated exactly below.
    bool screened = false;
    if (!LP && p.use_f32 && prune && __shfl_sync(kFull, load_ub(p.ub_key), 0) < INF) {
      const F32Guard g{p.f32_a, p.f32_b};
      auto rownorm32 = [&](double x) -> float {
        return cconst ? 0.0f : __double2float_rn(__dmul_rn(__dsub_rn(x, cm), rsd));
      };
      auto rowthr32 = [&](double u, int i, int i0) -> float {
        return f32_threshold(rowthr(u, i, i0), g);
      };
      auto rowthr32_r = [&](double u, int i, int i0) -> float {
        return f32_threshold(rowthr_dir(std::true_type{}, cbp[1], u, i, i0), g);
      };
      auto rowraw_r = [&](int r) -> double { return crow[m - 1 - r]; };
      auto on_pick = [&](bool use_r, float other_vmin) -> bool {
        if (!tight || !p.probe_excess) return false;
        const CbPrefix& o = cbp[use_r ? 0 : 1];  // the dropped direction's prefixes
        if (o.end_eq <= 0 || o.end_eq >= m) return false;
        // rounded down, and less twice the bound's guard for the prefix's own error
        // f32_lower without its division and root: (sqrt(y) - b)^2 >= y - 2 b sqrt(y)
        // >= y (1 - b) - b with y = R / a (2 sqrt(y) <= 1 + y)
        const float y = __fmul_rd(other_vmin, p.f32_ia);
        const float lb = __fsub_rd(__fmul_rd(y, __fsub_rd(1.0f, p.f32_b)), p.f32_b);
        const double x = __dsub_rd(__dsub_rd(static_cast<double>(lb), static_cast<double>(o.eq)),
                                   2.0 * cb_guard);
        if (!(x > 0.0)) return false;
        __syncwarp();
        // (the prefix less at most x: rounded so that it stays an upper bound)
        if (lane == 0) {
#if EAPDTW_CB_F32
          cbp[use_r ? 1 : 0].eq = __fsub_ru(cbp[use_r ? 1 : 0].eq, __double2float_rd(x));
#else
          cbp[use_r ? 1 : 0].eq = __dsub_rd(cbp[use_r ? 1 : 0].eq, x);
#endif
        }
        __syncwarp();
        return true;
      };
      {
        // both directions probed, then the likelier to die (dtw_f32.cuh)
        int st = 0;
        const float r32 = f32_probe_pair<kSearchStepBlock, false>(
            rowraw, rowraw_r, rownorm32, m, qsp32, m, p.w, p.f32_cmax, get_ub, rowthr32,
            rowthr32_r, rowbuf32, rowbuf32 + rowbuf32_len, p.probe_strips, probe_st, c_cells32, st,
            on_pick);
        screened = st == 0 && r32 == f_inf();
      }
      // the cumulative-bound prefixes restart for the exact pass
      if (lane == 0) cbp[0] = CbPrefix{cb_t(0), cb_t(0), -1, -1};
      __syncwarp();
    }
    const double d = screened ? INF
                              : dtw_dispatch<false, LP>(AD_K, rowraw, rownorm, m, qsp, m, p.w,
                                                        get_ub, rowthr, rowbuf, c_cells, c_ovf);
    ++c_calls;
    if (d == INF) {
      ++c_aband;
    } else if (lane == 0) {
      if (p.approx) {
        // Speculative statistics: d is within the guard of the exact value,
        // so guard(d) bounds it from above, and guard(guard(d)) bounds what
        // an approximate evaluation of any candidate at least as good can
        // return: that is the threshold.  The candidate itself is listed for
        // the exact pass (capi.cu); the record only takes exact values.
        const double u2 = lb_guard(p, lb_guard(p, d));
        atomicMin(p.ub_key, static_cast<unsigned long long>(__double_as_longlong(u2)));
        if (!p.ub_only) {
          const unsigned long long at = atomicAdd(p.vcount, 1ull);
          if (at < static_cast<unsigned long long>(p.vcap)) p.vlist[at] = cand;
        }
      } else {
        atomicMin(p.ub_key, static_cast<unsigned long long>(__double_as_longlong(d)));
        // ub_only: d is an upper bound (a narrower band's DTW), a threshold
        // but not an answer
        if (!p.ub_only)
          best_record_update(p.best, d, static_cast<unsigned long long>(cand + p.index_offset));
      }
    }
  };

  // ---- direct mode (the probe, the rank pass's upper-bound wave): every
  //      candidate is a DTW task, claimed one at a time.
  // ---- cascade mode: LB chunks and queued DTW tasks (below).
  // Both modes feed the ONE call site of run_dtw at the bottom of the loop
  // (code size: the kernel is instruction-cache sensitive).
  {
    // ---- cascade mode.  Survivor queue protocol (no CAS retries):
    //   producers reserve slots with atomicAdd(qtail) and fill them;
    //   a consumer takes a slot with atomicAdd(qhead) only when head < tail
    //   was observed, so it may hold a "future" slot that a producer fills a
    //   little later -- meanwhile it keeps producing.  Once every chunk has
    //   been published (chunks_done == nchunks) a future slot beyond the final
    //   tail is void.
    // chunk c covers candidates begin + c*span + lane*stride
    const long long span = p.chunk_span > 0 ? p.chunk_span : 32 * p.stride;
    const long long nlist =
        p.list ? min(static_cast<long long>(vload(p.nlist)), p.list_cap) : 0;
    const long long nchunks = p.list ? (nlist + 31) / 32 : (p.end - p.begin + span - 1) / span;
    bool chunks_left = true, flushed = false;
    long long myslot = -1;
    long long my_next = 0, my_end = 0;  // claimed chunk range
    unsigned long long my_chunks = 0;
    // Per-warp compaction stacks between the tiers (local candidate indices):
    // Kim survivors -> [A] -> EQ -> [B] -> EC -> [C] -> phase-A screen -> queue.
    // A tier runs only on a full warp of candidates (or when flushing), so
    // lanes stay busy although each tier discards most of its input.  Each
    // tier runs in two legs: the first kLbHead positions of order[] (largest
    // |q|: most prunes happen there), then the candidates still pending are
    // re-gathered into full warps [A2], [B2] with their partial sums.
    // Survivors carry their EQ / EC totals (rounded down) to the DTW, for the
    // cumulative-bound row thresholds.
    unsigned char* wbase = reinterpret_cast<unsigned char*>(stacks) + warp * kStackBytesPerWarp;
    int* stkA = reinterpret_cast<int*>(wbase);
    int* stkA2 = stkA + kStack;
    int* stkB = stkA2 + kStack;
    int* stkB2 = stkB + kStack;
    int* stkC = stkB2 + kStack;
    float* teqB = reinterpret_cast<float*>(stkC + kStack);  // B: EQ total
    float* teqB2 = teqB + kStack;                             // B2: EQ total
    float2* totC = reinterpret_cast<float2*>(teqB2 + kStack); // C: (EQ, EC) totals
    double* accA2 = reinterpret_cast<double*>(totC + kStack);
    double* accB2 = accA2 + kStack;
    int nA = 0, nA2 = 0, nB = 0, nB2 = 0, nC = 0;

    // push: ballot-compacted append of the lanes with keep; pop: up to 32
    // entries, lane L gets entry n-take+L (valid iff L < take).
    auto push = [&](int* stk, int& n, bool keep, long long cand, double* acc_arr, double acc,
                    float* f_arr, float f, float2* f2_arr, float2 f2) {
      const unsigned mask = __ballot_sync(kFull, keep);
      if (keep) {
        const int at = n + __popc(mask & ((1u << lane) - 1u));
        stk[at] = static_cast<int>(cand - p.begin);
        if (acc_arr) acc_arr[at] = acc;
        if (f_arr) f_arr[at] = f;
        if (f2_arr) f2_arr[at] = f2;
      }
      n += __popc(mask);
      __syncwarp();
    };
    auto pop = [&](int* stk, int& n, long long& cand, const double* acc_arr, double& acc,
                   const float* f_arr, float& f, const float2* f2_arr, float2& f2) -> bool {
      const int take = min(32, n);
      const bool ok = lane < take;
      const int at = ok ? n - take + lane : 0;
      cand = ok ? p.begin + stk[at] : p.begin;
      acc = (ok && acc_arr) ? acc_arr[at] : 0.0;
      f = (ok && f_arr) ? f_arr[at] : 0.0f;
      f2 = (ok && f2_arr) ? f2_arr[at] : make_float2(0.0f, 0.0f);
      __syncwarp();
      n -= take;
      return ok;
    };
    const float2 z2 = make_float2(0.0f, 0.0f);

    const long long nlist_d =
        p.list ? min(static_cast<long long>(vload(p.nlist)), p.list_cap) : 0;
    // Warp specialisation by scheduler (SMSP = warp slot mod 4): with
    // p.producer_smsp, the warps of SMSP 0 run the lower-bound tiers and take
    // a DTW task only once the queue holds a backlog (or their chunks are
    // done); the other SMSPs drain the queue first.  Each SMSP's instruction
    // cache then holds mostly one of the two code paths (ncu: instruction-
    // fetch stalls were the largest stall reason with every warp mixing both).
    unsigned warp_slot;
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(warp_slot));
    // (The same split by SM -- smid % M == 0 produces, M = 2, 3, 4 -- measured
    // +0.3 to +1 ms on the cfg4 sweep: not kept.)
    const bool producer = p.producer_smsp != 0 && (warp_slot & 3u) == 0u;
    for (;;) {
      long long cand = -1;
      float2 tot = z2;
      bool have_tot = false;
      if (p.direct) {
        unsigned long long c = 0;
        if (lane == 0) c = atomicAdd(p.work, 1ull);
        c = __shfl_sync(kFull, c, 0);
        if (p.list) {  // the candidates come from the list
          if (static_cast<long long>(c) >= nlist_d) break;
          cand = p.list[c];
        } else {
          cand = p.begin + static_cast<long long>(c) * p.stride;
          if (cand >= p.end) break;
        }
        ++c_cand;
        goto dtw_task;
      }
      {
      bool void_slot = false;
      if (lane == 0) {
        if (myslot < 0) {
          const unsigned long long h = vload(p.qhead), t = vload(p.qtail);
          if (h < t && (!producer || !chunks_left || t - h > static_cast<unsigned long long>(p.producer_smsp)))
            myslot = static_cast<long long>(atomicAdd(p.qhead, 1ull));
        }
        if (myslot >= 0) {
          cand = vload(p.queue + myslot);
          if (cand < 0 && flushed &&
              vload(p.chunks_done) == static_cast<unsigned long long>(nchunks) &&
              static_cast<unsigned long long>(myslot) >= vload(p.qtail))
            void_slot = true;
        }
      }
      cand = __shfl_sync(kFull, cand, 0);
      void_slot = __shfl_sync(kFull, void_slot, 0);
      if (cand >= 0) {
        if (lane == 0) {
          __threadfence();
          const unsigned long long raw =
              *reinterpret_cast<const volatile unsigned long long*>(p.qtot + myslot);
          tot = make_float2(__uint_as_float(static_cast<unsigned>(raw)),
                            __uint_as_float(static_cast<unsigned>(raw >> 32)));
        }
        tot.x = __shfl_sync(kFull, tot.x, 0);
        tot.y = __shfl_sync(kFull, tot.y, 0);
        have_tot = p.use_lb != 0;
        myslot = -1;
        goto dtw_task;
      }
      myslot = __shfl_sync(kFull, myslot, 0);
      if (void_slot) break;
      if (flushed) {
        if (myslot < 0) {
          // Nothing of its own left: keep consuming while other warps may
          // still publish survivors (a short list or the sweep's tail would
          // otherwise leave their DTW tasks to a few warps).
          bool done = false;
          if (lane == 0)
            done = vload(p.chunks_done) >= static_cast<unsigned long long>(nchunks) &&
                   vload(p.qhead) >= vload(p.qtail);
          if (__shfl_sync(kFull, done, 0)) break;
          PHASE_BEGIN();
          __nanosleep(256);
          PHASE_END(kClkWait);
        }
        continue;  // claim a new slot, or wait for the pending one to be filled
      }

      PHASE_BEGIN();
      if (chunks_left) {
        // ---- tier 1 on the next chunk of 32 candidates: LB_Kim on the two
        //      aligned extremities (search.cpp:81-87), with the DTW's own IEEE
        //      divisions (exact, so compared without a guard).
        // chunks are claimed kSuperChunk at a time, so the tier stacks hold
        // candidates from a short stretch of the reference (EQ staging below)
        if (my_next >= my_end) {
          unsigned long long c0 = 0;
          if (lane == 0) c0 = atomicAdd(p.work, static_cast<unsigned long long>(kSuperChunk));
          my_next = static_cast<long long>(__shfl_sync(kFull, c0, 0));
          my_end = my_next + kSuperChunk;
        }
        const long long chunk = my_next++;
        if (chunk >= nchunks) {
          chunks_left = false;  // flush the stacks below, then retire
        } else {
          ++my_chunks;
          long long s = p.begin + static_cast<long long>(chunk) * span + lane * p.stride;
          if (p.list) {  // rank pass: the chunk's candidates come from the list
            const long long li = chunk * 32 + lane;
            s = li < nlist ? p.list[li] : p.end;
          }
#if EAPDTW_KIM_PREFETCH
          // pull the next chunk of this claim toward the SM while this one
          // is processed (the Kim tier is memory-latency bound)
          if (!p.list && my_next < my_end && my_next < nchunks) {
            const long long s2 = s + span;
            if (s2 < p.end) {
#if EAPDTW_KIM_PREFETCH == 1
              asm volatile("prefetch.global.L1 [%0];" ::"l"(p.mean + s2));
              asm volatile("prefetch.global.L1 [%0];" ::"l"(p.sd + s2));
              asm volatile("prefetch.global.L1 [%0];" ::"l"(ref + s2));
              asm volatile("prefetch.global.L1 [%0];" ::"l"(ref + s2 + m - 1));
#else
              asm volatile("prefetch.global.L2 [%0];" ::"l"(p.mean + s2));
              asm volatile("prefetch.global.L2 [%0];" ::"l"(p.sd + s2));
              asm volatile("prefetch.global.L2 [%0];" ::"l"(ref + s2));
              asm volatile("prefetch.global.L2 [%0];" ::"l"(ref + s2 + m - 1));
#endif
            }
          }
#endif
          const bool valid = s < p.end;
          if (!valid) s = p.begin;  // loads stay in bounds
          c_cand += __popc(__ballot_sync(kFull, valid));
          bool alive = valid;
          if (p.use_lb && m >= 2 && alive) {
            const double mean = p.mean[s];
            const double sd = p.sd[s];
            const bool constant = sd < kMinStddev;
#if EAPDTW_KIM_CORNER_RSD
            // corners by reciprocal normalisation too: one reciprocal instead
            // of two divisions per candidate; the corner bound is then
            // guarded like the layers
            const double rsd0 = constant ? 0.0 : __drcp_rn(sd);
            const double c0 = __dmul_rn(__dsub_rn(ref[s], mean), rsd0);
            const double cl = __dmul_rn(__dsub_rn(ref[s + m - 1], mean), rsd0);
            const double kim = __dadd_rn(sq_cost(qsp[1], c0), sq_cost(qsp[m], cl));
            const double ub = load_ub(p.ub_key);
            if (kim > lb_guard(p, ub)) {
#else
            const double c0 = constant ? 0.0 : __ddiv_rn(__dsub_rn(ref[s], mean), sd);
            const double cl = constant ? 0.0 : __ddiv_rn(__dsub_rn(ref[s + m - 1], mean), sd);
            const double kim = __dadd_rn(sq_cost(qsp[1], c0), sq_cost(qsp[m], cl));
            const double ub = load_ub(p.ub_key);
            if (kim > ub) {
#endif
              alive = false;
              ++c_kim;
            } else {
              // LB_Kim over L points at each end (the UCR-suite form,
              // extended): a warping path visits one cell of each layer
              // max(i, j) = k from the start and one of each layer from the
              // end, so the minimum cost of each layer adds to the corners.
              // Cells outside the band only lower a minimum.  A sum in another
              // order than the DTW's, so it prunes with the Keogh guard.  L
              // grows with m: the layers cost O(L^2) per candidate and pay
              // off only when what they save (Keogh, DTW) is long.
              auto layers = [&](auto l_tag) -> double {
                constexpr int L = decltype(l_tag)::value;
                double cf[L], cb[L];
#if EAPDTW_KIM_RSD
                // reciprocal normalisation (the bound is guarded anyway, like
                // the Keogh tiers); the corners t = 0 keep their exact values
#if EAPDTW_KIM_CORNER_RSD
                const double rsd = rsd0;
#else
                const double rsd = constant ? 0.0 : __drcp_rn(sd);
#endif
                cf[0] = c0;
                cb[0] = cl;
#pragma unroll
                for (int t = 1; t < L; ++t) {
                  cf[t] = __dmul_rn(__dsub_rn(ref[s + t], mean), rsd);
                  cb[t] = __dmul_rn(__dsub_rn(ref[s + m - 1 - t], mean), rsd);
                }
#else
#pragma unroll
                for (int t = 0; t < L; ++t) {
                  cf[t] = constant ? 0.0 : __ddiv_rn(__dsub_rn(ref[s + t], mean), sd);
                  cb[t] = constant ? 0.0 : __ddiv_rn(__dsub_rn(ref[s + m - 1 - t], mean), sd);
                }
#endif
#if EAPDTW_KIM_F32
                // The layers in FP32 (half the instructions and registers of
                // this unrolled block; the bound is guarded anyway).  A float
                // cost exceeds the exact one by at most ~5.1 u R^2 (u = 2^-24,
                // R = qmax + cmax >= |q - c|: both values and the difference
                // round once each); a layer's minimum inherits that, the sums
                // round down, and p.kim_f32_guard = 72 u R^2 (14 layer terms
                // at L = 8) is taken off the total.
                {
                  float cff[L], cbf[L];
#pragma unroll
                  for (int t = 0; t < L; ++t) {
                    cff[t] = __double2float_rn(cf[t]);
                    cbf[t] = __double2float_rn(cb[t]);
                  }
                  auto sqf = [](float a, float b) {
                    const float d = __fsub_rn(a, b);
                    return __fmul_rn(d, d);
                  };
                  float lbf = 0.0f;
#pragma unroll
                  for (int l = 1; l < L; ++l) {
                    const float qa = qsp32[1 + l], qz = qsp32[m - l];
                    float f = sqf(qa, cff[l]);
                    float bk = sqf(qz, cbf[l]);
#pragma unroll
                    for (int t = 0; t < l; ++t) {
                      f = fmin3f(f, sqf(qa, cff[t]), sqf(qsp32[1 + t], cff[l]));
                      bk = fmin3f(bk, sqf(qz, cbf[t]), sqf(qsp32[m - t], cbf[l]));
                    }
                    lbf = __fadd_rd(lbf, __fadd_rd(f, bk));
                  }
                  return __dadd_rn(kim, __dsub_rd(static_cast<double>(lbf), p.kim_f32_guard));
                }
#endif
                double lb = kim;
#pragma unroll
                for (int l = 1; l < L; ++l) {
                  double f = sq_cost(qsp[1 + l], cf[l]);
                  double bk = sq_cost(qsp[m - l], cb[l]);
#pragma unroll
                  for (int t = 0; t < l; ++t) {
                    f = dmin2(f, dmin2(sq_cost(qsp[1 + l], cf[t]), sq_cost(qsp[1 + t], cf[l])));
                    bk = dmin2(bk, dmin2(sq_cost(qsp[m - l], cb[t]), sq_cost(qsp[m - t], cb[l])));
                  }
                  lb = __dadd_rn(lb, __dadd_rn(f, bk));
                }
                return lb;
              };
              double kim3 = kim;
              if (m >= 2 * kKimLayersLong && m >= kKimLongFrom)
                kim3 = layers(std::integral_constant<int, kKimLayersLong>{});
              else if (m >= 2 * kKimLayers)
                kim3 = layers(std::integral_constant<int, kKimLayers>{});
              if (kim3 > lb_guard(p, ub)) {
                alive = false;
                ++c_kim;
              }
            }
          }
          if (p.use_lb) push(stkA, nA, alive, s, nullptr, 0.0, nullptr, 0.0f, nullptr, z2);
          else push(stkC, nC, alive, s, nullptr, 0.0, nullptr, 0.0f, totC, z2);
        }
      }
      PHASE_END(kClkKim);
      const bool flush = !chunks_left;

      // Early-abandoning LB_Keogh over order[k0, k1) (lower_bounds.cpp:57-88),
      // lane per candidate, continuing the partial sum `acc`; the vote every
      // kLbGroup positions lets the warp stop once every lane has abandoned.
      //   EQ: query envelope qperm[k] (warp-uniform) vs the candidate
      //       normalised by reciprocal multiplication;
      //   EC: query value vs the candidate's (global raw) envelope, normalised.
      // Lanes without a candidate point at p.begin: loads stay in bounds.
      auto lb_range = [&](auto ec_tag, const double* xs, long long s, bool pending,
                          const double mean, const double rsd, double ubg, int k0, int k1,
                          double& acc) -> bool {
        constexpr bool EC = decltype(ec_tag)::value;
        bool alive = pending;
        const double2* es = EC ? p.env + s : nullptr;
#if EAPDTW_LB_F32
        // The terms in FP32 (a third fewer instructions, and FFMA's latency in
        // the accumulation instead of DMUL + DADD): the candidate value (EQ)
        // or the normalised envelope (EC) is formed in FP64 and converted --
        // the envelope outward (upper up, lower down), which only shrinks a
        // term -- and groups of kLbGroup terms accumulate in a float.  What the
        // roundings can ADD to the sum is bounded in lb_f32_excess (applied to
        // the pruning threshold by the caller and taken off the totals).
        const float2* __restrict__ qperm32 = p.qperm32;
        auto term = [&](int k, float& g) {
          const int j = order[k];
          float a, U, L;
          if (!EC) {
            const float2 b = qperm32[k];
            a = __double2float_rn(__dmul_rn(__dsub_rn(xs[j], mean), rsd));
            U = b.x;
            L = b.y;
          } else {
            const double2 e = es[j];
            a = qsp32[j + 1];
            U = __double2float_ru(__dmul_rn(__dsub_rn(e.x, mean), rsd));
            L = __double2float_rd(__dmul_rn(__dsub_rn(e.y, mean), rsd));
          }
          const float dd = fmax3f(__fsub_rn(a, U), __fsub_rn(L, a), 0.0f);
          g = __fmaf_rn(dd, dd, g);
        };
        for (int kb = k0; kb < k1; kb += kLbGroup) {
          float g = 0.0f;
          if (kb + kLbGroup <= k1) {
#pragma unroll
            for (int u = 0; u < kLbGroup; ++u) term(kb + u, g);
          } else {
            for (int k = kb; k < k1; ++k) term(k, g);
          }
          acc = __dadd_rn(acc, static_cast<double>(g));
          if (pending && acc > ubg) {
            pending = false;
            alive = false;
          }
          if (!__any_sync(kFull, pending)) break;
        }
#else
        auto term = [&](int k) {
          const int j = order[k];
          double a, U, L;
          if (!EC) {
            const double2 b = qperm[k];
            a = __dmul_rn(__dsub_rn(xs[j], mean), rsd);
            U = b.x;
            L = b.y;
          } else {
            const double2 e = es[j];
            a = qsp[j + 1];
            U = __dmul_rn(__dsub_rn(e.x, mean), rsd);
            L = __dmul_rn(__dsub_rn(e.y, mean), rsd);
          }
          const double e1 = __dsub_rn(a, U), e2 = __dsub_rn(L, a);
          const double dd = e1 > 0.0 ? e1 : (e2 > 0.0 ? e2 : 0.0);
          acc = __dadd_rn(acc, __dmul_rn(dd, dd));
        };
        // groups of kLbGroup positions: all their loads are in flight together
        for (int kb = k0; kb < k1; kb += kLbGroup) {
          if (kb + kLbGroup <= k1) {
#pragma unroll
            for (int u = 0; u < kLbGroup; ++u) term(kb + u);
          } else {
            for (int k = kb; k < k1; ++k) term(k);
          }
          if (pending && acc > ubg) {
            pending = false;
            alive = false;
          }
          if (!__any_sync(kFull, pending)) break;
        }
#endif
        return alive;
      };

      // ---- tiers 2/3: LB_Keogh EQ (search.cpp:92) then EC (search.cpp:97-99),
      //      prune iff lb > ub*(1+g_rel) + g_abs.
      const int head = min(m, kLbHead);
      const bool have_ec = p.env != nullptr;
      // EC == false: EQ tier (A -> A2 -> B, or C without an EC tier).
      auto stage = [&](auto ec_tag, bool leg2) {
        constexpr bool EC = decltype(ec_tag)::value;
        long long s;
        double acc_d = 0.0;
        float teq = 0.0f;
        float2 unused2;
        float unusedf;
        bool pending;
        if (!EC) {
          pending = leg2 ? pop(stkA2, nA2, s, accA2, acc_d, nullptr, unusedf, nullptr, unused2)
                         : pop(stkA, nA, s, nullptr, acc_d, nullptr, unusedf, nullptr, unused2);
        } else {
          pending = leg2 ? pop(stkB2, nB2, s, accB2, acc_d, teqB2, teq, nullptr, unused2)
                         : pop(stkB, nB, s, nullptr, acc_d, teqB, teq, nullptr, unused2);
        }
        double acc = acc_d;  // a leg-2 partial sum
        const double mean = p.mean[s];
        const double sd = p.sd[s];
        const double rsd = sd < kMinStddev ? 0.0 : __drcp_rn(sd);
#if EAPDTW_LB_F32
        // (prune iff the float sum exceeds what a true sum of ubg can round to)
        const double ubg0 = lb_guard(p, load_ub(p.ub_key));
        const double ubg = __dadd_ru(ubg0, lb_f32_excess(p, ubg0));
#else
        const double ubg = lb_guard(p, load_ub(p.ub_key));
#endif
        // EQ: stage the batch's stretch of the reference in the warp's buffer
        // when it fits, so the order[]-permuted reads hit shared memory
        // instead of L2 (the DP row buffer is free between DTW tasks).
        const double* xs = ref + s;
        if (!EC) {
          int lo = pending ? static_cast<int>(s - p.begin) : INT_MAX;
          int hi = pending ? static_cast<int>(s - p.begin) : INT_MIN;
          for (int off = 16; off > 0; off >>= 1) {
            lo = min(lo, __shfl_xor_sync(kFull, lo, off));
            hi = max(hi, __shfl_xor_sync(kFull, hi, off));
          }
          // p.lb_block_order: order[] visits the first kLbHead positions, then
          // the rest (by descending |q| inside each part), so a leg only needs
          // its own part of the stretch and the staging fits for survivors
          // spread over up to wlen - part positions (all m positions: only
          // for candidates within ~130 of one another at m = 1024)
          const int p0 = p.lb_block_order ? (leg2 ? head : 0) : 0;
          const int part = p.lb_block_order ? (leg2 ? m - head : head) : m;
          const long long len = static_cast<long long>(hi) - lo + part;
#ifdef EAPDTW_PHASE_CLOCKS
          if (lane == 0) atomicAdd(&p.counters[hi >= lo && len <= static_cast<long long>(wlen)
                                                   ? kStageHit : kStageMiss], 1ull);
#endif
          if (!gmem && hi >= lo && len <= static_cast<long long>(wlen)) {
            double* sbuf = rowbuf - pad;
            const double* src = ref + p.begin + lo + p0;
            for (int t = lane; t < static_cast<int>(len); t += 32) sbuf[t] = src[t];
            __syncwarp();
            if (pending) xs = sbuf + (s - p.begin - lo) - p0;
          }
        }
        const bool alive = lb_range(ec_tag, xs, s, pending, mean, rsd, ubg, leg2 ? head : 0,
                                    leg2 ? m : head, acc);
        __syncwarp();
        if (pending && !alive) {
          if (EC) ++c_ec;
          else ++c_eq;
        }
#if EAPDTW_LB_F32
        // rounded down, less what the float terms may have added: a weaker, sound total
        const float tot = fmaxf(0.0f, __double2float_rd(__dsub_rd(acc, lb_f32_excess(p, acc))));
#else
        const float tot = __double2float_rz(acc);  // rounded down: a weaker, sound total
#endif
        if (!leg2 && head < m) {
          if (EC) push(stkB2, nB2, alive, s, accB2, acc, teqB2, teq, nullptr, z2);
          else push(stkA2, nA2, alive, s, accA2, acc, nullptr, 0.0f, nullptr, z2);
        } else if (EC) {
          push(stkC, nC, alive, s, nullptr, 0.0, nullptr, 0.0f, totC, make_float2(teq, tot));
        } else if (have_ec) {
          push(stkB, nB, alive, s, nullptr, 0.0, teqB, tot, nullptr, z2);
        } else {
          push(stkC, nC, alive, s, nullptr, 0.0, nullptr, 0.0f, totC, make_float2(tot, 0.0f));
        }
      };
      // ---- phase A: the first screen_rows DTW rows, lane per candidate (an
      //      exact EAPrunedDTW prefix; a killed candidate is an abandoned
      //      DTW), then publish the survivors (+ totals) to the queue.
      auto screen_stage = [&]() {
        long long s;
        double unused;
        float unusedf;
        float2 tot;
        bool alive = pop(stkC, nC, s, nullptr, unused, nullptr, unusedf, totC, tot);
        if (p.screen_rows > 0) {
          const double mean = p.mean[s];
          const double sd = p.sd[s];
          const bool constant = sd < kMinStddev;
          const double* xs = ref + s;
          auto c_of = [&](int r) -> double {
            return constant ? 0.0 : __ddiv_rn(__dsub_rn(xs[r - 1], mean), sd);
          };
          unsigned nrows = 0;
          const bool killed = screen_prefix<kScreenSlots>(alive, c_of, p.screen_rows, qsp, m,
                                                          p.w, load_ub(p.ub_key), nrows);
          c_cells_lane += static_cast<unsigned long long>(nrows) * kScreenSlots;
          if (killed) {
            alive = false;
            ++c_scr;
          }
        }
        const unsigned mask = __ballot_sync(kFull, alive);
        if (mask) {
          unsigned long long qb = 0;
          if (lane == 0) qb = atomicAdd(p.qtail, static_cast<unsigned long long>(__popc(mask)));
          qb = __shfl_sync(kFull, qb, 0);
          if (alive) {
            const unsigned long long slot = qb + __popc(mask & ((1u << lane) - 1u));
            p.qtot[slot] = tot;
            __threadfence();  // the totals are visible before the slot is
            reinterpret_cast<volatile long long*>(p.queue)[slot] = s;
          }
        }
      };

      // Most downstream ready stage first, so every push lands in a stack
      // holding < 32 entries (capacity kStack = 64); a partial warp runs only
      // when flushing and once everything upstream has drained.
      for (;;) {
        const bool up_a = (nA | nA2) == 0, up_b = up_a && nB == 0, up_c = up_b && nB2 == 0;
        if (nC >= 32 || (flush && nC > 0 && up_c)) {
          PHASE_BEGIN();
          screen_stage();
          PHASE_END(kClkScreen);
        } else {
          // one inlined copy per tier (code size: the kernel is i-cache bound)
          int tier = 0;  // 1: EQ, 2: EC
          bool leg2 = false;
          if (nB2 >= 32 || (flush && nB2 > 0 && up_b)) {
            tier = 2;
            leg2 = true;
          } else if (nB >= 32 || (flush && nB > 0 && up_a)) {
            tier = 2;
          } else if (nA2 >= 32 || (flush && nA2 > 0 && nA == 0)) {
            tier = 1;
            leg2 = true;
          } else if (nA >= 32 || (flush && nA > 0)) {
            tier = 1;
          }
          if (tier == 0) break;
          PHASE_BEGIN();
          if (tier == 2) stage(std::true_type{}, leg2);
          else stage(std::false_type{}, leg2);
          PHASE_END(tier == 2 ? kClkEc : kClkEq);
        }
      }

      if (flush) {
        // Every candidate of this warp's chunks is now published: only then
        // may they count as done (the queue's void-slot rule relies on it).
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(p.chunks_done, my_chunks);
        flushed = true;
      }
      continue;
      }
    dtw_task:
      PHASE_BEGIN();
      run_dtw(cand, have_tot, static_cast<double>(tot.x), static_cast<double>(tot.y));
      PHASE_END(kClkDtw);
    }
  }

  // Per-lane tier counts are summed over the warp; the others are warp-uniform.
  for (int off = 16; off > 0; off >>= 1) {
    c_kim += __shfl_xor_sync(kFull, c_kim, off);
    c_eq += __shfl_xor_sync(kFull, c_eq, off);
    c_ec += __shfl_xor_sync(kFull, c_ec, off);
    c_scr += __shfl_xor_sync(kFull, c_scr, off);
    c_cells_lane += __shfl_xor_sync(kFull, c_cells_lane, off);
  }
  // screened (killed) candidates are DTW evaluations abandoned in phase A
  c_calls += c_scr;
  c_aband += c_scr;
  c_cells += c_cells_lane;
  if (lane == 0) {
    atomicAdd(&p.counters[kCntKim], c_kim);
    atomicAdd(&p.counters[kCntKeoghEq], c_eq);
    atomicAdd(&p.counters[kCntKeoghEc], c_ec);
    atomicAdd(&p.counters[kCntDtwCalls], c_calls);
    atomicAdd(&p.counters[kCntDtwAbandoned], c_aband);
    atomicAdd(&p.counters[kCntCells], c_cells);
    atomicAdd(&p.counters[kCntCandidates], c_cand);
    atomicAdd(&p.counters[kCntOverflows], c_ovf);
    atomicAdd(&p.counters[kCntScreened], c_scr);
    atomicAdd(&p.counters[kCntCellsF32], c_cells32);
#ifdef EAPDTW_PHASE_CLOCKS
    atomicAdd(&p.counters[kClkTotal], static_cast<unsigned long long>(clock64() - t_kernel0));
#endif
  }
}

// ---------------------------------------------------------------------------
// Rank pass: a warm start for the threshold.  A uniform sample (the probe, a
// strided coarse pass) finds a near-final threshold only after ~1e6 exact
// candidates; ranking every S-th candidate by its layered LB_Kim and running
// the cascade over the ~k most promising ones finds a better one for less
// (DESIGN.md section 6).  The bound here only ranks: no soundness needed.
// ---------------------------------------------------------------------------
template <int L>
__device__ double kim_layers_rank(const double* __restrict__ ref, long long s, int m, double mean,
                                  double sd, const double* __restrict__ q1) {
  const bool constant = sd < kMinStddev;
  const double rsd = constant ? 0.0 : __drcp_rn(sd);
  double cf[L], cb[L];
#pragma unroll
  for (int t = 0; t < L; ++t) {
    cf[t] = __dmul_rn(__dsub_rn(ref[s + t], mean), rsd);
    cb[t] = __dmul_rn(__dsub_rn(ref[s + m - 1 - t], mean), rsd);
  }
  double lb = __dadd_rn(sq_cost(q1[1], cf[0]), sq_cost(q1[m], cb[0]));
#pragma unroll
  for (int l = 1; l < L; ++l) {
    double f = sq_cost(q1[1 + l], cf[l]);
    double bk = sq_cost(q1[m - l], cb[l]);
#pragma unroll
    for (int t = 0; t < l; ++t) {
      f = dmin2(f, dmin2(sq_cost(q1[1 + l], cf[t]), sq_cost(q1[1 + t], cf[l])));
      bk = dmin2(bk, dmin2(sq_cost(q1[m - l], cb[t]), sq_cost(q1[m - t], cb[l])));
    }
    lb = __dadd_rn(lb, __dadd_rn(f, bk));
  }
  return lb;
}

constexpr int kRankBins = 1 << 16;  // float bits >> 15 of a non-negative bound

__global__ void __launch_bounds__(256) rank_kernel(SearchParams p, long long S, long long nsamp,
                                                   float* __restrict__ lbv,
                                                   unsigned* __restrict__ hist) {
  const int m = p.m;
  const int L = min(m / 2, m >= kKimLongFrom ? kKimLayersLong : kKimLayers);
  for (long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; k < nsamp;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long s = p.begin + k * S;
    const double mean = p.mean[s], sd = p.sd[s];
    double lb;
    if (L >= 8) lb = kim_layers_rank<8>(p.ref, s, m, mean, sd, p.q);
    else if (L >= 3) lb = kim_layers_rank<3>(p.ref, s, m, mean, sd, p.q);
    else lb = kim_layers_rank<1>(p.ref, s, m, mean, sd, p.q);
    const float f = fminf(__double2float_rd(lb), 3.0e38f);
    lbv[k] = f;
    atomicAdd(&hist[__float_as_uint(f) >> 15], 1u);
  }
}

// One block: the first bin where the cumulative count reaches k; *thr = the
// first float-bit pattern past it (all candidates when fewer than k).
__global__ void __launch_bounds__(1024) rank_threshold_kernel(const unsigned* __restrict__ hist,
                                                              long long k, unsigned* thr) {
  __shared__ unsigned long long part[1024];
  constexpr int per = kRankBins / 1024;
  const int t = threadIdx.x;
  unsigned long long c = 0;
  for (int b = 0; b < per; ++b) c += hist[t * per + b];
  part[t] = c;
  __syncthreads();
  if (t == 0) {
    unsigned long long acc = 0;
    unsigned out = 0xffffffffu;
    for (int i = 0; i < 1024 && out == 0xffffffffu; ++i) {
      if (acc + part[i] >= static_cast<unsigned long long>(k)) {
        for (int b = 0; b < per; ++b) {
          acc += hist[i * per + b];
          if (acc >= static_cast<unsigned long long>(k)) {
            out = static_cast<unsigned>(i * per + b + 1) << 15;
            break;
          }
        }
      } else {
        acc += part[i];
      }
    }
    *thr = out;
  }
}

__global__ void __launch_bounds__(256) rank_select_kernel(const float* __restrict__ lbv,
                                                          long long nsamp, long long begin,
                                                          long long S, const unsigned* thr_lo,
                                                          const unsigned* thr,
                                                          long long cap, long long* list,
                                                          unsigned long long* nlist) {
  const unsigned th = *thr, tl = thr_lo ? *thr_lo : 0u;
  const int lane = threadIdx.x & 31;
  for (long long k0 = static_cast<long long>(blockIdx.x) * blockDim.x; k0 < nsamp;
       k0 += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long k = k0 + threadIdx.x;
    const bool sel = k < nsamp && __float_as_uint(lbv[k]) < th && __float_as_uint(lbv[k]) >= tl;
    const unsigned mask = __ballot_sync(kFull, sel);
    if (!mask) continue;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(nlist, static_cast<unsigned long long>(__popc(mask)));
    base = __shfl_sync(kFull, base, 0);
    const unsigned long long at = base + __popc(mask & ((1u << lane) - 1u));
    if (sel && at < static_cast<unsigned long long>(cap)) list[at] = begin + k * S;
  }
}

size_t rank_scratch_bytes(long long ncand, long long S) {
  const long long nsamp = (ncand + S - 1) / S;
  return static_cast<size_t>(nsamp) * 4 + kRankBins * 4 + 64;
}

cudaError_t launch_rank(const SearchParams& p, long long S, void* scratch, cudaStream_t stream) {
  const long long nsamp = (p.end - p.begin + S - 1) / S;
  if (nsamp <= 0) return cudaSuccess;
  unsigned* hist = static_cast<unsigned*>(scratch);
  float* lbv = reinterpret_cast<float*>(hist + kRankBins + 16);
  cudaError_t e = cudaMemsetAsync(hist, 0, (kRankBins + 16) * 4, stream);
  if (e != cudaSuccess) return e;
  const int blocks = static_cast<int>(std::min<long long>((nsamp + 255) / 256, 148LL * 8));
  rank_kernel<<<blocks, 256, 0, stream>>>(p, S, nsamp, lbv, hist);
  return cudaGetLastError();
}

cudaError_t launch_rank_select(const SearchParams& p, long long S, int wave, long long k,
                               long long cap, void* scratch, long long* list,
                               unsigned long long* nlist, cudaStream_t stream) {
  const long long nsamp = (p.end - p.begin + S - 1) / S;
  if (nsamp <= 0) return cudaSuccess;
  unsigned* hist = static_cast<unsigned*>(scratch);
  unsigned* thr = hist + kRankBins;  // 16 slots: one threshold per wave
  const float* lbv = reinterpret_cast<const float*>(hist + kRankBins + 16);
  cudaError_t e = cudaMemsetAsync(nlist, 0, 8, stream);
  if (e != cudaSuccess) return e;
  rank_threshold_kernel<<<1, 1024, 0, stream>>>(hist, k, thr + wave);
  const int blocks = static_cast<int>(std::min<long long>((nsamp + 255) / 256, 148LL * 8));
  rank_select_kernel<<<blocks, 256, 0, stream>>>(lbv, nsamp, p.begin, S,
                                                 wave > 0 ? thr + wave - 1 : nullptr, thr + wave,
                                                 cap, list, nlist);
  return cudaGetLastError();
}

int search_blocks_per_sm_by_regs() { return kSearchMinBlocks; }

cudaError_t launch_search(const SearchParams& p, int blocks, int warps, cudaStream_t stream) {
  const size_t smem = search_smem_bytes(p.m, warps, p.ad_k, p.gscratch != nullptr);
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(kern), smem);
    if (e != cudaSuccess) return e;
    kern<<<blocks, warps * 32, smem, stream>>>(p);
    return cudaGetLastError();
  };
  if (p.gscratch) return p.prune == 2 ? go(search_kernel<0, true, true>) : go(search_kernel<0, false, true>);
  if (p.prune == 2) return go(search_kernel<0, true>);
  switch (p.ad_k) {
    case 1: return go(search_kernel<1>);
    case 3: return go(search_kernel<3>);
    case 5: return go(search_kernel<5>);
    default: return go(search_kernel<0>);
  }
}

// ---------------------------------------------------------------------------
// Pairwise kernel: warp per pair.  Drop-in for ea_pruned_dtw_windowed /
// dtw_windowed (dtw.cpp:316-396) over a batch; the caller has oriented the
// pair (longer series on rows) and resolved effective_window.
// ---------------------------------------------------------------------------
template <bool WITH_CB, bool LEFT>
__global__ void __launch_bounds__(256) pairwise_kernel(PairParams p) {
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const int lc = p.lc;
  const int pad = smem_pad(p.ad_k);
  const size_t plen = padded_len(max(lc, p.lr), p.ad_k);
  // padded, 1-based; in global scratch for series too long for shared memory
  double* colsp = (p.gscratch ? p.gscratch + (static_cast<size_t>(blockIdx.x) * wpb + warp) * 2 * plen
                              : smem + static_cast<size_t>(warp) * 2 * plen) + pad;
  double* rowbuf = colsp + plen;
  const double INF = d_inf();
  unsigned long long cells = 0, ovf = 0;
  for (int k = lane; k < static_cast<int>(plen); k += 32) {
    colsp[k - pad] = INF;
    rowbuf[k - pad] = INF;
  }
  __syncwarp();
  for (long long pr = static_cast<long long>(blockIdx.x) * wpb + warp; pr < p.npairs;
       pr += static_cast<long long>(gridDim.x) * wpb) {
    const double* rows = p.rows + pr * p.row_stride;
    const double* cg = p.cols + pr * p.col_stride;
    for (int k = lane; k < lc; k += 32) colsp[k + 1] = cg[k];
    __syncwarp();
    const double ub0 = p.ub ? p.ub[pr] : INF;
    auto rowraw = [&](int r) -> double { return rows[r]; };
    auto rownorm = [](double x) -> double { return x; };
    auto get_ub = [&]() -> double { return p.prune ? ub0 : INF; };
    const double* cb = WITH_CB ? p.cb + pr * p.lr : nullptr;
    const int lr = p.lr, w = p.w;
    // row_threshold (dtw.cpp:81-86): ub - cb[min(i+w, lr) - 1], clamped at 0.
    auto rowthr = [&](double u, int i, int) -> double {
      if (!WITH_CB || i > lr) return u;
      const int k = min(i + w, lr);
      const double t = __dsub_rn(u, cb[k - 1]);
      return t > 0.0 ? t : 0.0;
    };
    const double d = dtw_dispatch<WITH_CB, LEFT>(p.ad_k, rowraw, rownorm, lr, colsp, lc, w, get_ub,
                                           rowthr, rowbuf, cells, ovf);
    if (lane == 0) p.out[pr] = d;
    __syncwarp();
  }
  if (lane == 0 && p.cells) atomicAdd(p.cells, cells);
}

// Shape of a pairwise launch: warps per block, blocks, and whether the
// per-warp buffers (2 padded series of max(lr, lc)) fit shared memory.
static void pairwise_shape(const PairParams& p, int& warps, int& blocks, bool& gmem) {
  warps = 8;
  const size_t plen = padded_len(max(p.lc, p.lr), p.ad_k);
  while (warps > 1 && static_cast<size_t>(warps) * 2 * plen * 8 > 200 * 1024) warps /= 2;
  gmem = static_cast<size_t>(warps) * 2 * plen * 8 > 200 * 1024;
  if (gmem) warps = 8;
  const long long need = (p.npairs + warps - 1) / warps;
  blocks = static_cast<int>(min(need, gmem ? 148LL * 4 : 148LL * 32));
}

size_t pairwise_gscratch_doubles(const PairParams& p) {
  int warps, blocks;
  bool gmem;
  pairwise_shape(p, warps, blocks, gmem);
  return gmem ? static_cast<size_t>(blocks) * warps * 2 * padded_len(max(p.lc, p.lr), p.ad_k) : 0;
}

cudaError_t launch_pairwise(const PairParams& p, cudaStream_t stream) {
  int warps, blocks;
  bool gmem;
  pairwise_shape(p, warps, blocks, gmem);
  if (gmem && !p.gscratch) return cudaErrorInvalidValue;
  const size_t plen = padded_len(max(p.lc, p.lr), p.ad_k);
  const size_t smem = gmem ? 0 : static_cast<size_t>(warps) * 2 * plen * sizeof(double);
  auto go = [&](auto kern) -> cudaError_t {
    const cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(kern), smem);
    if (e != cudaSuccess) return e;
    kern<<<blocks, warps * 32, smem, stream>>>(p);
    return cudaGetLastError();
  };
  if (p.prune == 2) return go(pairwise_kernel<false, true>);  // left pruning only
  return p.cb ? go(pairwise_kernel<true, false>) : go(pairwise_kernel<false, false>);
}

// ---------------------------------------------------------------------------
// Batched NN1 (cfg5): per query a running cutoff over the database, the
// harness loop of SURVEY.md 3.3 (ea_pruned_dtw(db[k], q, bsf), dtw.cpp:364-368).
// Block = (query, database split); warps claim database rows in order; an
// exact LB_Kim (first/last, valid for any band) gates the DTW.
// ---------------------------------------------------------------------------
// Layered LB_Kim over raw (already normalised) series: the first and last
// LL points of the row against the query (qsp 1-based), see search_kernel.
template <int LL>
__device__ double kim_layers_raw(const double* __restrict__ rw, int L, const double* qsp) {
  double cf[LL], cb[LL];
#pragma unroll
  for (int t = 0; t < LL; ++t) {
    cf[t] = rw[t];
    cb[t] = rw[L - 1 - t];
  }
  double lb = __dadd_rn(sq_cost(qsp[1], cf[0]), sq_cost(qsp[L], cb[0]));
#pragma unroll
  for (int l = 1; l < LL; ++l) {
    double f = sq_cost(qsp[1 + l], cf[l]);
    double bk = sq_cost(qsp[L - l], cb[l]);
#pragma unroll
    for (int t = 0; t < l; ++t) {
      f = dmin2(f, dmin2(sq_cost(qsp[1 + l], cf[t]), sq_cost(qsp[1 + t], cf[l])));
      bk = dmin2(bk, dmin2(sq_cost(qsp[L - l], cb[t]), sq_cost(qsp[L - t], cb[l])));
    }
    lb = __dadd_rn(lb, __dadd_rn(f, bk));
  }
  return lb;
}

#ifndef EAPDTW_NN1_MINB
#define EAPDTW_NN1_MINB 4  // 4 blocks/SM (64 registers, spills off the step loop): cfg5 -2% vs 3, 2: +17%
#endif
// Per-warp buffer of nn1_kernel (doubles): the exact engine's row, aliased by
// the FP32 screen's two float rows (forward and reversed pass).
static __host__ __device__ inline size_t nn1_warp_doubles(int len, int ad_k) {
  return padded_len(len, ad_k) + 64;
}

__global__ void __launch_bounds__(256, EAPDTW_NN1_MINB) nn1_kernel(Nn1Params p) {
  extern __shared__ double smem[];
  __shared__ unsigned long long s_next;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int L = p.len;
  const int pad = smem_pad(p.ad_k);
  const size_t plen = padded_len(L, p.ad_k);
  const size_t wlen = nn1_warp_doubles(L, p.ad_k);
  const long long qi = blockIdx.x / p.splits;
  const int part = blockIdx.x % p.splits;
  const long long k0 = p.nd * part / p.splits, k1 = p.nd * (part + 1) / p.splits;
  __shared__ int s_qbig;  // some |q| > f32_cmax: no FP32 screen for this query
  double* qsp = smem + pad;  // padded, 1-based
  double* rowbuf = smem + plen + static_cast<size_t>(warp) * wlen + pad;
  float* q32base = reinterpret_cast<float*>(smem + plen + static_cast<size_t>(blockDim.x / 32) * wlen);
  const float* qsp32 = q32base + kPadR;
  const int q32n = static_cast<int>(q32_len(L));
  float* rowbuf32 = reinterpret_cast<float*>(rowbuf);  // aliases the FP64 row (dtw_f32.cuh)
  // this warp's FP32 probe state (two F32Strip), after the float query
  F32Strip* probe_st = reinterpret_cast<F32Strip*>(
                           reinterpret_cast<unsigned char*>(q32base) + (q32_len(L) * 4 + 15) / 16 * 16) +
                       2 * warp;
  const double INF = d_inf();
  if (threadIdx.x == 0) {
    s_next = 0;
    s_qbig = 0;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < static_cast<int>(plen); k += blockDim.x) {
    const int j = k - pad;
    const double qv = (j >= 1 && j <= L) ? p.queries[qi * L + j - 1] : INF;
    smem[k] = qv;
    if (j >= 1 && j <= L && !(fabs(qv) <= static_cast<double>(p.f32_cmax))) s_qbig = 1;
  }
  for (int k = threadIdx.x; k < q32n; k += blockDim.x) {
    const int j = k - kPadR;
    q32base[k] = (j >= 1 && j <= L) ? __double2float_rn(p.queries[qi * L + j - 1]) : f_inf();
  }
  for (int k = lane; k < static_cast<int>(plen); k += 32) rowbuf[k - pad] = INF;
  __syncthreads();
  const bool use_f32 = p.use_f32 != 0 && s_qbig == 0;
  const F32Guard g{p.f32_a, p.f32_b};
  unsigned long long* key = p.ub_keys + qi;
  unsigned long long cells = 0, cells32 = 0, calls = 0, ovf = 0;
  // Rows are claimed 32 at a time: lane L screens row kb+L with LB_Kim_FL
  // (lower_bounds.cpp:51-55, exact, unguarded) and the layered LB_Kim (any
  // band; another summation order, so guarded like the search's), then the
  // warp evaluates the survivors in index order.
  const int KL = L >= 16 ? 8 : (L >= 6 ? 3 : 1);
  // Warm start: each warp first evaluates the row with the smallest layered
  // LB_Kim among its 1/8 of the block's rows, so the running cutoff starts
  // near its final value (the main loop skips those rows).
  __shared__ long long s_warm[32];
  long long my_warm = -1;
  if (p.warm && KL > 1) {
    double bl = INF;
    long long bk = -1;
    const int nw = blockDim.x >> 5;
    for (long long kk = k0 + warp * 32 + lane; kk < k1; kk += static_cast<long long>(nw) * 32) {
      const double* rw = p.db + kk * L;
      const double lb = KL == 8 ? kim_layers_raw<8>(rw, L, qsp) : kim_layers_raw<3>(rw, L, qsp);
      if (lb < bl) {
        bl = lb;
        bk = kk;
      }
    }
    for (int off = 16; off > 0; off >>= 1) {
      const double ol = __shfl_xor_sync(kFull, bl, off);
      const long long ok = __shfl_xor_sync(kFull, bk, off);
      if (ol < bl || (ol == bl && ok >= 0 && (bk < 0 || ok < bk))) {
        bl = ol;
        bk = ok;
      }
    }
    my_warm = bk;
    if (lane == 0) s_warm[warp] = bk;
  } else if (lane == 0) {
    s_warm[warp] = -1;
  }
  __syncthreads();
  const int nwarm = p.warm && KL > 1 ? static_cast<int>(blockDim.x >> 5) : 0;
  bool warm_pending = my_warm >= 0;
  for (;;) {
    long long kb;
    unsigned surv;
    if (warm_pending) {  // this warp's warm-start row, alone
      warm_pending = false;
      kb = my_warm;
      surv = 1u;
    } else {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(&s_next, 32ull);
    t = __shfl_sync(kFull, t, 0);
    kb = k0 + static_cast<long long>(t);
    if (kb >= k1) break;
    {
      const long long kk = kb + lane;
      bool keep = kk < k1;
      if (keep && L >= 2) {
        const double* rw = p.db + kk * L;
        const double ubl = load_ub(key);
        const double kim = __dadd_rn(sq_cost(qsp[1], rw[0]), sq_cost(qsp[L], rw[L - 1]));
        if (kim > ubl) {
          keep = false;
        } else if (KL > 1) {
          double lb;
          if (KL == 8) lb = kim_layers_raw<8>(rw, L, qsp);
          else lb = kim_layers_raw<3>(rw, L, qsp);
          if (lb > ubl * (1.0 + p.guard_rel) + p.guard_abs) keep = false;
        }
      }
      for (int w2 = 0; w2 < nwarm; ++w2)  // warm-start rows are done already
        if (s_warm[w2] == kk) keep = false;
      surv = __ballot_sync(kFull, keep);
    }
    }
    for (; surv; surv &= surv - 1) {
    const long long k = kb + (__ffs(surv) - 1);
    const double* row = p.db + k * L;
    // warp-uniform threshold (lanes need not load in lockstep)
    const double ub = __shfl_sync(kFull, load_ub(key), 0);
    if (L >= 2) {  // LB_Kim_FL again with the current threshold (exact)
      const double kim = __dadd_rn(sq_cost(qsp[1], row[0]), sq_cost(qsp[L], row[L - 1]));
      if (kim > ub) continue;
    }
    auto rowraw = [&](int r) -> double { return row[r]; };
    auto rownorm = [](double x) -> double { return x; };
    auto get_ub = [&]() -> double { return load_ub(key); };
    auto rowthr = [](double u, int, int) -> double { return u; };
    bool screened = false;
    if (use_f32 && __shfl_sync(kFull, ub, 0) < INF) {  // FP32 screen (dtw_f32.cuh)
      auto rownorm32 = [](double x) -> float { return __double2float_rn(x); };
      auto rowthr32 = [&](double u, int, int) -> float { return f32_threshold(u, g); };
      {
        // both directions probed, then the likelier to die (dtw_f32.cuh)
        auto rowraw_r = [&](int r) -> double { return row[L - 1 - r]; };
        int st = 0;
        const float r32 = f32_probe_pair<kNn1StepBlock, true>(
            rowraw, rowraw_r, rownorm32, L, qsp32, L, p.w, p.f32_cmax, get_ub, rowthr32, rowthr32,
            rowbuf32, rowbuf32 + (L + 2 + kPadL + kPadR + 8), p.probe_strips, probe_st, cells32, st);
        screened = st == 0 && r32 == f_inf();
      }
      __syncwarp();
    }
    const double d = screened ? INF
                              : dtw_dispatch<false>(p.ad_k, rowraw, rownorm, L, qsp, L, p.w,
                                                    get_ub, rowthr, rowbuf, cells, ovf);
    ++calls;
    if (d != INF && lane == 0) {
      atomicMin(key, static_cast<unsigned long long>(__double_as_longlong(d)));
      best_record_update(p.best + qi, d, static_cast<unsigned long long>(k + p.index_offset));
    }
    }
  }
  if (lane == 0) {
    atomicAdd(p.cells, cells);
    atomicAdd(p.cells + 1, cells32);
    atomicAdd(p.dtw_calls, calls);
  }
}

cudaError_t launch_nn1(const Nn1Params& p, cudaStream_t stream) {
  // 8 warps per block, fewer for long series (each warp's row buffer is in
  // shared memory with the block's query)
  int warps = 8;
  auto smem_of = [&](int wv) {
    return padded_len(p.len, p.ad_k) * sizeof(double) +
           static_cast<size_t>(wv) * nn1_warp_doubles(p.len, p.ad_k) * sizeof(double) +
           (q32_len(p.len) * sizeof(float) + 15) / 16 * 16 +
           static_cast<size_t>(wv) * 2 * sizeof(F32Strip);
  };
  while (warps > 1 && smem_of(warps) > 200 * 1024) warps /= 2;
  const size_t smem = smem_of(warps);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  const long long blocks = p.nq * p.splits;
  cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(nn1_kernel), smem);
  if (e != cudaSuccess) return e;
  nn1_kernel<<<static_cast<unsigned>(blocks), warps * 32, smem, stream>>>(p);
  return cudaGetLastError();
}

__global__ void init_best_kernel(BestRecord* rec, unsigned long long* keys, long long count) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < count) {
    rec[i].d = d_inf();
    rec[i].idx = ~0ull;
    if (keys) keys[i] = 0x7ff0000000000000ull;
  }
}

cudaError_t launch_init_best(BestRecord* rec, unsigned long long* keys, long long count,
                             cudaStream_t stream) {
  init_best_kernel<<<static_cast<unsigned>((count + 255) / 256), 256, 0, stream>>>(rec, keys, count);
  return cudaGetLastError();
}

// Series validation (series.hpp:24-31) for references copied from the host:
// one streaming pass sets *flag if any sample is non-finite.
__global__ void check_finite_kernel(const double* __restrict__ x, long long n,
                                    unsigned long long* flag) {
  bool bad = false;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x[i]));
    bad |= (b & 0x7ff0000000000000ull) == 0x7ff0000000000000ull;
  }
  if (__any_sync(kFull, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1ull);
}

cudaError_t launch_check_finite(const double* x, long long n, unsigned long long* flag,
                                cudaStream_t stream) {
  const long long blocks = std::min<long long>((n + 255) / 256, 148LL * 16);
  check_finite_kernel<<<static_cast<unsigned>(std::max<long long>(1, blocks)), 256, 0, stream>>>(x, n, flag);
  return cudaGetLastError();
}

// FP64 issue-rate probe: 8 independent DADD chains per thread; used by the
// bench to measure the FP64 pipe peak that the DTW roofline is quoted against.
__global__ void fp64_probe_kernel(double* sink, int iters) {
  double a = 1e-3 * (threadIdx.x + 1);
  double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
  for (int i = 0; i < iters; ++i) {
    x0 = __dadd_rn(x0, a); x1 = __dadd_rn(x1, a); x2 = __dadd_rn(x2, a); x3 = __dadd_rn(x3, a);
    x4 = __dadd_rn(x4, a); x5 = __dadd_rn(x5, a); x6 = __dadd_rn(x6, a); x7 = __dadd_rn(x7, a);
  }
  const double r = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (r == 0.123456789) sink[threadIdx.x] = r;  // keep the chains alive
}

cudaError_t launch_fp64_probe(double* sink, int blocks, int iters, cudaStream_t stream) {
  fp64_probe_kernel<<<blocks, 256, 0, stream>>>(sink, iters);
  return cudaGetLastError();
}

// FP32 issue-rate probe (the roofline of the FP32 screening engine): 8
// independent FADD chains per thread.
__global__ void fp32_probe_kernel(float* sink, int iters) {
  const float a = 1e-3f * (threadIdx.x + 1);
  float x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
  for (int i = 0; i < iters; ++i) {
    x0 = __fadd_rn(x0, a); x1 = __fadd_rn(x1, a); x2 = __fadd_rn(x2, a); x3 = __fadd_rn(x3, a);
    x4 = __fadd_rn(x4, a); x5 = __fadd_rn(x5, a); x6 = __fadd_rn(x6, a); x7 = __fadd_rn(x7, a);
  }
  const float r = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (r == 0.123456789f) sink[threadIdx.x] = r;  // keep the chains alive
}

cudaError_t launch_fp32_probe(float* sink, int blocks, int iters, cudaStream_t stream) {
  fp32_probe_kernel<<<blocks, 256, 0, stream>>>(sink, iters);
  return cudaGetLastError();
}

}  // namespace eapdtw_b200
