// Microbenchmark: the stats chain's inner loop (kernels.cu stats_chain_kernel)
// in isolation, one warp of 32 chains, rows in shared memory: cycles/slide
// for variants of the load / store pattern.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kRow = 66, kTile = 64;

template <int VAR>  // 0: kernel loop (prefetch + STS); 1: no STS; 2: no prefetch; 3: unrolled 2 batches;
                   // 4: 2-batch unroll, squares of the next batch computed during this one
__global__ void chain(int tiles, double* out, long long* cyc, int active) {
  extern __shared__ __align__(16) double dsm[];
  double* rin_s = dsm;
  double* rout_s = dsm + 32 * kRow;
  double* acc_s = dsm + 64 * kRow;
  const int lane = threadIdx.x;
  for (int i = lane; i < 32 * kRow; i += 32) {
    rin_s[i] = 1.0 + 1e-3 * i;
    rout_s[i] = 0.5 + 1e-3 * i;
  }
  __syncwarp();
  double sum = lane, sq = lane;
  const double* rin = rin_s + lane * kRow;
  const double* rout = rout_s + lane * kRow;
  double* as = acc_s + lane * kRow;
  double* aq = acc_s + (32 + lane) * kRow;
  long long t0 = clock64();
  if (lane < active)
  for (int t = 0; t < tiles; ++t) {
    double ci[10], co[10];
    auto load = [&](int k, double* vi, double* vo) {
#pragma unroll
      for (int u = 0; u < 5; ++u) {
        const double2 a = *reinterpret_cast<const double2*>(rin + k + 2 * u);
        const double2 c = *reinterpret_cast<const double2*>(rout + k + 2 * u);
        vi[2 * u] = a.x; vi[2 * u + 1] = a.y; vo[2 * u] = c.x; vo[2 * u + 1] = c.y;
      }
    };
    auto batch = [&](int k, const double* vi, const double* vo) {
      double ps[8], pq[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double xi = vi[u + 1], xo = vo[u + 1];
        sum = __dsub_rn(__dadd_rn(sum, xi), xo);
        sq = __dsub_rn(__dadd_rn(sq, __dmul_rn(xi, xi)), __dmul_rn(xo, xo));
        ps[u] = sum; pq[u] = sq;
      }
      if (VAR != 1) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          *reinterpret_cast<double2*>(as + k + 2 * u) = make_double2(ps[2 * u], ps[2 * u + 1]);
          *reinterpret_cast<double2*>(aq + k + 2 * u) = make_double2(pq[2 * u], pq[2 * u + 1]);
        }
      }
    };
    auto batch_sq = [&](int k, const double* vi, const double* vo, const double* qi, const double* qo) {
      double ps[8], pq[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        sum = __dsub_rn(__dadd_rn(sum, vi[u + 1]), vo[u + 1]);
        sq = __dsub_rn(__dadd_rn(sq, qi[u]), qo[u]);
        ps[u] = sum; pq[u] = sq;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        *reinterpret_cast<double2*>(as + k + 2 * u) = make_double2(ps[2 * u], ps[2 * u + 1]);
        *reinterpret_cast<double2*>(aq + k + 2 * u) = make_double2(pq[2 * u], pq[2 * u + 1]);
      }
    };
    auto squares = [&](const double* vi, const double* vo, double* qi, double* qo) {
#pragma unroll
      for (int u = 0; u < 8; ++u) { qi[u] = __dmul_rn(vi[u + 1], vi[u + 1]); qo[u] = __dmul_rn(vo[u + 1], vo[u + 1]); }
    };
    auto run_defer = [&](int k, const double* vi, const double* vo, const double* qi, const double* qo,
                         double* ps, double* pq, int kprev, const double* pps, const double* ppq) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        sum = __dsub_rn(__dadd_rn(sum, vi[u + 1]), vo[u + 1]);
        sq = __dsub_rn(__dadd_rn(sq, qi[u]), qo[u]);
        ps[u] = sum; pq[u] = sq;
        if (kprev >= 0 && (u & 1)) {  // previous batch's results, long ready
          const int w = u >> 1;
          *reinterpret_cast<double2*>(as + kprev + 2 * w) = make_double2(pps[2 * w], pps[2 * w + 1]);
          *reinterpret_cast<double2*>(aq + kprev + 2 * w) = make_double2(ppq[2 * w], ppq[2 * w + 1]);
        }
      }
    };
    if (VAR == 5) {
      double di[10], dd[10], qa[8], qb[8], qc[8], qd[8], pa[8], pb[8], pc[8], pd[8];
      load(0, ci, co);
      squares(ci, co, qa, qb);
      int kp = -1;
#pragma unroll 1
      for (int k = 0; k < kTile; k += 16) {
        load(k + 8, di, dd);
        squares(di, dd, qc, qd);
        run_defer(k, ci, co, qa, qb, pa, pb, kp, pc, pd);
        if (k + 16 < kTile) { load(k + 16, ci, co); squares(ci, co, qa, qb); }
        run_defer(k + 8, di, dd, qc, qd, pc, pd, k, pa, pb);
        kp = k + 8;
      }
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        *reinterpret_cast<double2*>(as + kp + 2 * w) = make_double2(pc[2 * w], pc[2 * w + 1]);
        *reinterpret_cast<double2*>(aq + kp + 2 * w) = make_double2(pd[2 * w], pd[2 * w + 1]);
      }
    } else if (VAR == 4) {
      double di[10], dd[10], qa[8], qb[8], qc[8], qd[8];
      load(0, ci, co);
      squares(ci, co, qa, qb);
#pragma unroll 1
      for (int k = 0; k < kTile; k += 16) {
        load(k + 8, di, dd);
        squares(di, dd, qc, qd);
        batch_sq(k, ci, co, qa, qb);
        if (k + 16 < kTile) { load(k + 16, ci, co); squares(ci, co, qa, qb); }
        batch_sq(k + 8, di, dd, qc, qd);
      }
    } else if (VAR == 2) {
#pragma unroll 1
      for (int k = 0; k < kTile; k += 8) {
        load(k, ci, co);
        batch(k, ci, co);
      }
    } else if (VAR == 3) {
      double di[10], dd[10];
      load(0, ci, co);
#pragma unroll 1
      for (int k = 0; k < kTile; k += 16) {
        load(k + 8, di, dd);
        batch(k, ci, co);
        if (k + 16 < kTile) load(k + 16, ci, co);
        batch(k + 8, di, dd);
      }
    } else {
      load(0, ci, co);
#pragma unroll 1
      for (int k = 0; k < kTile; k += 8) {
        double ni[10], no[10];
        if (k + 8 < kTile) load(k + 8, ni, no);
        batch(k, ci, co);
#pragma unroll
        for (int u = 0; u < 10; ++u) { ci[u] = ni[u]; co[u] = no[u]; }
      }
    }
  }
  long long t1 = clock64();
  out[lane] = sum + sq + acc_s[lane * 7];
  if (lane == 0) *cyc = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 32 * 8);
  cudaMalloc(&cyc, 8);
  const int tiles = 2000;
  const int smem = 128 * kRow * 8;
  cudaFuncSetAttribute(chain<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(chain<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(chain<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(chain<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"kernel loop", "no STS", "no prefetch", "2-batch unroll", "2-batch + squares ahead", "+ deferred stores"};
  cudaFuncSetAttribute(chain<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(chain<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int act : {16})
  for (int v = 2; v < 6; ++v) {
    if (v == 0) chain<0><<<1, 32, smem>>>(tiles, out, cyc, act);
    if (v == 1) chain<1><<<1, 32, smem>>>(tiles, out, cyc, act);
    if (v == 2) chain<2><<<1, 32, smem>>>(tiles, out, cyc, act);
    if (v == 3) chain<3><<<1, 32, smem>>>(tiles, out, cyc, act);
    if (v == 4) chain<4><<<1, 32, smem>>>(tiles, out, cyc, act);
    if (v == 5) chain<5><<<1, 32, smem>>>(tiles, out, cyc, act);
    long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("lanes %2d %-24s %.2f cycles/slide\n", act, names[v], c / (64.0 * tiles));
  }
  return 0;
}
