// Microbenchmark: cycles per slide of the RunningStats chain (2 dependent
// DADD per slide for the sum, DMUL/DADD/DMUL/DSUB for the sum of squares)
// in one warp with k active lanes, inputs from registers or shared memory.
#include <cstdio>
#include <cuda_runtime.h>

template <int SRC>  // 0: registers, 1: shared memory (lane rows, 16-byte loads)
__global__ void chain(int active, int iters, double* out, long long* cyc) {
  __shared__ __align__(16) double sm[32 * 66];
  const int lane = threadIdx.x;
  for (int i = lane; i < 32 * 66; i += 32) sm[i] = 1.0 + 1e-3 * i;
  __syncwarp();
  double sum = lane, sq = lane;
  double r[8];
  for (int u = 0; u < 8; ++u) r[u] = 1.0 + lane * 1e-3 + u;
  long long t0 = clock64();
  if (lane < active) {
    for (int it = 0; it < iters; ++it) {
      if (SRC == 1) {
        const double* row = sm + lane * 66 + ((it * 8) & 63);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double2 v = *reinterpret_cast<const double2*>(row + 2 * u);
          r[2 * u] = v.x;
          r[2 * u + 1] = v.y;
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double xi = r[u], xo = r[(u + 3) & 7];
        sum = __dsub_rn(__dadd_rn(sum, xi), xo);
        sq = __dsub_rn(__dadd_rn(sq, __dmul_rn(xi, xi)), __dmul_rn(xo, xo));
      }
    }
  }
  long long t1 = clock64();
  out[lane] = sum + sq;
  if (lane == 0) *cyc = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 32 * 8);
  cudaMalloc(&cyc, 8);
  const int iters = 20000;
  for (int src = 0; src < 2; ++src)
    for (int k : {1, 2, 4, 8, 16, 32}) {
      if (src == 0) chain<0><<<1, 32>>>(k, iters, out, cyc);
      else chain<1><<<1, 32>>>(k, iters, out, cyc);
      long long c = 0;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      printf("src=%s lanes=%2d: %.2f cycles/slide\n", src ? "smem" : "regs", k, c / (8.0 * iters));
    }
  // several warps (one per SMSP) on one SM
  return 0;
}
