// Microbenchmark: FP64 issue cost per warp instruction on one SMSP (one warp,
// 32 lanes, 8 independent chains of DADD or DMUL) and with 4 warps per block.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>  // 0: DADD, 1: DMUL, 2: FADD (fp32)
__global__ void k(int iters, double* out, long long* cyc) {
  double a[8];
  float f[8];
  for (int u = 0; u < 8; ++u) { a[u] = threadIdx.x + u; f[u] = threadIdx.x + u; }
  const double c = 1.0000001;
  const float cf = 1.0000001f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (OP == 0) a[u] = __dadd_rn(a[u], c);
      if (OP == 1) a[u] = __dmul_rn(a[u], c);
      if (OP == 2) f[u] = __fadd_rn(f[u], cf);
    }
  }
  long long t1 = clock64();
  double s = 0;
  for (int u = 0; u < 8; ++u) s += a[u] + f[u];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * 8);
  cudaMalloc(&cyc, 8);
  const int iters = 20000;
  const char* nm[] = {"DADD", "DMUL", "FADD"};
  for (int op = 0; op < 3; ++op)
    for (int warps : {1, 4, 8}) {
      if (op == 0) k<0><<<1, 32 * warps>>>(iters, out, cyc);
      if (op == 1) k<1><<<1, 32 * warps>>>(iters, out, cyc);
      if (op == 2) k<2><<<1, 32 * warps>>>(iters, out, cyc);
      long long c = 0;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      printf("%s warps=%d: %.2f cycles per warp-instruction per warp (8 chains)\n", nm[op], warps,
             c / (8.0 * iters));
    }
  return 0;
}
