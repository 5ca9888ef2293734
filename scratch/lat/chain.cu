// stats-chain microbenchmark: cycles per slide of the (sum, sumsq) chain
#include <cstdio>
#define TILE 448
__global__ void chain(const double* in, int nslides, double* out, long long* cyc, int mode) {
  __shared__ double s_in[TILE], s_out[TILE], s_sum[TILE], s_sq[TILE];
  for (int k = threadIdx.x; k < TILE; k += blockDim.x) { s_in[k] = in[k]; s_out[k] = in[k + 1]; }
  __syncthreads();
  double sum = 0, sq = 0;
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int t = 0; t < nslides / TILE; ++t) {
      for (int k = 0; k + 8 <= TILE; k += 8) {
        double a[8], b[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) { a[u] = s_in[k + u]; b[u] = s_out[k + u]; }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          sum = __dsub_rn(__dadd_rn(sum, a[u]), b[u]);
          sq = __dsub_rn(__dadd_rn(sq, __dmul_rn(a[u], a[u])), __dmul_rn(b[u], b[u]));
          if (mode & 1) { s_sum[k + u] = sum; s_sq[k + u] = sq; }
        }
      }
      if (mode & 2) __syncwarp();
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[blockIdx.x] = sum + sq + s_sum[5] + s_sq[7]; cyc[blockIdx.x] = t1 - t0; }
}
int main() {
  double *in, *out; long long* cyc; cudaMalloc(&in, 8 * 1024); cudaMalloc(&out, 8 * 4096); cudaMalloc(&cyc, 8 * 4096);
  cudaMemset(in, 0, 8 * 1024);
  const int ns = TILE * 200;
  for (int mode = 0; mode < 2; ++mode)
    for (int blocks : {1, 148, 1036}) {
      chain<<<blocks, 64>>>(in, ns, out, cyc, mode);
      chain<<<blocks, 64>>>(in, ns, out, cyc, mode);
      long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0); chain<<<blocks, 64>>>(in, ns, out, cyc, mode); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("mode %d blocks %4d: %.1f cycles/slide (block 0), kernel %.3f ms\n", mode, blocks, (double)h / ns, ms);
    }
  return 0;
}
