// stats chain: global-memory variants, 8 chains per warp (lanes 0..7), 125 warps
#include <cstdio>
#define B 16
__global__ void k(const double* __restrict__ ref, double* __restrict__ o1, double* __restrict__ o2,
                  int nsl, int mode, long long* cyc) {
  const int lane = threadIdx.x;
  if (lane >= 8) return;
  const long long s0 = (blockIdx.x * 8LL + lane) * 100000;
  const double* pin = ref + s0 + 1024; const double* pout = ref + s0;
  double* os = o1 + s0; double* oq = o2 + s0;
  double sum = 0, sq = 0;
  double ai[B], ao[B], bi[B], bo[B];
  auto load = [&](int t0, double* vi, double* vo) {
#pragma unroll
    for (int u = 0; u < B; ++u) { vi[u] = pin[t0 + u]; vo[u] = pout[t0 + u]; } };
  auto run = [&](int t0, const double* vi, const double* vo) {
#pragma unroll
    for (int u = 0; u < B; ++u) {
      sum = __dsub_rn(__dadd_rn(sum, vi[u]), vo[u]);
      sq = __dsub_rn(__dadd_rn(sq, __dmul_rn(vi[u], vi[u])), __dmul_rn(vo[u], vo[u]));
      if (mode == 1) { os[t0 + u] = sum; oq[t0 + u] = sq; }
    } };
  long long c0 = clock64();
  load(0, ai, ao);
  for (int t = 0; t + 3 * B <= nsl; t += 2 * B) { load(t + B, bi, bo); run(t, ai, ao); load(t + 2 * B, ai, ao); run(t + B, bi, bo); }
  long long c1 = clock64();
  if (mode == 0) { os[0] = sum; oq[0] = sq; }
  if (lane == 0 && blockIdx.x == 0) *cyc = c1 - c0;
}
int main() {
  const long long n = 100000000LL + 2048;
  double *ref, *o1, *o2; long long* cyc;
  cudaMalloc(&ref, n * 8); cudaMalloc(&o1, n * 8); cudaMalloc(&o2, n * 8); cudaMalloc(&cyc, 8);
  cudaMemset(ref, 0, n * 8);
  const int nsl = 99999;
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0); k<<<125, 32>>>(ref, o1, o2, nsl, mode, cyc); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      printf("mode %d (%s): %.3f ms, %.1f cycles/slide\n", mode, mode ? "stores" : "no stores", ms, (double)h / nsl);
    }
  }
  return 0;
}
