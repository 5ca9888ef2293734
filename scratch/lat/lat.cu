// dependent-chain latency probes: DADD, DSETP+FSEL (min), SHFL.64, LDS.64
#include <cstdio>
__global__ void k_dadd(double* out, double x, int n, long long* cyc) {
  double a = x, b = x * 0.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { a = __dadd_rn(a, b); a = __dadd_rn(a, -b); }
  long long t1 = clock64();
  out[threadIdx.x] = a; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_dmul(double* out, double x, int n, long long* cyc) {
  double a = x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { a = __dmul_rn(a, 1.0000001); a = __dmul_rn(a, 0.9999999); }
  long long t1 = clock64();
  out[threadIdx.x] = a; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_dmin(double* out, double x, int n, long long* cyc) {
  double a = x, b = x * 0.5 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { a = b < a ? b : a; b = a < b ? b : a + 1.0e-300; }
  long long t1 = clock64();
  out[threadIdx.x] = a + b; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_shfl(double* out, double x, int n, long long* cyc) {
  double a = x + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { a = __shfl_up_sync(0xffffffffu, a, 1); a = __shfl_down_sync(0xffffffffu, a, 1); }
  long long t1 = clock64();
  out[threadIdx.x] = a; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_lds(double* out, double x, int n, long long* cyc) {
  __shared__ int idx[64];
  idx[threadIdx.x] = threadIdx.x; idx[threadIdx.x + 32] = threadIdx.x;
  __syncwarp();
  int a = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { a = idx[a]; a = idx[a + 32]; }
  long long t1 = clock64();
  out[threadIdx.x] = a; if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024); cudaMalloc(&c, 8);
  const int n = 4096; long long h;
  auto run = [&](const char* name, void (*k)(double*, double, int, long long*)) {
    k<<<1, 32>>>(o, 1.5, n, c); k<<<1, 32>>>(o, 1.5, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-6s %.1f cycles per dependent op\n", name, h / (2.0 * n));
  };
  run("dadd", k_dadd); run("dmul", k_dmul); run("dmin", k_dmin); run("shfl64", k_shfl); run("lds32", k_lds);
  return 0;
}
