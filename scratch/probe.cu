// Throw-away microbenchmark: FP64 latencies and throughput on B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat_dadd(double* out, double a, long long* cyc, int n) {
  double x = a; long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = __dadd_rn(x, a); }
  long long t1 = clock64(); out[threadIdx.x] = x; if (threadIdx.x==0) *cyc = t1 - t0;
}
__global__ void lat_min(double* out, double a, long long* cyc, int n) {
  double x = a, y = a * 0.5; long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = (x < y ? x : y) ; y = __dadd_rn(y, 1e-300); x = __dadd_rn(x, a);}
  long long t1 = clock64(); out[threadIdx.x] = x; if (threadIdx.x==0) *cyc = t1 - t0;
}
__global__ void lat_shfl(double* out, double a, long long* cyc, int n) {
  double x = a + threadIdx.x; long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = __shfl_up_sync(0xffffffff, x, 1); }
  long long t1 = clock64(); out[threadIdx.x] = x; if (threadIdx.x==0) *cyc = t1 - t0;
}
__global__ void tput_dfma(double* out, double a, int n) {
  double x0=a,x1=a+1,x2=a+2,x3=a+3,x4=a+4,x5=a+5,x6=a+6,x7=a+7;
  for (int i = 0; i < n; ++i) {
    x0=__dadd_rn(x0,a);x1=__dadd_rn(x1,a);x2=__dadd_rn(x2,a);x3=__dadd_rn(x3,a);
    x4=__dadd_rn(x4,a);x5=__dadd_rn(x5,a);x6=__dadd_rn(x6,a);x7=__dadd_rn(x7,a);
  }
  out[blockIdx.x*blockDim.x+threadIdx.x] = x0+x1+x2+x3+x4+x5+x6+x7;
}
__global__ void tput_dsetp(double* out, double a, int n) {
  double x0=a,x1=a+1,x2=a+2,x3=a+3,x4=a+4,x5=a+5,x6=a+6,x7=a+7;
  double y = a*0.75;
  for (int i = 0; i < n; ++i) {
    x0=x0<y?x0:y; x1=x1<y?x1:y; x2=x2<y?x2:y; x3=x3<y?x3:y;
    x4=x4<y?x4:y; x5=x5<y?x5:y; x6=x6<y?x6:y; x7=x7<y?x7:y; y = y*1.0000001;
  }
  out[blockIdx.x*blockDim.x+threadIdx.x] = x0+x1+x2+x3+x4+x5+x6+x7;
}
int main() {
  double* d; long long* c; cudaMalloc(&d, 1<<26); cudaMalloc(&c, 8);
  long long h; int n = 1<<16;
  lat_dadd<<<1,32>>>(d, 1e-3, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("dadd lat %.2f cyc\n", (double)h/n);
  lat_min<<<1,32>>>(d, 1e-3, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("min+dadd chain %.2f cyc\n", (double)h/n);
  lat_shfl<<<1,32>>>(d, 1e-3, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("shfl64 lat %.2f cyc\n", (double)h/n);
  int dev; cudaGetDevice(&dev); cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("SMs %d clock %d kHz\n", p.multiProcessorCount, p.clockRate);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep=0; rep<2; ++rep) {
  int blocks = p.multiProcessorCount*8, thr = 256; int it = 1<<14;
  cudaEventRecord(e0); tput_dfma<<<blocks,thr>>>(d, 1e-3, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = (double)blocks*thr*it*8; printf("DADD tput %.3e ops/s (%.1f ops/clk/SM at 1.965GHz)\n", ops/(ms*1e-3), ops/(ms*1e-3)/148/1.965e9);
  cudaEventRecord(e0); tput_dsetp<<<blocks,thr>>>(d, 1e-3, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  ops = (double)blocks*thr*it*8; printf("min(d) tput %.3e ops/s (%.1f /clk/SM)\n", ops/(ms*1e-3), ops/(ms*1e-3)/148/1.965e9);
  }
  return 0;
}
