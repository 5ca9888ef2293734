// bounds.cu -- the reference's lower-bound helpers (proj/include/eapdtw/
// lower_bounds.hpp:12-63) as device kernels, for the C ABI's boundary API
// (eapdtw_compute_envelope / _lb_kim_fl / _lb_keogh / _cumulative_bound).
// These are single-pair helpers a caller of the reference uses directly (its
// acceptance criterion 6, cascade_decision); the search itself runs the fused
// tiers of search_kernel.  Ordered sums (lb_keogh, cumulative_bound) run in
// one thread in the reference's order, so their bits are the reference's.
#include <algorithm>

#include "kernels.cuh"

namespace eapdtw_b200 {

// LB_Kim first/last (lower_bounds.cpp:51-55)
__global__ void lb_kim_fl_kernel(const double* __restrict__ q, const double* __restrict__ c,
                                 long long l, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0)
    *out = __dadd_rn(sq_cost(q[0], c[0]), sq_cost(q[l - 1], c[l - 1]));
}

// LB_Keogh (lower_bounds.cpp:57-88): visit positions in `order` (natural when
// null), accumulate in that order, abandon once the total strictly exceeds
// abandon_above.  contrib must be zeroed by the caller (unvisited = 0).
__global__ void lb_keogh_kernel(const double* __restrict__ up, const double* __restrict__ lo,
                                const double* __restrict__ x, long long l, double abandon_above,
                                const unsigned long long* __restrict__ order, double* total,
                                double* __restrict__ contrib, int* abandoned) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double t = 0.0;
  int ab = 0;
  for (long long k = 0; k < l; ++k) {
    const long long j = order ? static_cast<long long>(order[k]) : k;
    const double v = x[j];
    double d = 0.0;
    if (v > up[j]) d = sq_cost(v, up[j]);
    else if (v < lo[j]) d = sq_cost(v, lo[j]);
    t = __dadd_rn(t, d);
    contrib[j] = d;
    if (t > abandon_above) {
      ab = 1;
      break;
    }
  }
  *total = t;
  *abandoned = ab;
}

// cumulative_bound (lower_bounds.cpp:90-103): cb[k] = cb[k+1] + c[k+1]
__global__ void cumulative_bound_kernel(const double* __restrict__ c, long long l,
                                        double* __restrict__ cb) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  cb[l - 1] = 0.0;
  for (long long k = l - 1; k-- > 0;) cb[k] = __dadd_rn(cb[k + 1], c[k + 1]);
}

cudaError_t launch_lb_kim_fl(const double* q, const double* c, long long l, double* out,
                             cudaStream_t s) {
  lb_kim_fl_kernel<<<1, 32, 0, s>>>(q, c, l, out);
  return cudaGetLastError();
}

cudaError_t launch_lb_keogh(const double* up, const double* lo, const double* x, long long l,
                            double abandon_above, const unsigned long long* order, double* total,
                            double* contrib, int* abandoned, cudaStream_t s) {
  lb_keogh_kernel<<<1, 32, 0, s>>>(up, lo, x, l, abandon_above, order, total, contrib, abandoned);
  return cudaGetLastError();
}

cudaError_t launch_cumulative_bound(const double* c, long long l, double* cb, cudaStream_t s) {
  cumulative_bound_kernel<<<1, 32, 0, s>>>(c, l, cb);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Sliding max/min of any radius (compute_envelope, lower_bounds.cpp:9-49):
// the tiled shared-memory kernel when its tile holds the window, else the same
// sparse-table doubling in global memory over the series padded by r
// identities on each side: M_{2s}[i] = max(M_s[i], M_s[i+s]); with K = 2r+1
// and P the largest power of two <= K, the window of p (padded [p, p+2r]) is
// max(M_P[p], M_P[p + K - P]).  Max and min are exact picks, so any order
// gives the reference's values.
// ---------------------------------------------------------------------------
template <bool MAX>
__device__ __forceinline__ double pick2(double a, double b) {
  return MAX ? (a > b ? a : b) : (a < b ? a : b);
}

template <bool MAX>
__global__ void env_pad_kernel(const double* __restrict__ x, long long n, long long r,
                               double* __restrict__ buf) {
  const double ident = MAX ? -d_inf() : d_inf();
  for (long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; k < n + 2 * r;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long p = k - r;
    buf[k] = (p >= 0 && p < n) ? x[p] : ident;
  }
}

template <bool MAX>
__global__ void env_double_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                  long long len, long long s) {
  for (long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; k < len;
       k += static_cast<long long>(gridDim.x) * blockDim.x)
    dst[k] = k + s < len ? pick2<MAX>(src[k], src[k + s]) : src[k];
}

template <bool MAX>
__global__ void env_final_kernel(const double* __restrict__ m, long long n, long long K,
                                 long long P, double* __restrict__ env) {
  for (long long p = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; p < n;
       p += static_cast<long long>(gridDim.x) * blockDim.x)
    env[2 * p + (MAX ? 0 : 1)] = pick2<MAX>(m[p], m[p + K - P]);
}

size_t envelope_any_scratch_doubles(long long n, long long r) {
  return envelope_tile(static_cast<int>(std::min<long long>(r, 1 << 20))) >= 256
             ? 0
             : 2 * static_cast<size_t>(n + 2 * r);
}

cudaError_t launch_envelope_any(const double* x, long long n, long long r, double* env,
                                double* scratch, cudaStream_t s) {
  if (r <= (1 << 20) && envelope_tile(static_cast<int>(r)) >= 256)
    return launch_envelope(x, n, static_cast<int>(r), env, s);
  const long long len = n + 2 * r, K = 2 * r + 1;
  long long P = 1;
  while (2 * P <= K) P *= 2;
  const int blocks = static_cast<int>(std::min<long long>((len + 255) / 256, 148LL * 8));
  auto run = [&](auto max_tag) -> cudaError_t {
    constexpr bool MAX = decltype(max_tag)::value;
    double* a = scratch;
    double* b = scratch + len;
    env_pad_kernel<MAX><<<blocks, 256, 0, s>>>(x, n, r, a);
    for (long long st = 1; st < P; st *= 2) {
      env_double_kernel<MAX><<<blocks, 256, 0, s>>>(a, b, len, st);
      std::swap(a, b);
    }
    env_final_kernel<MAX><<<blocks, 256, 0, s>>>(a, n, K, P, env);
    return cudaGetLastError();
  };
  cudaError_t e = run(std::true_type{});
  if (e == cudaSuccess) e = run(std::false_type{});
  return e;
}

}  // namespace eapdtw_b200
