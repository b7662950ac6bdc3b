// k-means on the spectral embedding (replaces the (n, c, d) broadcast of
// kmeans_cluster, metrics.py:143-176, which needs 51 GB at config 3).
// Distances in fp64 from the fp32 embedding; one warp per row computes all c
// squared distances, picks the first minimum (np.argmin tie rule) and adds
// the row into its centroid's sum.  The sums are accumulated in 64-bit FIXED
// POINT (integer atomics are associative), so they -- and hence the next
// centroids and labels -- are identical run to run, unlike fp64 atomics whose
// rounding depends on arrival order.  The scale 2^s is chosen from max|X|
// (device-side, no host sync) so the n-row sum cannot overflow; each input is
// rounded to 2^-s absolute (s >= 40 for n <= 2^20 and |X| < 1).

#include <mutex>

#include "sped_common.cuh"

namespace {

__global__ void row_dist2_kernel(int64_t n, int32_t d, const float* __restrict__ X,
                                 const double* __restrict__ center, double* __restrict__ dist,
                                 int32_t accumulate_min) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  double s = 0.0;
  for (int j = lane; j < d; j += 32) {
    const double t = (double)X[row * d + j] - center[j];
    s += t * t;
  }
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) dist[row] = accumulate_min ? fmin(dist[row], s) : s;
}

__global__ void absmax_kernel(int64_t count, const float* __restrict__ X, unsigned int* bits) {
  unsigned int m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, __float_as_uint(fabsf(X[i])));  // order of non-negative floats = order of bits
  for (int off = 16; off > 0; off >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0) atomicMax(bits, m);
}

// fixed-point scale 2^s: n * max|X| * 2^s < 2^62
__device__ __forceinline__ double fixed_scale(int64_t n, const unsigned int* bits) {
  const float mx = __uint_as_float(*bits);
  int e = 0;
  frexpf(mx > 0.f ? mx : 1.f, &e);  // mx < 2^e
  int ln = 0;
  while (((int64_t)1 << ln) < n + 1) ++ln;  // n < 2^ln
  return ldexp(1.0, 62 - ln - e);
}

__global__ void assign_kernel(int64_t n, int32_t d, int32_t c, const float* __restrict__ X,
                              const double* __restrict__ centers, int32_t* __restrict__ labels,
                              long long* __restrict__ fsums, unsigned long long* __restrict__ counts,
                              double* __restrict__ min_d2, const unsigned int* __restrict__ bits) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  double best = 0.0;
  int arg = 0;
  for (int j = 0; j < c; ++j) {
    double s = 0.0;
    for (int q = lane; q < d; q += 32) {
      const double t = (double)X[row * d + q] - centers[(int64_t)j * d + q];
      s += t * t;
    }
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (j == 0 || s < best) {
      best = s;
      arg = j;
    }
  }
  if (lane == 0) {
    labels[row] = arg;
    min_d2[row] = best;
    atomicAdd(counts + arg, 1ULL);
  }
  const double sc = fixed_scale(n, bits);
  for (int q = lane; q < d; q += 32)
    atomicAdd(reinterpret_cast<unsigned long long*>(fsums + (int64_t)arg * d + q),
              (unsigned long long)__double2ll_rn((double)X[row * d + q] * sc));
}

__global__ void fixed_to_double_kernel(int64_t count, int64_t n, const unsigned int* bits,
                                       double* sums) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= count) return;
  const long long v = reinterpret_cast<const long long*>(sums)[i];
  sums[i] = (double)v / fixed_scale(n, bits);
}

unsigned int* maxbits_scratch() {
  static unsigned int* p[16] = {};
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 16) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!p[dev] && cudaMalloc(&p[dev], sizeof(unsigned int)) != cudaSuccess) {
    cudaGetLastError();
    p[dev] = nullptr;
  }
  return p[dev];
}

}  // namespace

using namespace sped;

extern "C" int sped_row_dist2(int64_t n, int32_t d, const float* X, const double* center,
                              double* dist, int32_t accumulate_min, sped_stream_t stream) {
  SPED_CHECK_ARG(n >= 0 && d >= 1, "bad dist arguments");
  if (n == 0) return SPED_OK;
  SPED_CHECK_ARG(X && center && dist, "null array");
  row_dist2_kernel<<<grid_for(n, 8), 256, 0, as_stream(stream)>>>(n, d, X, center, dist,
                                                                   accumulate_min);
  SPED_LAUNCH_CHECK();
  return SPED_OK;
}

extern "C" int sped_kmeans_assign(int64_t n, int32_t d, int32_t c, const float* X,
                                  const double* centers, int32_t* labels, double* sums,
                                  int64_t* counts, double* min_d2, sped_stream_t stream) {
  SPED_CHECK_ARG(n >= 0 && d >= 1 && c >= 1, "bad kmeans arguments");
  if (n == 0) return SPED_OK;
  SPED_CHECK_ARG(X && centers && labels && sums && counts && min_d2, "null array");
  cudaStream_t s = as_stream(stream);
  unsigned int* bits = maxbits_scratch();
  if (!bits) {
    set_error("kmeans: device scratch allocation failed");
    return SPED_ERR_CUDA;
  }
  SPED_CUDA(cudaMemsetAsync(bits, 0, sizeof(unsigned int), s));
  absmax_kernel<<<grid_for(n * d, 256, num_sms() * 8), 256, 0, s>>>(n * (int64_t)d, X, bits);
  SPED_CUDA(cudaMemsetAsync(sums, 0, sizeof(double) * (size_t)c * d, s));
  SPED_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * (size_t)c, s));
  assign_kernel<<<grid_for(n, 8), 256, 0, s>>>(n, d, c, X, centers, labels,
                                               reinterpret_cast<long long*>(sums),
                                               reinterpret_cast<unsigned long long*>(counts),
                                               min_d2, bits);
  SPED_LAUNCH_CHECK();
  fixed_to_double_kernel<<<grid_for((int64_t)c * d, 256), 256, 0, s>>>((int64_t)c * d, n, bits,
                                                                        sums);
  SPED_LAUNCH_CHECK();
  return SPED_OK;
}
