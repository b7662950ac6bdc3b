// k-means on the spectral embedding (replaces the (n, c, d) broadcast of
// kmeans_cluster, metrics.py:143-176, which needs 51 GB at config 3).
// Distances in fp64 from the fp32 embedding; one warp per row computes all c
// squared distances, picks the first minimum (np.argmin tie rule) and adds
// the row into its centroid's fp64 sum.

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

__global__ void assign_kernel(int64_t n, int32_t d, int32_t c, const float* __restrict__ X,
                              const double* __restrict__ centers, int32_t* __restrict__ labels,
                              double* __restrict__ sums, unsigned long long* __restrict__ counts,
                              double* __restrict__ min_d2) {
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
  for (int q = lane; q < d; q += 32) atomicAdd(sums + (int64_t)arg * d + q, (double)X[row * d + q]);
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
  SPED_CUDA(cudaMemsetAsync(sums, 0, sizeof(double) * (size_t)c * d, s));
  SPED_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * (size_t)c, s));
  assign_kernel<<<grid_for(n, 8), 256, 0, s>>>(n, d, c, X, centers, labels, sums,
                                               reinterpret_cast<unsigned long long*>(counts),
                                               min_d2);
  SPED_LAUNCH_CHECK();
  return SPED_OK;
}
