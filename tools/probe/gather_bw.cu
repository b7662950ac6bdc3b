// Memory-system probes for the SpMM roofline: streaming copy, random row
// gathers from a DRAM-sized table and from an L2-resident table.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

template <int VEC>  // floats per lane-load (4 = 16 B)
__global__ void gather_rows(const float* __restrict__ table, const int* __restrict__ idx, float* __restrict__ out,
                            int64_t nrows_out, int row_floats) {
  // one group of (row_floats/4) lanes per output row
  const int lpr = row_floats / 4;
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t row = gid / lpr;
  const int l = gid % lpr;
  if (row >= nrows_out) return;
  const int src = __ldg(idx + row);
  float4 v = __ldg(reinterpret_cast<const float4*>(table + (int64_t)src * row_floats) + l);
  reinterpret_cast<float4*>(out + row * row_floats)[l] = v;
}

__global__ void gather_sum(const float* __restrict__ table, const int* __restrict__ idx, float* __restrict__ out,
                           int64_t nrows_out, int row_floats, int per) {
  // each group sums `per` random rows (gather-only traffic, small output)
  const int lpr = row_floats / 4;
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t row = gid / lpr;
  const int l = gid % lpr;
  if (row >= nrows_out) return;
  float4 acc = make_float4(0, 0, 0, 0);
#pragma unroll 8
  for (int j = 0; j < per; ++j) {
    const int src = __ldg(idx + row * per + j);
    float4 v = __ldg(reinterpret_cast<const float4*>(table + (int64_t)src * row_floats) + l);
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  reinterpret_cast<float4*>(out + row * row_floats)[l] = acc;
}

__global__ void copy_kernel(const float4* __restrict__ a, float4* __restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // streaming copy 2 GB
  {
    int64_t n = (int64_t)1 << 27;  // float4s = 2 GiB
    float4 *a, *b;
    cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16);
    cudaMemset(a, 0, n * 16);
    for (int r = 0; r < 2; ++r) copy_kernel<<<148 * 16, 256>>>(a, b, n);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) copy_kernel<<<148 * 16, 256>>>(a, b, n);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("copy: %.1f GB/s (read+write)\n", 5.0 * 2 * n * 16 / (ms * 1e6));
    cudaFree(a); cudaFree(b);
  }
  std::mt19937_64 rng(1);
  for (int row_floats : {8, 16, 32, 64, 128}) {
    for (int64_t table_mb : {64LL, 1280LL}) {
      int64_t trows = table_mb * 1024 * 1024 / (row_floats * 4);
      int per = 16;
      int64_t orows = 1 << 20;
      float *table, *out; int* idx;
      cudaMalloc(&table, trows * row_floats * 4);
      cudaMemset(table, 0, trows * row_floats * 4);
      cudaMalloc(&out, orows * row_floats * 4);
      std::vector<int> h(orows * per);
      for (auto& x : h) x = (int)(rng() % trows);
      cudaMalloc(&idx, h.size() * 4);
      cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
      int64_t threads = orows * (row_floats / 4);
      unsigned grid = (unsigned)((threads + 255) / 256);
      for (int r = 0; r < 2; ++r) gather_sum<<<grid, 256>>>(table, idx, out, orows, row_floats, per);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) gather_sum<<<grid, 256>>>(table, idx, out, orows, row_floats, per);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      double gathered = 5.0 * orows * per * row_floats * 4;
      printf("random gather rows of %4d B from %5lld MB table: %.1f GB/s gathered (%.2f ms/launch)\n",
             row_floats * 4, (long long)table_mb, gathered / (ms * 1e6), ms / 5);
      cudaFree(table); cudaFree(out); cudaFree(idx);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
