// Throughput of vector fp32 reductions (red.global.add.v4.f32) into an
// L2-resident table of 128-B rows, alone and next to random 128-B DRAM row
// gathers in the same kernel.  Question behind it: can a cold row PUSH its own
// row into the partial sums of its hub neighbours (L2 atomics) instead of the
// hub rows pulling cold rows from DRAM (config 4)?
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o l2_red l2_red.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ void red4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}
__device__ __forceinline__ void ld8(const float* p, float (&v)[8]) {
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]),
                 "=f"(v[7]) : "l"(p));
}

// MODE 0: reds only; 1: gathers only; 2: both (per row: PER reds + PER gathers)
template <int MODE, int PER>
__global__ void __launch_bounds__(256) push_kernel(float* __restrict__ hubP, const int* __restrict__ hub_idx,
                                                   const float* __restrict__ cold, const int* __restrict__ cold_idx,
                                                   float* __restrict__ out, int64_t rows) {
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t row = gid >> 2;
  const int l = gid & 3;
  if (row >= rows) return;
  float acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.f;
  float own[8];
  ld8(cold + row * 32 + l * 8, own);  // the row's own slice (streamed)
  if (MODE != 0) {
#pragma unroll 2
    for (int j = 0; j < PER; ++j) {
      float v[8];
      ld8(cold + (int64_t)__ldg(cold_idx + row * PER + j) * 32 + l * 8, v);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] += v[i];
    }
  }
  if (MODE != 1) {
#pragma unroll 2
    for (int j = 0; j < PER; ++j) {
      float* p = hubP + (int64_t)__ldg(hub_idx + row * PER + j) * 32 + l * 8;
      red4(p, own[0], own[1], own[2], own[3]);
      red4(p + 4, own[4], own[5], own[6], own[7]);
    }
  }
  float* o = out + row * 32 + l * 8;
  *reinterpret_cast<float4*>(o) = make_float4(acc[0] + own[0], acc[1], acc[2], acc[3]);
  *reinterpret_cast<float4*>(o + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
}

template <int MODE, int PER>
float run(float* hubP, const int* hi, const float* cold, const int* ci, float* out, int64_t rows) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  unsigned grid = (unsigned)((rows * 4 + 255) / 256);
  for (int r = 0; r < 2; ++r) push_kernel<MODE, PER><<<grid, 256>>>(hubP, hi, cold, ci, out, rows);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) push_kernel<MODE, PER><<<grid, 256>>>(hubP, hi, cold, ci, out, rows);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("CUDA error %s\n", cudaGetErrorString(e));
  return ms / 5;
}

int main() {
  const int64_t rows = 8'000'000;   // cold rows (1.02 GB table)
  constexpr int PER = 4;            // hub neighbours / cold neighbours per cold row
  float *cold, *out, *hubP;
  int *hi, *ci;
  cudaMalloc(&cold, rows * 128); cudaMalloc(&out, rows * 128);
  cudaMemset(cold, 0, rows * 128);
  cudaMalloc(&hi, rows * PER * 4); cudaMalloc(&ci, rows * PER * 4);
  std::mt19937_64 g(1);
  std::vector<int> h(rows * PER);
  for (auto& x : h) x = (int)(g() % rows);
  cudaMemcpy(ci, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  for (int64_t H : {50'000, 200'000, 400'000}) {
    cudaMalloc(&hubP, H * 128);
    cudaMemset(hubP, 0, H * 128);
    for (int skew = 0; skew < 3; ++skew) {
      // skew 0: uniform hub ids; 1: id = H u^3; 2: id = H u^8 (a few rows take most pushes)
      std::uniform_real_distribution<double> U(0.0, 1.0);
      const double pw = skew == 0 ? 1.0 : (skew == 1 ? 3.0 : 8.0);
      for (auto& x : h) { int64_t v = (int64_t)(H * std::pow(U(g), pw)); x = (int)(v >= H ? H - 1 : v); }
      cudaMemcpy(hi, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
      float t0 = run<0, PER>(hubP, hi, cold, ci, out, rows);
      float t1 = run<1, PER>(hubP, hi, cold, ci, out, rows);
      float t2 = run<2, PER>(hubP, hi, cold, ci, out, rows);
      const double red_bytes = (double)rows * PER * 128;
      printf("H=%ld rows (%.1f MB) skew u^%.0f: reds only %.3f ms (%.2f TB/s of pushed bytes, %.1f G rows/s) | "
             "gathers only %.3f ms | both %.3f ms\n",
             (long)H, H * 128 / 1e6, pw, t0, red_bytes / t0 / 1e9, rows * PER / t0 / 1e6, t1, t2);
    }
    cudaFree(hubP);
  }
  return 0;
}
