// L2-resident random row gathers with U independent loads in flight per
// lane (register-held, 32-B or 16-B lane vectors): the ceiling the SBM
// SpMM terms (configs 3/5) run against.  Also prints the persisting-L2 and
// access-policy-window limits of the device.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

template <int U, int VB>  // VB: bytes per lane load (16 or 32)
__global__ void __launch_bounds__(256) gsum(const float* __restrict__ table, const int* __restrict__ idx,
                                            float* __restrict__ out, int64_t nrows_out, int row_bytes, int per) {
  const int lpr = row_bytes / VB;
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t row = gid / lpr;
  const int l = gid % lpr;
  if (row >= nrows_out) return;
  constexpr int NF = VB / 4;
  float acc[NF];
#pragma unroll
  for (int i = 0; i < NF; ++i) acc[i] = 0.f;
  const int* ip = idx + row * per;
  for (int j = 0; j < per; j += U) {
    float v[U][NF];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float* p = table + (int64_t)__ldg(ip + j + u) * (row_bytes / 4) + l * NF;
      if constexpr (VB == 32) {
        asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(v[u][0]), "=f"(v[u][1]), "=f"(v[u][2]), "=f"(v[u][3]), "=f"(v[u][4]),
                       "=f"(v[u][5]), "=f"(v[u][6]), "=f"(v[u][7]) : "l"(p));
      } else {
        float4 t = __ldg(reinterpret_cast<const float4*>(p));
        v[u][0] = t.x; v[u][1] = t.y; v[u][2] = t.z; v[u][3] = t.w;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int i = 0; i < NF; ++i) acc[i] += v[u][i];
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NF; ++i) s += acc[i];
  out[gid] = s;
}

template <int U, int VB>
void run(const float* table, const int* idx, float* out, int64_t orows, int row_bytes, int per, int64_t trows_mb) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  int64_t threads = orows * (row_bytes / VB);
  unsigned grid = (unsigned)((threads + 255) / 256);
  for (int r = 0; r < 2; ++r) gsum<U, VB><<<grid, 256>>>(table, idx, out, orows, row_bytes, per);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) gsum<U, VB><<<grid, 256>>>(table, idx, out, orows, row_bytes, per);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double gathered = 5.0 * orows * per * row_bytes;
  printf("table %4lld MB rows %3d B lane %2d B U=%d: %8.1f GB/s gathered\n", (long long)trows_mb, row_bytes, VB, U,
         gathered / (ms * 1e6));
}

int main() {
  int dev = 0, v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxPersistingL2CacheSize, dev);
  printf("max persisting L2 set-aside: %d B (%.1f MB)\n", v, v / 1048576.0);
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxAccessPolicyWindowSize, dev);
  printf("max access-policy window: %d B (%.1f MB)\n", v, v / 1048576.0);
  cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, dev);
  printf("L2: %d B (%.1f MB)\n", v, v / 1048576.0);
  std::mt19937_64 rng(1);
  for (int row_bytes : {128, 256, 512}) {
    for (int64_t table_mb : {16LL, 48LL}) {
      int64_t trows = table_mb * 1024 * 1024 / row_bytes;
      const int per = 16;
      const int64_t orows = (1 << 22) / (row_bytes / 128);
      float *table, *out; int* idx;
      cudaMalloc(&table, trows * row_bytes);
      cudaMemset(table, 0, trows * row_bytes);
      cudaMalloc(&out, orows * (row_bytes / 16) * 4);
      std::vector<int> h(orows * per);
      for (auto& x : h) x = (int)(rng() % trows);
      cudaMalloc(&idx, h.size() * 4);
      cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
      run<1, 32>(table, idx, out, orows, row_bytes, per, table_mb);
      run<2, 32>(table, idx, out, orows, row_bytes, per, table_mb);
      run<4, 32>(table, idx, out, orows, row_bytes, per, table_mb);
      run<1, 16>(table, idx, out, orows, row_bytes, per, table_mb);
      run<4, 16>(table, idx, out, orows, row_bytes, per, table_mb);
      cudaFree(table); cudaFree(out); cudaFree(idx);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
