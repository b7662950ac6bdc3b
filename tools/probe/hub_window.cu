// Does the persisting-L2 window deliver the static-cache hit rate on a
// power-law gather stream?  Random 128-B row gathers from a 1.28 GB table
// (10^7 rows x 32 floats) with row r drawn with probability ~ its degree in
// a Chung-Lu-like law (rows sorted by degree: row 0 hottest), against:
//   none       -- plain LRU L2
//   window X   -- persisting access-policy window over the top X rows
//   hint X     -- per-load evict_last for rows < X, evict_first otherwise
// Reports ms per launch and the implied gathered GB/s.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t pol_last() { uint64_t p; asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ uint64_t pol_first() { uint64_t p; asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p; }

template <int MODE>  // 0 plain, 1 hint
__global__ void gather(const float* __restrict__ t, const int* __restrict__ idx, float* __restrict__ out,
                       int64_t nout, int per, int hot) {
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t row = gid / 4;
  const int l = gid % 4;
  if (row >= nout) return;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int j = 0; j < per; ++j) {
    const int r = __ldg(idx + row * per + j);
    const float* p = t + (int64_t)r * 32 + l * 8;
    float v[8];
    if (MODE == 0) {
      asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]) : "l"(p));
    } else {
      const uint64_t pol = r < hot ? pol_last() : pol_first();
      asm volatile("ld.global.nc.L2::cache_hint.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                   : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]) : "l"(p), "l"(pol));
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] += v[i];
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i];
  out[gid] = s;
}

int main() {
  const int64_t n = 10000000, nout = 1 << 22;
  const int per = 16;
  // degree-like weights: Pareto(shape 1.1) rescaled, sorted descending
  std::mt19937_64 rng(7);
  std::vector<double> wgt(n);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  for (auto& x : wgt) x = std::min(2.0 * std::pow(1.0 - U(rng), -1.0 / 1.1), 1e5);
  std::sort(wgt.begin(), wgt.end(), std::greater<double>());
  std::vector<double> cdf(n);
  double s = 0;
  for (int64_t i = 0; i < n; ++i) { s += wgt[i]; cdf[i] = s; }
  std::vector<int> h(nout * per);
  for (auto& x : h) {
    const double q = U(rng) * s;
    x = (int)(std::lower_bound(cdf.begin(), cdf.end(), q) - cdf.begin());
    if (x >= n) x = n - 1;
  }
  // shuffle the gather order (the SpMM walks rows in degree order, but each
  // row's neighbours are random)
  float *t, *out; int* idx;
  cudaMalloc(&t, n * 128); cudaMemset(t, 0, n * 128);
  cudaMalloc(&out, nout * 4 * 4);
  cudaMalloc(&idx, h.size() * 4);
  cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  int dev = 0, maxp = 0;
  cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const unsigned grid = (unsigned)((nout * 4 + 255) / 256);
  auto run = [&](const char* name, int mode, int hot, size_t win_rows, size_t setaside_mb) {
    size_t sa = std::min((size_t)maxp, setaside_mb << 20);
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, sa);
    cudaStreamAttrValue v = {};
    if (win_rows) {
      v.accessPolicyWindow.base_ptr = t;
      v.accessPolicyWindow.num_bytes = win_rows * 128;
      v.accessPolicyWindow.hitRatio = std::min(1.0, (double)sa / (win_rows * 128.0));
      v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    }
    cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v);
    cudaCtxResetPersistingL2Cache();
    for (int r = 0; r < 2; ++r) {
      if (mode) gather<1><<<grid, 256, 0, st>>>(t, idx, out, nout, per, hot);
      else gather<0><<<grid, 256, 0, st>>>(t, idx, out, nout, per, hot);
    }
    cudaEventRecord(e0, st);
    for (int r = 0; r < 5; ++r) {
      if (mode) gather<1><<<grid, 256, 0, st>>>(t, idx, out, nout, per, hot);
      else gather<0><<<grid, 256, 0, st>>>(t, idx, out, nout, per, hot);
    }
    cudaEventRecord(e1, st); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-28s %.3f ms/launch  %.0f GB/s gathered\n", name, ms / 5, 5.0 * nout * per * 128 / (ms * 1e6));
    v.accessPolicyWindow.num_bytes = 0; v.accessPolicyWindow.base_ptr = nullptr;
    cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v);
  };
  printf("max set-aside %.1f MB; ref fraction top 309657: %.3f, top 619314: %.3f\n", maxp / 1048576.0,
         cdf[309656] / s, cdf[619313] / s);
  run("none", 0, 0, 0, 0);
  run("window 309K / 40 MB", 0, 0, 309657, 40);
  run("window 619K / 79 MB", 0, 0, 619314, 79);
  run("window 309K / 79 MB", 0, 0, 309657, 79);
  run("hint 309K", 1, 309657, 0, 0);
  run("hint 619K", 1, 619314, 0, 0);
  run("hint 1M", 1, 1000000, 0, 0);
  run("window 309K + hint 1M", 1, 1000000, 309657, 40);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
