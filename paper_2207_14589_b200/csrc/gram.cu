// K5: Gram of the block pair [V | M] for the solver step (replaces the
// tall-skinny BLAS contractions of mu_eg_step, solvers.py:130-135, and the
// Gram-Schmidt inner products of _orthonormalize, solvers.py:84-102).
//
// Output G (fp64, row-major k x k each): S = V^T V, C = V^T M, Q = M^T M.
// Z = [V | M] is n x K2 (K2 = 2k, or k without M).  The K2 x K2 Gram is cut
// into 64 x 64 output tiles (upper triangle only, Z^T Z is symmetric) and the
// n rows into `splits` ranges; each CTA stages 32-row slabs of the two
// column tiles in shared memory and accumulates a 4x4 register tile per
// thread in fp32, flushing into fp64 accumulators after every slab (so the
// fp32 sums never span more than 32 rows).  Per-split partial tiles are
// summed in split order by a second kernel -> deterministic.
//
// Roofline: reads 4*n*K2 bytes once per column-tile pair; at k <= 64 it is
// HBM/L2 bound, at k = 128 SIMT fp32 bound (the tcgen05 3xTF32 path is the
// planned upgrade).

#include <cstdlib>

#include "sped_common.cuh"

namespace sped {
namespace {

constexpr int GT = 64;       // output tile
constexpr int GROWS = 32;    // rows per staged slab
constexpr int GTHREADS = 256;

__device__ __forceinline__ float z_at(const float* V, const float* M, int32_t k, int64_t r,
                                      int32_t c) {
  return c < k ? V[r * k + c] : M[r * k + (c - k)];
}

__global__ void __launch_bounds__(GTHREADS) gram_partial_kernel(
    int64_t n, int32_t k, int32_t K2, const float* __restrict__ V, const float* __restrict__ M,
    const int2* __restrict__ tiles, int64_t rows_per_split, double* __restrict__ partial) {
  __shared__ float sa[GROWS][GT + 4];
  __shared__ float sb[GROWS][GT + 4];
  const int2 tile = tiles[blockIdx.x];
  const int ti = tile.x * GT, tj = tile.y * GT;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_split;
  const int64_t r1 = min(n, r0 + rows_per_split);
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int64_t rb = r0; rb < r1; rb += GROWS) {
    // stage GROWS x GT of column tiles ti and tj
    for (int idx = threadIdx.x; idx < GROWS * GT; idx += GTHREADS) {
      const int rr = idx / GT, cc = idx % GT;
      const int64_t r = rb + rr;
      float va = 0.f, vb = 0.f;
      if (r < r1) {
        if (ti + cc < K2) va = z_at(V, M, k, r, ti + cc);
        if (tj + cc < K2) vb = z_at(V, M, k, r, tj + cc);
      }
      sa[rr][cc] = va;
      sb[rr][cc] = vb;
    }
    __syncthreads();
    float f[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) f[i][j] = 0.f;
#pragma unroll 8
    for (int rr = 0; rr < GROWS; ++rr) {
      const float4 a = *reinterpret_cast<const float4*>(&sa[rr][ty * 4]);
      const float4 b = *reinterpret_cast<const float4*>(&sb[rr][tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w};
      const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) f[i][j] = fmaf(av[i], bv[j], f[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] += (double)f[i][j];
    __syncthreads();
  }
  double* out = partial + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * GT * GT;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) out[(ty * 4 + i) * GT + tx * 4 + j] = acc[i][j];
}

// Sum partial tiles over splits (split order) and scatter into S, C, Q.
__global__ void gram_reduce_kernel(int32_t k, int32_t K2, const int2* __restrict__ tiles,
                                   int32_t ntiles, int32_t splits,
                                   const double* __restrict__ partial, double* __restrict__ G) {
  const int t = blockIdx.x;
  const int2 tile = tiles[t];
  for (int e = threadIdx.x; e < GT * GT; e += blockDim.x) {
    const int i = tile.x * GT + e / GT, j = tile.y * GT + e % GT;
    if (i >= K2 || j >= K2 || j < i) continue;
    double s = 0.0;
    for (int sp = 0; sp < splits; ++sp) s += partial[((int64_t)sp * ntiles + t) * GT * GT + e];
    // (i, j) of Z^T Z with i <= j; write it and its mirror into S/C/Q
    auto put = [&](int a, int b, double val) {
      if (a < k && b < k) G[a * k + b] = val;                           // S
      else if (a < k && b >= k) G[k * k + a * k + (b - k)] = val;       // C = V^T M
      else if (a >= k && b >= k) G[2 * k * k + (a - k) * k + (b - k)] = val;  // Q
    };
    put(i, j, s);
    if (i != j) put(j, i, s);
  }
}

__global__ void tiles_init(int2* tiles, int nt) {
  int c = 0;
  for (int i = 0; i < nt; ++i)
    for (int j = i; j < nt; ++j) tiles[c++] = make_int2(i, j);
}

void gram_geometry(int64_t n, int32_t k, bool with_m, int* ntiles, int* splits,
                   int64_t* rows_per_split) {
  const int K2 = with_m ? 2 * k : k;
  const int nt = (K2 + GT - 1) / GT;
  *ntiles = nt * (nt + 1) / 2;
  const int target = num_sms() * 4;
  int64_t sp = (target + *ntiles - 1) / *ntiles;
  int64_t rps = (n + sp - 1) / sp;
  if (rps < 256) rps = 256;
  rps = (rps + GROWS - 1) / GROWS * GROWS;
  *rows_per_split = rps;
  *splits = (int)((n + rps - 1) / rps);
  if (*splits < 1) *splits = 1;
}

}  // namespace

bool gram_tc_supported(int32_t k, bool with_m);
size_t gram_tc_workspace(int64_t n, int32_t k);
int gram_tc(int64_t n, int32_t k, const float* V, const float* M, double* G, void* ws,
            cudaStream_t s, bool diag_q);

static bool use_tc(int32_t k, bool with_m) { return gram_tc_supported(k, with_m); }

}  // namespace sped

using namespace sped;

extern "C" size_t sped_gram_workspace_bytes(int64_t n, int32_t k) {
  size_t best = gram_tc_supported(k, true) ? gram_tc_workspace(n, k) : 0;
  for (int wm = 0; wm < 2; ++wm) {
    int ntiles, splits;
    int64_t rps;
    gram_geometry(n, k, wm == 1, &ntiles, &splits, &rps);
    size_t b = 256 + sizeof(int2) * ntiles + sizeof(double) * (size_t)splits * ntiles * GT * GT;
    if (b > best) best = b;
  }
  return best;
}

static int gram_impl(int64_t n, int32_t k, const float* V, const float* M, double* G,
                     void* workspace, size_t workspace_bytes, sped_stream_t stream, bool diag_q) {
  SPED_CHECK_ARG(n >= 1 && k >= 1 && V && G && workspace, "bad gram arguments");
  cudaStream_t s = as_stream(stream);
  const bool with_m = (M != nullptr);
  if (use_tc(k, with_m)) {
    SPED_CHECK_ARG(workspace_bytes >= gram_tc_workspace(n, k), "gram workspace too small");
    return gram_tc(n, k, V, M, G, workspace, s, diag_q);
  }
  const int K2 = with_m ? 2 * k : k;
  int ntiles, splits;
  int64_t rps;
  gram_geometry(n, k, with_m, &ntiles, &splits, &rps);
  const size_t need = 256 + sizeof(int2) * ntiles + sizeof(double) * (size_t)splits * ntiles * GT * GT;
  SPED_CHECK_ARG(workspace_bytes >= need, "gram workspace too small (%zu < %zu)", workspace_bytes,
                 need);
  int2* tiles = reinterpret_cast<int2*>(workspace);
  double* partial = reinterpret_cast<double*>(
      (reinterpret_cast<uintptr_t>(tiles + ntiles) + 255) & ~uintptr_t(255));
  const int nt = (K2 + GT - 1) / GT;
  tiles_init<<<1, 1, 0, s>>>(tiles, nt);
  SPED_LAUNCH_CHECK();
  if (!with_m) SPED_CUDA(cudaMemsetAsync(G, 0, sizeof(double) * k * k, s));
  dim3 grid(ntiles, splits);
  gram_partial_kernel<<<grid, GTHREADS, 0, s>>>(n, k, K2, V, with_m ? M : V, tiles, rps, partial);
  SPED_LAUNCH_CHECK();
  gram_reduce_kernel<<<ntiles, 256, 0, s>>>(k, K2, tiles, ntiles, splits, partial, G);
  SPED_LAUNCH_CHECK();
  return SPED_OK;
}

extern "C" int sped_gram(int64_t n, int32_t k, const float* V, const float* M, double* G,
                         void* workspace, size_t workspace_bytes, sped_stream_t stream) {
  return gram_impl(n, k, V, M, G, workspace, workspace_bytes, stream, false);
}

// mu-EG needs S, C and only diag(Q): at k = 128 the tensor-core kernel then
// skips the Q MMA group (off-diagonal Q entries are returned as 0); other k
// compute the full Q as sped_gram.
extern "C" int sped_gram_mueg(int64_t n, int32_t k, const float* V, const float* M, double* G,
                              void* workspace, size_t workspace_bytes, sped_stream_t stream) {
  SPED_CHECK_ARG(M != nullptr, "sped_gram_mueg needs M");
  return gram_impl(n, k, V, M, G, workspace, workspace_bytes, stream, true);
}
