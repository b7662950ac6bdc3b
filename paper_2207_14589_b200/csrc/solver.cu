// K6 + k x k algebra of the solver step.
//
// mu-EigenGame (mu_eg_step, solvers.py:121-144) in Gram form (SURVEY 8a,
// verified to 1.2e-16 in fp64):  with S = V^T V, C = V^T MV, Q = MV^T MV,
//   U = triu(C, 1);  d_i = C_ii - (S U)_ii;  A = I - eta (U + diag d)
//   ||W_i||^2 = (A^T S A)_ii + 2 eta (A^T C)_ii + eta^2 Q_ii
//   V' = (V A + eta MV) diag(1/||W_i||)
// so one step is: Gram pass (gram.cu) -> this k x k kernel -> one update
// pass (block_update below).  No extra pass for the column norms.
//
// Oja (oja_step + MGS _orthonormalize, solvers.py:84-118) in CholQR2 form:
//   W = V + eta MV, Gram(W) = S + eta (C + C^T) + eta^2 Q = R^T R,
//   W1 = W R^{-1}, then one more Gram/Cholesky pass on W1 (CholQR2 equals
//   MGS's Q to 3.5e-17 in fp64, SURVEY finding 8).
//
// All k x k algebra runs on the device in fp64 so the whole step can be
// captured in one CUDA graph (no host round trip).

#include <cstdlib>

#include "async_copy.cuh"
#include "sped_common.cuh"

namespace sped {
namespace {

__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = (lane < (int)(blockDim.x >> 5)) ? red[lane] : 0.0;
    for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
    if (lane == 0) red[0] = t;
  }
  __syncthreads();
  t = red[0];
  __syncthreads();
  return t;
}

// one CTA per column i
__global__ void mueg_coeffs_kernel(int32_t k, const double* __restrict__ G, double eta,
                                   float* __restrict__ A, float* __restrict__ scale,
                                   int32_t* __restrict__ flag) {
  extern __shared__ double acol[];  // column i of A (k doubles)
  __shared__ double red[32];
  const int i = blockIdx.x;
  const double* S = G;
  const double* C = G + (int64_t)k * k;
  const double* Q = G + 2 * (int64_t)k * k;
  // d_i = C_ii - sum_{j<i} S_ij C_ji
  double part = 0.0;
  for (int j = threadIdx.x; j < i; j += blockDim.x) part += S[(int64_t)i * k + j] * C[(int64_t)j * k + i];
  const double d = C[(int64_t)i * k + i] - block_sum(part, red);
  // column i of A
  for (int a = threadIdx.x; a < k; a += blockDim.x) {
    double v;
    if (a < i) v = -eta * C[(int64_t)a * k + i];
    else if (a == i) v = 1.0 - eta * d;
    else v = 0.0;
    acol[a] = v;
    A[(int64_t)a * k + i] = (float)v;
  }
  __syncthreads();
  // ||W_i||^2 = sum_b A_bi (S A)_bi + 2 eta sum_a A_ai C_ai + eta^2 Q_ii
  part = 0.0;
  for (int b = threadIdx.x; b <= i; b += blockDim.x) {
    double sa = 0.0;
    for (int a = 0; a <= i; ++a) sa += S[(int64_t)b * k + a] * acol[a];
    part += acol[b] * sa + 2.0 * eta * acol[b] * C[(int64_t)b * k + i];
  }
  const double nrm2 = block_sum(part, red) + eta * eta * Q[(int64_t)i * k + i];
  if (threadIdx.x == 0) {
    const double nrm = nrm2 > 0.0 ? sqrt(nrm2) : 0.0;
    if (!(nrm >= 1e-12)) {
      atomicExch(flag, 1);
      scale[i] = 0.f;
    } else {
      scale[i] = (float)(1.0 / nrm);
    }
  }
}

// single CTA: Cholesky of the (combined) Gram and the inverse of R
// (R lives in dynamic shared memory, k <= 160).
__global__ void oja_coeffs_kernel(int32_t k, const double* __restrict__ G, double eta,
                                  int32_t with_m, float* __restrict__ T,
                                  int32_t* __restrict__ flag) {
  extern __shared__ double R[];
  const double* S = G;
  const double* C = G + (int64_t)k * k;
  const double* Q = G + 2 * (int64_t)k * k;
  const int64_t kk = (int64_t)k * k;
  for (int64_t e = threadIdx.x; e < kk; e += blockDim.x) {
    const int64_t a = e / k, b = e % k;
    double g = S[e];
    if (with_m) g += eta * (C[a * k + b] + C[b * k + a]) + eta * eta * Q[e];
    R[e] = g;
  }
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  // upper Cholesky in place: Gram = R^T R, R upper triangular
  for (int j = 0; j < k; ++j) {
    if (threadIdx.x == 0) {
      double djj = R[(int64_t)j * k + j];
      for (int a = 0; a < j; ++a) djj -= R[(int64_t)a * k + j] * R[(int64_t)a * k + j];
      if (!(djj > 1e-24)) {
        bad = 1;
        djj = 1.0;
      }
      R[(int64_t)j * k + j] = sqrt(djj);
    }
    __syncthreads();
    const double rjj = R[(int64_t)j * k + j];
    for (int l = j + 1 + threadIdx.x; l < k; l += blockDim.x) {
      double v = R[(int64_t)j * k + l];
      for (int a = 0; a < j; ++a) v -= R[(int64_t)a * k + j] * R[(int64_t)a * k + l];
      R[(int64_t)j * k + l] = v / rjj;
    }
    __syncthreads();
  }
  // T = R^{-1} (upper): column l by back substitution, one thread per column.
  // T[a][l] (a < l) is kept in fp64 in R's unused strict lower triangle at
  // R[l][a]; the diagonal T[l][l] = 1/R[l][l].
  for (int l = threadIdx.x; l < k; l += blockDim.x) {
    const double tll = 1.0 / R[(int64_t)l * k + l];
    for (int i = l - 1; i >= 0; --i) {
      double acc = -R[(int64_t)i * k + l] * tll;
      for (int a = i + 1; a < l; ++a) acc -= R[(int64_t)i * k + a] * R[(int64_t)l * k + a];
      R[(int64_t)l * k + i] = acc / R[(int64_t)i * k + i];
    }
  }
  __syncthreads();
  for (int64_t e = threadIdx.x; e < kk; e += blockDim.x) {
    const int64_t i = e / k, l = e % k;
    double t = 0.0;
    if (i == l) t = 1.0 / R[i * k + i];
    else if (i < l) t = R[l * k + i];
    T[e] = (float)t;
  }
  if (threadIdx.x == 0 && bad) atomicExch(flag, 1);
}

// out = (P A + M B) diag(scale); register-tiled for K in {16,32,64,128}:
// 64-row tiles, each thread owns RPT rows x 4 consecutive columns.
template <int K>
__global__ void __launch_bounds__(256) block_update_kernel(
    int64_t n, const float* __restrict__ P, const float* __restrict__ A,
    const float* __restrict__ M, const float* __restrict__ B, float eta,
    const float* __restrict__ scale, float* __restrict__ out) {
  constexpr int TR = 64;
  constexpr int CG = K / 4;          // column groups
  constexpr int RG = 256 / CG;       // row groups
  constexpr int RPT = TR / RG;       // rows per thread
  extern __shared__ float4 smem4[];
  float* As = reinterpret_cast<float*>(smem4);          // K*K
  float* Bs = As + K * K;                               // K*K (if B)
  float* Ps = Bs + (B ? K * K : 0);                     // TR*(K+1)
  float* Ms = Ps + TR * (K + 1);                        // TR*(K+1) (if M && B)
  for (int e = threadIdx.x; e < K * K; e += 256) {
    As[e] = A[e];
    if (B) Bs[e] = B[e];
  }
  const int cg = threadIdx.x % CG, rg = threadIdx.x / CG;
  float4 sc = make_float4(1.f, 1.f, 1.f, 1.f);
  if (scale) sc = *reinterpret_cast<const float4*>(scale + cg * 4);
  const int64_t ntiles = (n + TR - 1) / TR;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * TR;
    __syncthreads();
    for (int e = threadIdx.x; e < TR * K; e += 256) {
      const int rr = e / K, cc = e % K;
      const int64_t r = r0 + rr;
      Ps[rr * (K + 1) + cc] = r < n ? P[r * K + cc] : 0.f;
      if (M && B) Ms[rr * (K + 1) + cc] = r < n ? M[r * K + cc] : 0.f;
    }
    __syncthreads();
    float4 acc[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
    for (int a = 0; a < K; ++a) {
      const float4 av = *reinterpret_cast<const float4*>(As + a * K + cg * 4);
#pragma unroll
      for (int i = 0; i < RPT; ++i) acc[i] = f4_fma(Ps[(rg + i * RG) * (K + 1) + a], av, acc[i]);
    }
    if (M && B) {
#pragma unroll 4
      for (int a = 0; a < K; ++a) {
        const float4 bv = *reinterpret_cast<const float4*>(Bs + a * K + cg * 4);
#pragma unroll
        for (int i = 0; i < RPT; ++i) acc[i] = f4_fma(Ms[(rg + i * RG) * (K + 1) + a], bv, acc[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int64_t r = r0 + rg + i * RG;
      if (r >= n) continue;
      float4 v = acc[i];
      if (M && !B) v = f4_fma(eta, *reinterpret_cast<const float4*>(M + r * K + cg * 4), v);
      v = make_float4(v.x * sc.x, v.y * sc.y, v.z * sc.z, v.w * sc.w);
      *reinterpret_cast<float4*>(out + r * K + cg * 4) = v;
    }
  }
}

// Row-streaming update: one thread owns (row, 32-column block) and keeps its
// 32 outputs in registers; the input rows are read as float4s (each thread
// walks its row, neighbouring chunks hit L1), A / B come from shared memory
// as float4 broadcasts.  UPPER: A is upper triangular (mu-EG: I - eta(U +
// diag d)), so column block cb only needs rows i < 32*(cb+1).  Memory bound:
// reads P (+ M) once, writes out once.
template <int K, bool UPPER>
__global__ void __launch_bounds__(256) block_update_rows(
    int64_t n, const float* __restrict__ P, const float* __restrict__ A,
    const float* __restrict__ M, const float* __restrict__ B, float eta,
    const float* __restrict__ scale, float* __restrict__ out) {
  constexpr int NB = K / 32;  // column blocks per row
  extern __shared__ float4 rows_smem4[];
  float* As = reinterpret_cast<float*>(rows_smem4);
  float* Bs = As + K * K;  // only when B (dynamic size covers it)
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
    As[e] = A[e];
    if (B) Bs[e] = B[e];
  }
  __syncthreads();
  const int64_t total = n * NB;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = t / NB;
    const int cb = (int)(t % NB);
    float acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = 0.f;
    const float* prow = P + row * K;
    const int ilim = UPPER ? 32 * (cb + 1) : K;
#pragma unroll 1
    for (int i4 = 0; i4 < ilim; i4 += 4) {
      const float4 pv = __ldg(reinterpret_cast<const float4*>(prow + i4));
      const float pvv[4] = {pv.x, pv.y, pv.z, pv.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float* arow = As + (i4 + q) * K + cb * 32;
#pragma unroll
        for (int j4 = 0; j4 < 32; j4 += 4) {
          const float4 a4 = *reinterpret_cast<const float4*>(arow + j4);
          acc[j4 + 0] = fmaf(pvv[q], a4.x, acc[j4 + 0]);
          acc[j4 + 1] = fmaf(pvv[q], a4.y, acc[j4 + 1]);
          acc[j4 + 2] = fmaf(pvv[q], a4.z, acc[j4 + 2]);
          acc[j4 + 3] = fmaf(pvv[q], a4.w, acc[j4 + 3]);
        }
      }
    }
    if (M && B) {
      const float* mrow = M + row * K;
      const float* Bsrc = Bs;
#pragma unroll 1
      for (int i4 = 0; i4 < K; i4 += 4) {
        const float4 mv = __ldg(reinterpret_cast<const float4*>(mrow + i4));
        const float mvv[4] = {mv.x, mv.y, mv.z, mv.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float* brow = Bsrc + (i4 + q) * K + cb * 32;
#pragma unroll
          for (int j4 = 0; j4 < 32; j4 += 4) {
            const float4 b4 = *reinterpret_cast<const float4*>(brow + j4);
            acc[j4 + 0] = fmaf(mvv[q], b4.x, acc[j4 + 0]);
            acc[j4 + 1] = fmaf(mvv[q], b4.y, acc[j4 + 1]);
            acc[j4 + 2] = fmaf(mvv[q], b4.z, acc[j4 + 2]);
            acc[j4 + 3] = fmaf(mvv[q], b4.w, acc[j4 + 3]);
          }
        }
      }
    }
    float* orow = out + row * K + cb * 32;
    const float* mcol = M ? M + row * K + cb * 32 : nullptr;
#pragma unroll
    for (int j4 = 0; j4 < 32; j4 += 4) {
      float4 r = make_float4(acc[j4], acc[j4 + 1], acc[j4 + 2], acc[j4 + 3]);
      if (M && !B) r = f4_fma(eta, __ldg(reinterpret_cast<const float4*>(mcol + j4)), r);
      if (scale) {
        const float4 sc = *reinterpret_cast<const float4*>(scale + cb * 32 + j4);
        r = make_float4(r.x * sc.x, r.y * sc.y, r.z * sc.z, r.w * sc.w);
      }
      *reinterpret_cast<float4*>(orow + j4) = r;
    }
  }
}

// v2 update for k in {32, 64, 128}: out = (P A [+ M B | + eta M]) diag(s).
// Memory bound (reads P and M once, writes out once), so the kernel is built
// around the copy: warp 8 streams tiles of TR rows of P (and M) through a
// cp.async.bulk ring of NSTAGE shared-memory stages; warps 0-7 each take a
// row at a time, lane c owning output columns c, c+32, ... (KPL = K/32 per
// lane) with the matching columns of A (and B) held in REGISTERS.  The P row
// is read as float4 broadcasts (one shared-memory wavefront per 4 inputs),
// M and the output are coalesced 128-B rows.
template <int K>
#ifndef UPD_NSTAGE
#define UPD_NSTAGE 4
#endif
#ifndef UPD_STAGE_BYTES
#define UPD_STAGE_BYTES 16384
#endif
#ifndef UPD_CTAS
#define UPD_CTAS 2
#endif
struct UpdCfg {
  static constexpr int KPL = K / 32;
  static constexpr int NSTAGE = UPD_NSTAGE;
  static constexpr int STAGE_BYTES = UPD_STAGE_BYTES;  // P + M rows of one stage
};

// packed fp32 FMA (FFMA2 on sm_100a): acc.{lo,hi} += s * b.{lo,hi}
__device__ __forceinline__ void ffma2_s(uint64_t& acc, float s, uint64_t b) {
  uint64_t ss;
  asm("mov.b64 %0, {%1,%1};" : "=l"(ss) : "f"(s));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(ss), "l"(b));
}
__device__ __forceinline__ uint64_t pack_f2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}

template <int K, int MODE>  // MODE 0: P A; 1: P A + eta M; 2: P A + M B
__global__ void __launch_bounds__(288) block_update_v2(int64_t n, const float* __restrict__ P,
                                                      const float* __restrict__ A,
                                                      const float* __restrict__ M,
                                                      const float* __restrict__ B, float eta,
                                                      const float* __restrict__ scale,
                                                      float* __restrict__ out, int tr) {
  using namespace ::sped::async;
  constexpr int KPL = UpdCfg<K>::KPL, NS = UpdCfg<K>::NSTAGE;
  extern __shared__ __align__(128) float stage[];
  __shared__ uint64_t full[NS], empty[NS];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int stage_floats = tr * K * (MODE == 0 ? 1 : 2);
  const int64_t ntiles = (n + tr - 1) / tr;
  const int64_t my_tiles = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 256);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 8) {
    if (lane == 0) {
      for (int64_t j = 0; j < my_tiles; ++j) {
        const int st = (int)(j % NS);
        if (j >= NS) mbar_wait(&empty[st], (uint32_t)(((j / NS) - 1) & 1));
        const int64_t r0 = (blockIdx.x + j * gridDim.x) * (int64_t)tr;
        const int rows = (int)min((int64_t)tr, n - r0);
        const uint32_t bytes = (uint32_t)rows * K * 4u;
        float* dst = stage + (size_t)st * stage_floats;
        mbar_expect_tx(&full[st], (MODE == 0 ? 1u : 2u) * bytes);
        bulk_g2s(dst, P + r0 * K, bytes, &full[st]);
        if (MODE != 0) bulk_g2s(dst + tr * K, M + r0 * K, bytes, &full[st]);
      }
    }
    return;
  }
  // A (and B) columns of this lane in registers
  float a[K][KPL];
  float bm[MODE == 2 ? K : 1][KPL];
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < KPL; ++j) {
      a[i][j] = __ldg(A + i * K + lane + 32 * j);
      if (MODE == 2) bm[i][j] = __ldg(B + i * K + lane + 32 * j);
    }
  float sc[KPL];
#pragma unroll
  for (int j = 0; j < KPL; ++j) sc[j] = scale ? __ldg(scale + lane + 32 * j) : 1.f;
  for (int64_t j = 0; j < my_tiles; ++j) {
    const int st = (int)(j % NS);
    const int64_t r0 = (blockIdx.x + j * gridDim.x) * (int64_t)tr;
    const int rows = (int)min((int64_t)tr, n - r0);
    mbar_wait(&full[st], (uint32_t)((j / NS) & 1));
    const float* ps = stage + (size_t)st * stage_floats;
    const float* ms = ps + tr * K;
    // k = 32: two rows per pass (r, r + 8) reuse the A registers and
    // interleave two FMA chains; k = 64 keeps one row (register budget)
    constexpr int RB = (K == 32) ? 2 : 1;
    for (int r = warp; r < rows; r += 8 * RB) {
      const bool two = RB == 2 && (r + 8 < rows);
      const int r2 = two ? r + 8 : r;
      float acc[2][KPL];
#pragma unroll
      for (int q = 0; q < KPL; ++q) acc[0][q] = acc[1][q] = 0.f;
      const float4* prow0 = reinterpret_cast<const float4*>(ps + r * K);
      const float4* prow1 = reinterpret_cast<const float4*>(ps + r2 * K);
      if constexpr (KPL == 2 && RB == 1 && MODE != 2) {
        // k = 64: the lane's two columns (lane, lane + 32) as one packed FMA
        uint64_t accp = 0ull;
#pragma unroll
        for (int i4 = 0; i4 < K / 4; ++i4) {
          const float4 p0 = prow0[i4];
          ffma2_s(accp, p0.x, pack_f2(a[4 * i4 + 0][0], a[4 * i4 + 0][1]));
          ffma2_s(accp, p0.y, pack_f2(a[4 * i4 + 1][0], a[4 * i4 + 1][1]));
          ffma2_s(accp, p0.z, pack_f2(a[4 * i4 + 2][0], a[4 * i4 + 2][1]));
          ffma2_s(accp, p0.w, pack_f2(a[4 * i4 + 3][0], a[4 * i4 + 3][1]));
        }
        asm("mov.b64 {%0,%1}, %2;" : "=f"(acc[0][0]), "=f"(acc[0][1]) : "l"(accp));
      } else
#pragma unroll
      for (int i4 = 0; i4 < K / 4; ++i4) {
        const float4 p0 = prow0[i4];  // broadcasts
        const float4 p1 = (RB == 2) ? prow1[i4] : p0;
#pragma unroll
        for (int q = 0; q < KPL; ++q) {
          acc[0][q] = fmaf(p0.x, a[4 * i4 + 0][q], acc[0][q]);
          acc[0][q] = fmaf(p0.y, a[4 * i4 + 1][q], acc[0][q]);
          acc[0][q] = fmaf(p0.z, a[4 * i4 + 2][q], acc[0][q]);
          acc[0][q] = fmaf(p0.w, a[4 * i4 + 3][q], acc[0][q]);
          if (RB == 2) {
            acc[1][q] = fmaf(p1.x, a[4 * i4 + 0][q], acc[1][q]);
            acc[1][q] = fmaf(p1.y, a[4 * i4 + 1][q], acc[1][q]);
            acc[1][q] = fmaf(p1.z, a[4 * i4 + 2][q], acc[1][q]);
            acc[1][q] = fmaf(p1.w, a[4 * i4 + 3][q], acc[1][q]);
          }
        }
      }
      if (MODE == 2) {
        const float4* mrow0 = reinterpret_cast<const float4*>(ms + r * K);
        const float4* mrow1 = reinterpret_cast<const float4*>(ms + r2 * K);
#pragma unroll
        for (int i4 = 0; i4 < K / 4; ++i4) {
          const float4 m0 = mrow0[i4];
          const float4 m1 = (RB == 2) ? mrow1[i4] : m0;
#pragma unroll
          for (int q = 0; q < KPL; ++q) {
            acc[0][q] = fmaf(m0.x, bm[4 * i4 + 0][q], acc[0][q]);
            acc[0][q] = fmaf(m0.y, bm[4 * i4 + 1][q], acc[0][q]);
            acc[0][q] = fmaf(m0.z, bm[4 * i4 + 2][q], acc[0][q]);
            acc[0][q] = fmaf(m0.w, bm[4 * i4 + 3][q], acc[0][q]);
            if (RB == 2) {
              acc[1][q] = fmaf(m1.x, bm[4 * i4 + 0][q], acc[1][q]);
              acc[1][q] = fmaf(m1.y, bm[4 * i4 + 1][q], acc[1][q]);
              acc[1][q] = fmaf(m1.z, bm[4 * i4 + 2][q], acc[1][q]);
              acc[1][q] = fmaf(m1.w, bm[4 * i4 + 3][q], acc[1][q]);
            }
          }
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h == 1 && !two) break;
        const int rr = h ? r2 : r;
        float* orow = out + (r0 + rr) * K;
#pragma unroll
        for (int q = 0; q < KPL; ++q) {
          float o = acc[h][q];
          if (MODE == 1) o = fmaf(eta, ms[rr * K + lane + 32 * q], o);
          __stcs(orow + lane + 32 * q, o * sc[q]);
        }
      }
    }
    mbar_arrive(&empty[st]);
  }
}

// k = 32 without M*B (mu-EG / CholQR updates): half a warp per row, a lane
// owning two adjacent output columns, so every FMA is a packed FFMA2 (the P
// element as the scalar operand, the lane's two A entries as the pair): half
// the FMA instructions of the lane-per-column layout, the same per-element
// sums in the same order.  Same cp.async.bulk ring as block_update_v2.

template <int MODE>  // 0: P A; 1: P A + eta M
__global__ void __launch_bounds__(288, 2) block_update_k32_f2(int64_t n, const float* __restrict__ P,
                                                          const float* __restrict__ A,
                                                          const float* __restrict__ M, float eta,
                                                          const float* __restrict__ scale,
                                                          float* __restrict__ out, int tr) {
  using namespace ::sped::async;
  constexpr int K = 32, NS = UpdCfg<K>::NSTAGE;
  extern __shared__ __align__(128) float stage[];
  __shared__ uint64_t full[NS], empty[NS];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int stage_floats = tr * K * (MODE == 0 ? 1 : 2);
  const int64_t ntiles = (n + tr - 1) / tr;
  const int64_t my_tiles = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 256);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 8) {
    if (lane == 0) {
      for (int64_t j = 0; j < my_tiles; ++j) {
        const int st = (int)(j % NS);
        if (j >= NS) mbar_wait(&empty[st], (uint32_t)(((j / NS) - 1) & 1));
        const int64_t r0 = (blockIdx.x + j * gridDim.x) * (int64_t)tr;
        const int rows = (int)min((int64_t)tr, n - r0);
        const uint32_t bytes = (uint32_t)rows * K * 4u;
        float* dst = stage + (size_t)st * stage_floats;
        mbar_expect_tx(&full[st], (MODE == 0 ? 1u : 2u) * bytes);
        bulk_g2s(dst, P + r0 * K, bytes, &full[st]);
        if (MODE != 0) bulk_g2s(dst + tr * K, M + r0 * K, bytes, &full[st]);
      }
    }
    return;
  }
  const int hl = lane & 15, half = lane >> 4;
  uint64_t a2[K];  // {A[i][2hl], A[i][2hl+1]}
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const float2 t = __ldg(reinterpret_cast<const float2*>(A + i * K + 2 * hl));
    asm("mov.b64 %0, {%1,%2};" : "=l"(a2[i]) : "f"(t.x), "f"(t.y));
  }
  float2 sc = make_float2(1.f, 1.f);
  if (scale) sc = __ldg(reinterpret_cast<const float2*>(scale + 2 * hl));
  for (int64_t j = 0; j < my_tiles; ++j) {
    const int st = (int)(j % NS);
    const int64_t r0 = (blockIdx.x + j * gridDim.x) * (int64_t)tr;
    const int rows = (int)min((int64_t)tr, n - r0);
    mbar_wait(&full[st], (uint32_t)((j / NS) & 1));
    const float* ps = stage + (size_t)st * stage_floats;
    const float* ms = ps + tr * K;
    // a pass: 32 rows per CTA, each half-warp two rows (two FMA chains)
    for (int rb = 0; rb < rows; rb += 32) {
      const int ra = rb + warp * 2 + half, rc = ra + 16;
      const bool va = ra < rows, vc = rc < rows;
      const float4* pa = reinterpret_cast<const float4*>(ps + (va ? ra : 0) * K);
      const float4* pc = reinterpret_cast<const float4*>(ps + (vc ? rc : 0) * K);
      uint64_t acca = 0ull, accc = 0ull;
#pragma unroll
      for (int i4 = 0; i4 < K / 4; ++i4) {
        const float4 xa = pa[i4];  // one broadcast per half-warp
        const float4 xc = pc[i4];
        ffma2_s(acca, xa.x, a2[4 * i4 + 0]);
        ffma2_s(accc, xc.x, a2[4 * i4 + 0]);
        ffma2_s(acca, xa.y, a2[4 * i4 + 1]);
        ffma2_s(accc, xc.y, a2[4 * i4 + 1]);
        ffma2_s(acca, xa.z, a2[4 * i4 + 2]);
        ffma2_s(accc, xc.z, a2[4 * i4 + 2]);
        ffma2_s(acca, xa.w, a2[4 * i4 + 3]);
        ffma2_s(accc, xc.w, a2[4 * i4 + 3]);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const bool v = h ? vc : va;
        if (!v) continue;
        const int rr = h ? rc : ra;
        float2 o;
        asm("mov.b64 {%0,%1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(h ? accc : acca));
        if (MODE == 1) {
          const float2 m = *reinterpret_cast<const float2*>(ms + rr * K + 2 * hl);
          o.x = fmaf(eta, m.x, o.x);
          o.y = fmaf(eta, m.y, o.y);
        }
        __stcs(reinterpret_cast<float2*>(out + (r0 + rr) * K + 2 * hl), make_float2(o.x * sc.x, o.y * sc.y));
      }
    }
    mbar_arrive(&empty[st]);
  }
}

template <int K>
int launch_v2(int64_t n, const float* P, const float* A, const float* M, const float* B, float eta,
              const float* scale, float* out, cudaStream_t s) {
  using C = UpdCfg<K>;
  const int mode = M ? (B ? 2 : 1) : 0;
  const int tr = C::STAGE_BYTES / (K * 4 * (mode == 0 ? 1 : 2));
  const size_t smem = (size_t)C::NSTAGE * C::STAGE_BYTES;
  // register budget: A (and B) columns live in registers, so k = 64 with
  // M*B (Oja) takes the row-streaming kernel
  static PerDeviceOnce attr;  // per device: function attributes are per context
  {
    const int rc_ = attr([&]() -> int {
      SPED_CUDA(cudaFuncSetAttribute(block_update_v2<K, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      SPED_CUDA(cudaFuncSetAttribute(block_update_v2<K, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      if constexpr (K == 32) {
        SPED_CUDA(cudaFuncSetAttribute(block_update_v2<K, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        SPED_CUDA(cudaFuncSetAttribute(block_update_k32_f2<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        SPED_CUDA(cudaFuncSetAttribute(block_update_k32_f2<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      }
      return SPED_OK;
    });
    if (rc_ != SPED_OK) return rc_;
  }
  const int64_t ntiles = (n + tr - 1) / tr;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)num_sms() * UPD_CTAS));
  // the packed kernel reads A / scale and writes out as float2
  const bool pair_ok = ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(scale) |
                         reinterpret_cast<uintptr_t>(out)) % 8) == 0;
  if constexpr (K == 32) if (pair_ok) {
    if (mode == 0) {
      block_update_k32_f2<0><<<grid, 288, smem, s>>>(n, P, A, M, eta, scale, out, tr);
      SPED_LAUNCH_CHECK();
      return SPED_OK;
    }
    if (mode == 1) {
      block_update_k32_f2<1><<<grid, 288, smem, s>>>(n, P, A, M, eta, scale, out, tr);
      SPED_LAUNCH_CHECK();
      return SPED_OK;
    }
  }
  switch (mode) {
    case 0: block_update_v2<K, 0><<<grid, 288, smem, s>>>(n, P, A, M, B, eta, scale, out, tr); break;
    case 1: block_update_v2<K, 1><<<grid, 288, smem, s>>>(n, P, A, M, B, eta, scale, out, tr); break;
    default:
      if constexpr (K == 32) {
        block_update_v2<K, 2><<<grid, 288, smem, s>>>(n, P, A, M, B, eta, scale, out, tr);
        break;
      }
      set_error("update v2: M*B needs k = 32");
      return SPED_ERR_UNSUPPORTED;
  }
  SPED_LAUNCH_CHECK();
  return SPED_OK;
}

template <int K>
int launch_rows(int64_t n, const float* P, const float* A, const float* M, const float* B,
                float eta, const float* scale, float* out, bool upper, cudaStream_t s) {
  const int64_t total = n * (K / 32);
  const size_t smem = sizeof(float) * K * K * (B ? 2 : 1);
  static PerDeviceOnce attr;  // per device: function attributes are per context
  {
    const int rc_ = attr([&]() -> int {
      const int maxb = (int)(sizeof(float) * K * K * 2);
      SPED_CUDA(cudaFuncSetAttribute(block_update_rows<K, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, maxb));
      SPED_CUDA(cudaFuncSetAttribute(block_update_rows<K, false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, maxb));
      return SPED_OK;
    });
    if (rc_ != SPED_OK) return rc_;
  }
  int per_sm = (int)((200 * 1024) / (smem + 1024));
  per_sm = per_sm < 1 ? 1 : (per_sm > 8 ? 8 : per_sm);
  const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * per_sm);
  if (upper)
    block_update_rows<K, true><<<grid, 256, smem, s>>>(n, P, A, M, B, eta, scale, out);
  else
    block_update_rows<K, false><<<grid, 256, smem, s>>>(n, P, A, M, B, eta, scale, out);
  SPED_LAUNCH_CHECK();
  return SPED_OK;
}

// generic k: one thread per output element of a 32-row tile
__global__ void __launch_bounds__(256) block_update_generic(
    int64_t n, int32_t k, const float* __restrict__ P, const float* __restrict__ A,
    const float* __restrict__ M, const float* __restrict__ B, float eta,
    const float* __restrict__ scale, float* __restrict__ out) {
  const int64_t total = n * (int64_t)k;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total;
       o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = o / k;
    const int c = (int)(o % k);
    float acc = 0.f;
    for (int a = 0; a < k; ++a) acc = fmaf(P[r * k + a], A[(int64_t)a * k + c], acc);
    if (M) {
      if (B) {
        for (int a = 0; a < k; ++a) acc = fmaf(M[r * k + a], B[(int64_t)a * k + c], acc);
      } else {
        acc = fmaf(eta, M[o], acc);
      }
    }
    if (scale) acc *= scale[c];
    out[o] = acc;
  }
}

template <int K>
int launch_update(int64_t n, const float* P, const float* A, const float* M, const float* B,
                  float eta, const float* scale, float* out, cudaStream_t s) {
  constexpr int TR = 64;
  size_t smem = sizeof(float) * (K * K * (B ? 2 : 1) + TR * (K + 1) * ((M && B) ? 2 : 1));
  auto kern = block_update_kernel<K>;
  static PerDeviceOnce attr_set;  // per device: function attributes are per context
  {
    const int rc_ = attr_set([&]() -> int {
      SPED_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(sizeof(float) * (2 * K * K + 2 * TR * (K + 1)))));
      return SPED_OK;
    });
    if (rc_ != SPED_OK) return rc_;
  }
  const int64_t ntiles = (n + TR - 1) / TR;
  int per_sm = (int)((220 * 1024) / smem);
  if (per_sm < 1) per_sm = 1;
  if (per_sm > 8) per_sm = 8;
  unsigned grid = (unsigned)std::min<int64_t>(ntiles, (int64_t)num_sms() * per_sm);
  kern<<<grid, 256, smem, s>>>(n, P, A, M, B, eta, scale, out);
  SPED_LAUNCH_CHECK();
  return SPED_OK;
}

}  // namespace
}  // namespace sped

namespace sped {
int launch_update_tc128(int64_t n, const float* P, const float* A, const float* M, float eta,
                        const float* scale, float* out, cudaStream_t s);  // update_tc.cu
}  // namespace sped

using namespace sped;

extern "C" int sped_mueg_coeffs(int32_t k, const double* G, double eta, float* A, float* scale,
                                int32_t* flag, sped_stream_t stream) {
  SPED_CHECK_ARG(k >= 1 && G && A && scale && flag, "bad mueg_coeffs arguments");
  cudaStream_t s = as_stream(stream);
  mueg_coeffs_kernel<<<k, 128, sizeof(double) * k, s>>>(k, G, eta, A, scale, flag);
  SPED_LAUNCH_CHECK();
  return SPED_OK;
}

extern "C" int sped_oja_coeffs(int32_t k, const double* G, double eta, int32_t with_m, float* T,
                               int32_t* flag, sped_stream_t stream) {
  SPED_CHECK_ARG(k >= 1 && k <= 160 && G && T && flag, "bad oja_coeffs arguments (k <= 160)");
  cudaStream_t s = as_stream(stream);
  const size_t smem = sizeof(double) * (size_t)k * k;
  static PerDeviceOnce attr_set;  // per device: function attributes are per context
  {
    const int rc_ = attr_set([&]() -> int {
      SPED_CUDA(cudaFuncSetAttribute(oja_coeffs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(sizeof(double) * 160 * 160)));
      return SPED_OK;
    });
    if (rc_ != SPED_OK) return rc_;
  }
  oja_coeffs_kernel<<<1, 256, smem, s>>>(k, G, eta, with_m, T, flag);
  SPED_LAUNCH_CHECK();
  return SPED_OK;
}

extern "C" int sped_block_update(int64_t n, int32_t k, const float* P, const float* A,
                                 const float* M, const float* B, double eta, const float* scale,
                                 int32_t upper_flag, float* out, sped_stream_t stream) {
  SPED_CHECK_ARG(n >= 0 && k >= 1 && P && A && out, "bad block_update arguments");
  SPED_CHECK_ARG(out != P && out != M, "out must not alias inputs");
  if (n == 0) return SPED_OK;
  cudaStream_t s = as_stream(stream);
  const bool aligned = ((reinterpret_cast<uintptr_t>(P) | reinterpret_cast<uintptr_t>(out) |
                         reinterpret_cast<uintptr_t>(M) | reinterpret_cast<uintptr_t>(scale)) %
                        16) == 0;
  if (aligned) {
    const bool upper = (upper_flag != 0);
    switch (k) {
      case 16: return launch_update<16>(n, P, A, M, B, (float)eta, scale, out, s);
      case 32: return launch_v2<32>(n, P, A, M, B, (float)eta, scale, out, s);
      case 64: return (M && B) ? launch_rows<64>(n, P, A, M, B, (float)eta, scale, out, upper, s)
                               : launch_v2<64>(n, P, A, M, B, (float)eta, scale, out, s);
      case 128:
        // tcgen05 3xTF32 GEMM (update_tc.cu); the Oja M*B form streams rows
        if (M && B) return launch_rows<128>(n, P, A, M, B, (float)eta, scale, out, upper, s);
        return launch_update_tc128(n, P, A, M, (float)eta, scale, out, s);
      default: break;
    }
  }
  block_update_generic<<<grid_for(n * k, 256, num_sms() * 16), 256, 0, s>>>(n, k, P, A, M, B,
                                                                             (float)eta, scale, out);
  SPED_LAUNCH_CHECK();
  return SPED_OK;
}
