// K7: whole mu-EigenGame steps for small/medium graphs in ONE cooperative
// (grid-resident) launch.
//
// Configs 1-2 of BASELINE move 0.04-0.6 MB per polynomial term: the
// multi-kernel step is launch/drain bound (~21 dependent kernels per step,
// ~9 us each even under CUDA-graph replay).  Here one CTA per SM stays
// resident for `steps` complete steps and the phases are separated by grid
// barriers instead of kernel boundaries:
//
//   term 0 .. T-1   w' = a x + b L w + g w   (final: lam_f x + s w')
//                   -- grid barrier between terms (rows gather neighbours)
//   Gram partials   each CTA owns a contiguous, nnz-balanced row range for
//                   EVERY phase, so after the final term it can form its
//                   partial S = X^T X (upper), C = X^T M, diag Q = M^T M from
//                   its own rows with only a CTA barrier  -- grid barrier
//   reduce          one warp per Gram entry, fixed order (deterministic)
//                   -- grid barrier
//   coeffs+update   every CTA derives A and the column scales from the fp64
//                   Gram (redundantly: O(k^3) flops, no extra barrier) and
//                   writes X' = (X A + eta M) diag(scale) for its own rows
//                   -- grid barrier
//
// T + 2 grid barriers per step.
//
// Same arithmetic as the multi-kernel path (spmm.cu term schedule; mu-EG in
// Gram form, solvers.py:121-144 / SURVEY §8a; zero-norm columns flagged for
// the host's re-randomisation, solvers.py:136-143).  Every read of a block
// written inside the launch goes through ld.global.cg: a 32-B L1 sector can
// straddle two CTAs' row ranges, so no block data is ever cached in L1.

#include <cooperative_groups.h>

#include "sped_common.cuh"

namespace cg = cooperative_groups;

namespace sped {
namespace {

constexpr int PT_THREADS = 1024;
constexpr int PT_MAX_K = 32;
constexpr int PT_MAX_TERMS = 64;
constexpr int PT_STAGE_BYTES = 96 * 1024;  // dynamic smem for staged own rows

struct PArgs {
  int32_t n, k, nterms;
  const int32_t* indptr;
  const int32_t* indices;
  const float* values;  // NULL = implicit unit-weight combinatorial
  float alpha[PT_MAX_TERMS], beta[PT_MAX_TERMS], gamma[PT_MAX_TERMS];
  float w0, lamf, sfin;
  double eta;
  int32_t steps;
  float* V;  // in/out
  float* B0;
  float* B1;
  double* partials;  // [grid][nE]
  double* G;         // [nE]
  int32_t* flag;
};

// Gram entry e -> (column a, column b): S upper triangle (row-major), then
// C (k x k), then diag Q (the small_solver.cu order).
__device__ __forceinline__ void entry_cols(int e, int k, int nS, int nC, int& ca, int& cb) {
  if (e < nS) {
    int rem = e, ia = 0;
    while (rem >= k - ia) {
      rem -= k - ia;
      ++ia;
    }
    ca = ia;
    cb = ia + rem;
  } else if (e < nS + nC) {
    ca = (e - nS) / k;
    cb = (e - nS) % k;
  } else {
    ca = cb = e - nS - nC;
  }
}

__device__ __forceinline__ int row_lower_bound(const int32_t* indptr, int n, int64_t target) {
  int lo = 0, hi = n;  // first row r with indptr[r] >= target
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if ((int64_t)__ldg(indptr + mid) < target)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(PT_THREADS, 1) persistent_mueg_kernel(const PArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ float stage[];  // own rows of X and M for the Gram partials
  __shared__ double Gs[2 * PT_MAX_K * PT_MAX_K + PT_MAX_K];  // S, C, diag Q
  __shared__ float Acoef[PT_MAX_K * PT_MAX_K];
  __shared__ float scale[PT_MAX_K];

  const int n = a.n, k = a.k, tid = threadIdx.x;
  const int nb = gridDim.x, b = blockIdx.x;
  const int64_t nnz = __ldg(a.indptr + n);
  // nnz-balanced contiguous row range, identical for every phase
  const int r0 = (b == 0) ? 0 : row_lower_bound(a.indptr, n, nnz * b / nb);
  const int r1 = (b == nb - 1) ? n : row_lower_bound(a.indptr, n, nnz * (b + 1) / nb);
  const int64_t i0 = (int64_t)r0 * k, i1 = (int64_t)r1 * k;
  const int nS = k * (k + 1) / 2, nC = k * k, nE = nS + nC + k;
  const int stage_rows = max(1, PT_STAGE_BYTES / (int)(2 * sizeof(float) * k));
  const bool has_vals = (a.values != nullptr);
  const float eta_f = (float)a.eta;

  float* X = a.V;
  float* bufs[3] = {a.V, a.B0, a.B1};
  int xi = 0;  // which of bufs holds X

  for (int step = 0; step < a.steps; ++step) {
    float* P0 = bufs[(xi + 1) % 3];
    float* P1 = bufs[(xi + 2) % 3];
    // ---- M = p(L) X ---------------------------------------------------------
    const float* win = X;
    float* M = P0;
    for (int t = 0; t < a.nterms; ++t) {
      const bool final = (t == a.nterms - 1);
      float* wout = (t & 1) ? P1 : P0;
      const float sc = (t == 0) ? a.w0 : 1.f;
      const float al = a.alpha[t], be = a.beta[t] * sc, ga = a.gamma[t] * sc;
      for (int64_t i = i0 + tid; i < i1; i += PT_THREADS) {
        const int r = (int)(i / k), c = (int)(i - (int64_t)r * k);
        const int rb = __ldg(a.indptr + r), re = __ldg(a.indptr + r + 1);
        float acc0 = 0.f, acc1 = 0.f;
        int p = rb;
        for (; p + 1 < re; p += 2) {  // two independent gather chains
          const int c0 = __ldg(a.indices + p), c1 = __ldg(a.indices + p + 1);
          const float v0 = has_vals ? __ldg(a.values + p) : (c0 == r ? (float)(re - rb - 1) : -1.f);
          const float v1 = has_vals ? __ldg(a.values + p + 1) : (c1 == r ? (float)(re - rb - 1) : -1.f);
          acc0 = fmaf(v0, __ldcg(win + (int64_t)c0 * k + c), acc0);
          acc1 = fmaf(v1, __ldcg(win + (int64_t)c1 * k + c), acc1);
        }
        if (p < re) {
          const int c0 = __ldg(a.indices + p);
          const float v0 = has_vals ? __ldg(a.values + p) : (c0 == r ? (float)(re - rb - 1) : -1.f);
          acc0 = fmaf(v0, __ldcg(win + (int64_t)c0 * k + c), acc0);
        }
        float o = be * (acc0 + acc1);
        if (al != 0.f) o = fmaf(al, __ldcg(X + i), o);
        if (ga != 0.f) o = fmaf(ga, __ldcg(win + i), o);
        if (final) o = fmaf(a.lamf, __ldcg(X + i), a.sfin * o);
        wout[i] = o;
      }
      win = wout;
      M = wout;
      if (!final) grid.sync();
    }
    if (a.nterms == 0) {
      M = P0;
      for (int64_t i = i0 + tid; i < i1; i += PT_THREADS) M[i] = (a.lamf + a.sfin * a.w0) * __ldcg(X + i);
    }
    float* Xn = (M == P0) ? P1 : P0;  // free buffer for X'
    __syncthreads();                  // own rows of M complete

    // ---- Gram partials over own rows (fp64 accumulation, fixed order) ------
    {
      float* sX = stage;
      float* sM = stage + (size_t)stage_rows * k;
      double acc0 = 0.0, acc1 = 0.0;  // entries tid and tid + PT_THREADS
      for (int rr = r0; rr < r1; rr += stage_rows) {
        const int nr = min(stage_rows, r1 - rr);
        for (int i = tid; i < nr * k; i += PT_THREADS) {
          sX[i] = __ldcg(X + (int64_t)rr * k + i);
          sM[i] = __ldcg(M + (int64_t)rr * k + i);
        }
        __syncthreads();
        for (int e = tid, slot = 0; e < nE; e += PT_THREADS, ++slot) {
          int ca, cb;
          entry_cols(e, k, nS, nC, ca, cb);
          const float* P = (e < nS + nC) ? sX : sM;
          const float* R = (e < nS) ? sX : sM;
          double s = 0.0;
          for (int r = 0; r < nr; ++r) s += (double)P[r * k + ca] * (double)R[r * k + cb];
          if (slot == 0)
            acc0 += s;
          else
            acc1 += s;
        }
        __syncthreads();
      }
      if (tid < nE) a.partials[(size_t)b * nE + tid] = acc0;
      if (tid + PT_THREADS < nE) a.partials[(size_t)b * nE + tid + PT_THREADS] = acc1;
    }
    grid.sync();

    // ---- reduce: one warp per entry, fixed lane order + shuffle tree ------
    {
      const int warp = (b * PT_THREADS + tid) >> 5, lane = tid & 31;
      const int nwarps = nb * (PT_THREADS / 32);
      for (int e = warp; e < nE; e += nwarps) {
        double s = 0.0;
        for (int q = lane; q < nb; q += 32) s += __ldcg(a.partials + (size_t)q * nE + e);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
        if (lane == 0) a.G[e] = s;
      }
    }
    grid.sync();

    // ---- coefficients (every CTA, fp64) ------------------------------------
    for (int e = tid; e < nE; e += PT_THREADS) {
      int ca, cb;
      entry_cols(e, k, nS, nC, ca, cb);
      const double g = __ldcg(a.G + e);
      if (e < nS) {
        Gs[ca * k + cb] = g;
        Gs[cb * k + ca] = g;
      } else if (e < nS + nC) {
        Gs[k * k + ca * k + cb] = g;
      } else {
        Gs[2 * k * k + ca] = g;
      }
    }
    __syncthreads();
    if (tid < k) {
      const int i = tid;
      const double* S = Gs;
      const double* C = Gs + k * k;
      const double eta = a.eta;
      double d = C[i * k + i];
      for (int j = 0; j < i; ++j) d -= S[i * k + j] * C[j * k + i];
      double acol[PT_MAX_K];
      for (int r = 0; r < k; ++r)
        acol[r] = (r < i) ? -eta * C[r * k + i] : (r == i ? 1.0 - eta * d : 0.0);
      double nrm2 = eta * eta * Gs[2 * k * k + i];
      for (int bb = 0; bb <= i; ++bb) {
        double sa = 0.0;
        for (int r = 0; r <= i; ++r) sa += S[bb * k + r] * acol[r];
        nrm2 += acol[bb] * sa + 2.0 * eta * acol[bb] * C[bb * k + i];
      }
      for (int r = 0; r < k; ++r) Acoef[r * k + i] = (float)acol[r];
      const double nrm = nrm2 > 0.0 ? sqrt(nrm2) : 0.0;
      if (!(nrm >= 1e-12)) {
        if (b == 0) atomicExch(a.flag, 1);
        scale[i] = 0.f;
      } else {
        scale[i] = (float)(1.0 / nrm);
      }
    }
    __syncthreads();

    // ---- update own rows: X' = (X A + eta M) diag(scale) ------------------
    for (int64_t i = i0 + tid; i < i1; i += PT_THREADS) {
      const int r = (int)(i / k), c = (int)(i - (int64_t)r * k);
      const float* xr = X + (int64_t)r * k;
      float acc = 0.f;
      for (int q = 0; q <= c; ++q) acc = fmaf(__ldcg(xr + q), Acoef[q * k + c], acc);
      Xn[i] = fmaf(eta_f, __ldcg(M + i), acc) * scale[c];
    }
    X = Xn;
    xi = (Xn == bufs[(xi + 1) % 3]) ? (xi + 1) % 3 : (xi + 2) % 3;
    grid.sync();
  }
  if (X != a.V)
    for (int64_t i = i0 + tid; i < i1; i += PT_THREADS) a.V[i] = __ldcg(X + i);
}

}  // namespace
}  // namespace sped

using namespace sped;

extern "C" int sped_persistent_workspace_bytes(int32_t n, int32_t k, int64_t* bytes) {
  SPED_CHECK_ARG(n >= 1 && k >= 1 && bytes, "bad persistent workspace arguments");
  const int64_t nE = (int64_t)k * (k + 1) / 2 + (int64_t)k * k + k;
  *bytes = 2 * (int64_t)n * k * (int64_t)sizeof(float) +
           ((int64_t)num_sms() + 1) * nE * (int64_t)sizeof(double) + 256;
  return SPED_OK;
}

extern "C" int sped_persistent_mueg(int32_t n, int32_t k, const int32_t* indptr,
                                    const int32_t* indices, const float* values, int32_t n_terms,
                                    const double* alpha, const double* beta, const double* gamma,
                                    double w0_scale, double lam_f, double s_final, double eta,
                                    int32_t steps, float* V, int32_t* flag, void* workspace,
                                    int64_t workspace_bytes, sped_stream_t stream) {
  SPED_CHECK_ARG(n >= 1 && k >= 1 && V && flag && indptr && indices && workspace && steps >= 0,
                 "bad persistent_mueg arguments");
  if (k > PT_MAX_K || n_terms > PT_MAX_TERMS) {
    set_error("persistent solver supports k <= %d and <= %d terms", PT_MAX_K, PT_MAX_TERMS);
    return SPED_ERR_UNSUPPORTED;
  }
  int64_t need = 0;
  sped_persistent_workspace_bytes(n, k, &need);
  SPED_CHECK_ARG(workspace_bytes >= need, "persistent workspace too small (%lld < %lld)",
                 (long long)workspace_bytes, (long long)need);
  if (steps == 0) return SPED_OK;
  static bool attr = false;
  if (!attr) {
    SPED_CUDA(cudaFuncSetAttribute(persistent_mueg_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, PT_STAGE_BYTES));
    attr = true;
  }
  int per_sm = 0;
  SPED_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, persistent_mueg_kernel,
                                                          PT_THREADS, PT_STAGE_BYTES));
  if (per_sm < 1) {
    set_error("persistent solver kernel cannot be resident");
    return SPED_ERR_CUDA;
  }
  // one CTA per SM, but never more CTAs than there are rows
  const int grid = (int)std::min<int64_t>(num_sms(), n);
  const int64_t nE = (int64_t)k * (k + 1) / 2 + (int64_t)k * k + k;
  PArgs a;
  a.n = n;
  a.k = k;
  a.nterms = n_terms;
  a.indptr = indptr;
  a.indices = indices;
  a.values = values;
  for (int t = 0; t < n_terms; ++t) {
    a.alpha[t] = (float)alpha[t];
    a.beta[t] = (float)beta[t];
    a.gamma[t] = (float)gamma[t];
  }
  a.w0 = (float)w0_scale;
  a.lamf = (float)lam_f;
  a.sfin = (float)s_final;
  a.eta = eta;
  a.steps = steps;
  a.V = V;
  char* ws = static_cast<char*>(workspace);
  a.B0 = reinterpret_cast<float*>(ws);
  a.B1 = a.B0 + (size_t)n * k;
  size_t off = 2 * (size_t)n * k * sizeof(float);
  off = (off + 255) & ~size_t(255);
  a.partials = reinterpret_cast<double*>(ws + off);
  a.G = a.partials + (size_t)grid * nE;
  a.flag = flag;
  void* args[] = {&a};
  SPED_CUDA(cudaLaunchCooperativeKernel((const void*)persistent_mueg_kernel, dim3(grid),
                                        dim3(PT_THREADS), args, PT_STAGE_BYTES,
                                        as_stream(stream)));
  return SPED_OK;
}
