// K2: whole mu-EigenGame steps for desk-scale graphs in ONE thread block.
//
// For n*k <= SMALL_MAX_NK the solver state (V, MV and the two polynomial
// ping-pong blocks) lives in shared memory for the entire run: each launch
// performs `steps` complete steps (every polynomial term, the Gram of
// [V | MV], the k x k algebra and the update), separated only by
// __syncthreads.  This removes the ~20 kernel launches per step that bound
// configs 1-2 of BASELINE (0.2 MB per term, launch-bound).
//
// Same arithmetic as the multi-kernel path: terms w' = a*x + b*L w + g*w
// (final: lam_f*x + s*w'); mu-EG in Gram form (solvers.py:121-144, SURVEY
// §8a); column norms from the Gram, zero-norm columns flagged for the host.

#include "sped_common.cuh"

namespace sped {
namespace {

constexpr int SMALL_THREADS = 1024;
constexpr int SMALL_MAX_NK = 12288;     // 3 blocks of n*k floats = 144 KB
constexpr int SMALL_SMEM_BYTES = 190 * 1024;  // dynamic: 3 blocks + the CSR
constexpr int SMALL_MAX_K = 32;
constexpr int SMALL_MAX_TERMS = 64;

struct SmallArgs {
  int32_t n, k, nterms;
  const int32_t* indptr;
  const int32_t* indices;
  const float* values;  // NULL = implicit unit-weight combinatorial
  float alpha[SMALL_MAX_TERMS], beta[SMALL_MAX_TERMS], gamma[SMALL_MAX_TERMS];
  float w0, lamf, sfin;
  double eta;
  int32_t steps;
  float* V;             // in/out, n x k
  int32_t* flag;
};

// Gram entry e -> (column a, column b): S upper triangle (row-major), then
// C (k x k), then diag Q.
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

__device__ __forceinline__ int tid_init() { return threadIdx.x; }

__global__ void __launch_bounds__(SMALL_THREADS, 1) small_mueg_kernel(const SmallArgs a) {
  extern __shared__ float4 smem4[];
  const int n = a.n, k = a.k, nk = a.n * a.k;
  float* X = reinterpret_cast<float*>(smem4);  // V (the polynomial's x)
  float* P0 = X + nk;                          // ping-pong; the last term's output is MV
  float* P1 = P0 + nk;
  int32_t* sptr = reinterpret_cast<int32_t*>(P1 + nk);  // CSR staged in shared memory
  const int nnz = __ldg(a.indptr + n);
  int32_t* sidx = sptr + (n + 1);
  float* sval = reinterpret_cast<float*>(sidx + nnz);
  for (int i = tid_init(); i <= n; i += SMALL_THREADS) sptr[i] = __ldg(a.indptr + i);
  for (int i = tid_init(); i < nnz; i += SMALL_THREADS) {
    sidx[i] = __ldg(a.indices + i);
    if (a.values) sval[i] = __ldg(a.values + i);
  }
  float* MV = nullptr;
  __shared__ double G[3 * SMALL_MAX_K * SMALL_MAX_K];  // S, C, diag Q
  __shared__ float Acoef[SMALL_MAX_K * SMALL_MAX_K];
  __shared__ float scale[SMALL_MAX_K];
  __shared__ float part[SMALL_THREADS];
  const int tid = threadIdx.x;
  for (int i = tid; i < nk; i += SMALL_THREADS) X[i] = a.V[i];
  __syncthreads();
  const bool has_vals = (a.values != nullptr);

  const int nS = k * (k + 1) / 2;          // upper triangle of S
  const int nC = k * k;                    // all of C
  const int nE = nS + nC + k;              // + diag Q
  const int parts = max(1, SMALL_THREADS / nE);
  const int slots = SMALL_THREADS / parts;  // entries per pass

  for (int step = 0; step < a.steps; ++step) {
    // ---- MV = p(L) X -------------------------------------------------------
    const float* win = X;
    for (int t = 0; t < a.nterms; ++t) {
      const bool final = (t == a.nterms - 1);
      float* wout = (t & 1) ? P1 : P0;
      const float sc = (t == 0) ? a.w0 : 1.f;
      const float al = a.alpha[t], be = a.beta[t] * sc, ga = a.gamma[t] * sc;
      for (int i = tid; i < nk; i += SMALL_THREADS) {
        const int r = i / k, c = i - r * k;
        const int b = sptr[r], e = sptr[r + 1];
        float acc0 = 0.f, acc1 = 0.f;
        int p = b;
        for (; p + 1 < e; p += 2) {  // two independent chains
          const int c0 = sidx[p], c1 = sidx[p + 1];
          const float v0 = has_vals ? sval[p] : (c0 == r ? (float)(e - b - 1) : -1.f);
          const float v1 = has_vals ? sval[p + 1] : (c1 == r ? (float)(e - b - 1) : -1.f);
          acc0 = fmaf(v0, win[c0 * k + c], acc0);
          acc1 = fmaf(v1, win[c1 * k + c], acc1);
        }
        if (p < e) {
          const int c0 = sidx[p];
          const float v0 = has_vals ? sval[p] : (c0 == r ? (float)(e - b - 1) : -1.f);
          acc0 = fmaf(v0, win[c0 * k + c], acc0);
        }
        const float acc = acc0 + acc1;
        float o = be * acc;
        if (al != 0.f) o = fmaf(al, X[i], o);
        if (ga != 0.f) o = fmaf(ga, win[i], o);
        if (final) o = fmaf(a.lamf, X[i], a.sfin * o);
        wout[i] = o;
      }
      __syncthreads();
      win = wout;
      if (final) MV = wout;
    }
    if (a.nterms == 0) {
      MV = P0;
      for (int i = tid; i < nk; i += SMALL_THREADS) MV[i] = (a.lamf + a.sfin * a.w0) * X[i];
      __syncthreads();
    }
    float* Wa = (MV == P0) ? P1 : P0;  // free block for the update
    // ---- Gram: S (upper), C, diag Q; `parts` threads per entry, fixed order
    for (int e0 = 0; e0 < nE; e0 += slots) {
      const int e = e0 + tid / parts, q = tid % parts;
      float acc = 0.f;
      if (tid < slots * parts && e < nE) {
        const float *P, *R;
        int ca, cb;
        entry_cols(e, k, nS, nC, ca, cb);
        if (e < nS) {
          P = X;
          R = X;
        } else if (e < nS + nC) {
          P = X;
          R = MV;
        } else {
          P = MV;
          R = MV;
        }
        for (int r = q; r < n; r += parts) acc = fmaf(P[r * k + ca], R[r * k + cb], acc);
      }
      part[tid] = acc;
      __syncthreads();
      if (tid < slots && e0 + tid < nE) {
        const int e2 = e0 + tid;
        double s = 0.0;
        for (int qq = 0; qq < parts; ++qq) s += (double)part[tid * parts + qq];
        int ca, cb;
        entry_cols(e2, k, nS, nC, ca, cb);
        if (e2 < nS) {
          G[ca * k + cb] = s;
          G[cb * k + ca] = s;
        } else if (e2 < nS + nC) {
          G[k * k + ca * k + cb] = s;
        } else {
          G[2 * k * k + ca * k + ca] = s;
        }
      }
      __syncthreads();
    }
    // ---- k x k algebra (fp64), one thread per column ----------------------
    if (tid < k) {
      const int i = tid;
      const double* S = G;
      const double* C = G + k * k;
      const double eta = a.eta;
      double d = C[i * k + i];
      for (int j = 0; j < i; ++j) d -= S[i * k + j] * C[j * k + i];
      double acol[SMALL_MAX_K];
      for (int r = 0; r < k; ++r) acol[r] = (r < i) ? -eta * C[r * k + i] : (r == i ? 1.0 - eta * d : 0.0);
      double nrm2 = eta * eta * G[2 * k * k + i * k + i];
      for (int b = 0; b <= i; ++b) {
        double sa = 0.0;
        for (int r = 0; r <= i; ++r) sa += S[b * k + r] * acol[r];
        nrm2 += acol[b] * sa + 2.0 * eta * acol[b] * C[b * k + i];
      }
      for (int r = 0; r < k; ++r) Acoef[r * k + i] = (float)acol[r];
      const double nrm = nrm2 > 0.0 ? sqrt(nrm2) : 0.0;
      if (!(nrm >= 1e-12)) {
        atomicExch(a.flag, 1);
        scale[i] = 0.f;
      } else {
        scale[i] = (float)(1.0 / nrm);
      }
    }
    __syncthreads();
    // ---- update: X' = (X A + eta MV) diag(scale), into Wa, then swap ----
    for (int i = tid; i < nk; i += SMALL_THREADS) {
      const int r = i / k, c = i - r * k;
      float acc = 0.f;
      for (int q = 0; q <= c; ++q) acc = fmaf(X[r * k + q], Acoef[q * k + c], acc);
      Wa[i] = fmaf((float)a.eta, MV[i], acc) * scale[c];
    }
    __syncthreads();
    for (int i = tid; i < nk; i += SMALL_THREADS) X[i] = Wa[i];
    __syncthreads();
  }
  for (int i = tid; i < nk; i += SMALL_THREADS) a.V[i] = X[i];
}

}  // namespace
}  // namespace sped

using namespace sped;

extern "C" int sped_small_mueg(int32_t n, int32_t k, const int32_t* indptr, const int32_t* indices,
                               const float* values, int32_t n_terms, const double* alpha,
                               const double* beta, const double* gamma, double w0_scale,
                               double lam_f, double s_final, double eta, int32_t steps, float* V,
                               int32_t* flag, sped_stream_t stream) {
  SPED_CHECK_ARG(n >= 1 && k >= 1 && V && flag && indptr, "bad small_mueg arguments");
  int32_t nnz_h = 0;
  SPED_CUDA(cudaMemcpyAsync(&nnz_h, indptr + n, sizeof(int32_t), cudaMemcpyDeviceToHost,
                            as_stream(stream)));
  SPED_CUDA(cudaStreamSynchronize(as_stream(stream)));
  const size_t need = sizeof(float) * 3 * (size_t)n * k + sizeof(int32_t) * (n + 1) +
                      (size_t)nnz_h * (values ? 8 : 4) + 64;
  if ((int64_t)n * k > SMALL_MAX_NK || k > SMALL_MAX_K || n_terms > SMALL_MAX_TERMS ||
      need > (size_t)SMALL_SMEM_BYTES) {
    set_error("graph too large for the single-block solver (n*k=%lld)", (long long)n * k);
    return SPED_ERR_UNSUPPORTED;
  }
  SmallArgs a;
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
  a.flag = flag;
  const size_t smem = need;
  static bool attr = false;
  if (!attr) {
    SPED_CUDA(cudaFuncSetAttribute(small_mueg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   SMALL_SMEM_BYTES));
    attr = true;
  }
  small_mueg_kernel<<<1, SMALL_THREADS, smem, as_stream(stream)>>>(a);
  SPED_LAUNCH_CHECK();
  return SPED_OK;
}
