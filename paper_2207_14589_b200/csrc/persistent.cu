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
//                   -- no barrier between terms: generation-tagged words (below)
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
// Terms exchange rows WITHOUT grid barriers: an intermediate term's output
// element is one 64-bit word (fp32 value | 32-bit generation tag) stored
// with st.relaxed.gpu, and a gather spins (ld.relaxed.gpu) until the word
// carries the generation it expects -- the LL ("low latency") protocol of
// NCCL applied to the SpMM halo.  A row's next-generation value is written
// only after all of its neighbours' current values were read by it, and L is
// symmetric with an explicit diagonal, so every reader of a word finishes
// before the word's owner can reach the generation after next: two tagged
// buffers suffice.  Tags are a launch base (device counter in the workspace,
// advanced by each launch) + step*T + t + 1, so stale words of earlier
// launches never match.  A gather that waits past ~1 s sets bit 2 of `flag`
// and proceeds instead of hanging.
//
// 2 (or 3) grid barriers per step: Gram partials, [partials reduce,] update;
// the T - 1 barriers between terms of the barrier version are gone
// (config 1: 62 -> 50 us/step, config 2: 91 -> 72 us/step).  Up to 256 terms
// (negexp-limit(251), the reference's high-degree transform).
//
// Same arithmetic as the multi-kernel path (spmm.cu term schedule; mu-EG in
// Gram form, solvers.py:121-144 / SURVEY §8a; zero-norm columns flagged for
// the host's re-randomisation, solvers.py:136-143).  Every read of a block
// written inside the launch goes through ld.global.cg: a 32-B L1 sector can
// straddle two CTAs' row ranges, so no block data is ever cached in L1.

#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>

#include "sped_common.cuh"

namespace cg = cooperative_groups;

#ifdef PT_PROFILE  // probe build: CTA 0 records per-phase times of step 1
#define PT_MARK(name)                                                          \
  do {                                                                         \
    if (step == 1 && b == 0 && tid == 0 && pt_n < 64) {                        \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(pt_t[pt_n]));           \
      pt_name[pt_n++] = name;                                                  \
    }                                                                          \
  } while (0)
#else
#define PT_MARK(name) \
  do {                \
  } while (0)
#endif

namespace sped {
namespace {

constexpr int PT_MAX_K = 32;
constexpr int PT_MAX_TERMS = 256;  // term coefficients ride in the kernel parameters (3 KB)
constexpr int PT_DYN_BYTES = 180 * 1024;  // dynamic smem: own rows + CSR slice
constexpr int PT_NT = 512;                // threads per CTA
#ifndef PT_REDUNDANT_MAX
#define PT_REDUNDANT_MAX 8192  // partial-table entries every CTA reduces itself
#endif
// Gram entries (S upper, C, diag Q) at k = 32 and the passes over them
constexpr int PT_MAX_NE = PT_MAX_K * (PT_MAX_K + 1) / 2 + PT_MAX_K * PT_MAX_K + PT_MAX_K;
constexpr int PT_MAX_PASSES = (PT_MAX_NE + PT_NT - 1) / PT_NT;

struct PArgs {
  int32_t n, k, nterms;
  uint32_t* epoch;     // device tag base, advanced by steps*nterms per launch
  const int32_t* indptr;
  const int32_t* indices;
  const float* values;  // NULL = implicit unit-weight combinatorial
  float alpha[PT_MAX_TERMS], beta[PT_MAX_TERMS], gamma[PT_MAX_TERMS];
  float w0, lamf, sfin;
  double eta;
  int32_t steps;
  int32_t slots;  // nonzero slots per row (lanes per row = slots * k)
  float* V;  // in/out
  float* XB;   // X ping-pong partner of V (float, n x k)
  float* Mb;   // M when the CTA's rows are not smem-resident (float, n x k)
  unsigned long long* L0;  // tagged term outputs (fp32 | tag << 32), n x k
  unsigned long long* L1;
  double* partials;  // [grid][nE]
  double* G;         // [nE]
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

// Scatter reduced Gram entry e into the dense S (symmetric), C and diag Q.
__device__ __forceinline__ void put_gram(double* Gs, int e, int k, int nS, int nC, double g) {
  int ca, cb;
  entry_cols(e, k, nS, nC, ca, cb);
  if (e < nS) {
    Gs[ca * k + cb] = g;
    Gs[cb * k + ca] = g;
  } else if (e < nS + nC) {
    Gs[k * k + ca * k + cb] = g;
  } else {
    Gs[2 * k * k + ca] = g;
  }
}

__device__ __forceinline__ unsigned long long ld_ll(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_ll(unsigned long long* p, float x, uint32_t tag) {
  const unsigned long long v = ((unsigned long long)tag << 32) | __float_as_uint(x);
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
constexpr uint32_t LL_SPIN_LIMIT = 1u << 21;  // per wait, x ~0.5 us per L2 round trip

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

// Cholesky of the k x k fp64 Gram G (upper R, G = R^T R) and T = R^{-1}
// (upper), CTA-wide; R lives in Rw (k x k fp64 scratch), T goes out as fp32.
// Same arithmetic as oja_coeffs_kernel (solver.cu).  Returns nonzero when a
// pivot is not positive (rank collapse; the host re-randomises).
template <int PT_THREADS>
__device__ int cta_chol_inverse(int k, const double* G, double* Rw, float* T) {
  __shared__ int bad;
  const int tid = threadIdx.x;
  for (int e = tid; e < k * k; e += PT_THREADS) Rw[e] = G[e];
  if (tid == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < k; ++j) {
    if (tid == 0) {
      double djj = Rw[j * k + j];
      for (int q = 0; q < j; ++q) djj -= Rw[q * k + j] * Rw[q * k + j];
      if (!(djj > 1e-24)) {
        bad = 1;
        djj = 1.0;
      }
      Rw[j * k + j] = sqrt(djj);
    }
    __syncthreads();
    const double rjj = Rw[j * k + j];
    for (int l = j + 1 + tid; l < k; l += PT_THREADS) {
      double v = Rw[j * k + l];
      for (int q = 0; q < j; ++q) v -= Rw[q * k + j] * Rw[q * k + l];
      Rw[j * k + l] = v / rjj;
    }
    __syncthreads();
  }
  // back substitution per column l; T[i][l] (i < l) parked at Rw[l][i]
  for (int l = tid; l < k; l += PT_THREADS) {
    const double tll = 1.0 / Rw[l * k + l];
    for (int i = l - 1; i >= 0; --i) {
      double acc = -Rw[i * k + l] * tll;
      for (int q = i + 1; q < l; ++q) acc -= Rw[i * k + q] * Rw[l * k + q];
      Rw[l * k + i] = acc / Rw[i * k + i];
    }
  }
  __syncthreads();
  for (int e = tid; e < k * k; e += PT_THREADS) {
    const int i = e / k, l = e % k;
    T[e] = (float)(i == l ? 1.0 / Rw[i * k + i] : (i < l ? Rw[l * k + i] : 0.0));
  }
  __syncthreads();
  return bad;
}

// OJA = false: mu-EigenGame steps (solvers.py:121-144, Gram form);
// OJA = true: oja_step (solvers.py:114-118) with the MGS as CholQR2 -- W =
// X + eta M, then twice: Gram of the own rows -> all-CTA sum -> Cholesky ->
// rows times R^{-1}.
template <int PT_THREADS, bool OJA>
__global__ void __launch_bounds__(PT_THREADS, 1) persistent_mueg_kernel(const PArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ double Gs[2 * PT_MAX_K * PT_MAX_K + PT_MAX_K];  // S, C, diag Q
  __shared__ double Ad[PT_MAX_K * PT_MAX_K];                 // A (fp64)
  __shared__ double Tn[PT_MAX_K * PT_MAX_K];                 // column-norm terms
  __shared__ double red[PT_THREADS];
  __shared__ float Acoef[PT_MAX_K * PT_MAX_K];
  __shared__ float scale[PT_MAX_K];

  const int n = a.n, k = a.k, tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int nb = gridDim.x, b = blockIdx.x;
  const int64_t nnz = __ldg(a.indptr + n);
  // nnz-balanced contiguous row range, identical for every phase
  const int r0 = (b == 0) ? 0 : row_lower_bound(a.indptr, n, nnz * b / nb);
  const int r1 = (b == nb - 1) ? n : row_lower_bound(a.indptr, n, nnz * (b + 1) / nb);
  const int nr = r1 - r0;
  const int64_t i0 = (int64_t)r0 * k, i1 = (int64_t)r1 * k;
  const int nS = k * (k + 1) / 2, nC = k * k, nE = nS + nC + k;
  const bool has_vals = (a.values != nullptr);
  const float eta_f = (float)a.eta;

  // ---- shared-memory residency of this CTA's slice --------------------------
  // Layout of the dynamic buffer: [CSR slice of own rows][state].  The state
  // is either resident (own rows of X in two generations + M, kept across
  // phases) or a staging area the Gram streams own rows through.
  const size_t blk = (size_t)nr * k * sizeof(float);
  const bool resident = 3 * blk <= (size_t)PT_DYN_BYTES;
  const int e0 = __ldg(a.indptr + r0), e1 = __ldg(a.indptr + r1);
  const size_t csr_bytes =
      (sizeof(int32_t) * ((size_t)nr + 1 + (size_t)(e1 - e0) * (has_vals ? 2 : 1)) + 15) & ~size_t(15);
  const size_t min_state = resident ? 3 * blk : 2 * sizeof(float) * k * 64;
  const bool csr_smem = csr_bytes + min_state <= (size_t)PT_DYN_BYTES;
  const size_t state_off = csr_smem ? csr_bytes : 0;
  int32_t* cptr = reinterpret_cast<int32_t*>(dyn);
  int32_t* cidx = cptr + nr + 1;
  float* cval = reinterpret_cast<float*>(cidx + (e1 - e0));
  float* sXa = reinterpret_cast<float*>(dyn + state_off);
  float* sXb = sXa + (size_t)nr * k;  // resident mode only
  float* sM = sXb + (size_t)nr * k;   // resident mode only
  if (csr_smem) {
    for (int i = tid; i <= nr; i += PT_THREADS) cptr[i] = __ldg(a.indptr + r0 + i) - e0;
    for (int i = tid; i < e1 - e0; i += PT_THREADS) {
      cidx[i] = __ldg(a.indices + e0 + i);
      if (has_vals) cval[i] = __ldg(a.values + e0 + i);
    }
  }
  if (resident)
    for (int i = tid; i < nr * k; i += PT_THREADS) sXa[i] = a.V[i0 + i];
  // non-resident CTAs stage own rows in chunks through the state area
  const int stage_rows =
      max(1, (int)(((size_t)PT_DYN_BYTES - state_off) / (2 * sizeof(float) * k)));
  const int* rp = csr_smem ? cptr : a.indptr + r0;  // row pointers of own rows
  const int rbase = csr_smem ? 0 : e0;               // rp[] - rbase indexes ix/vx
  const int32_t* ix = csr_smem ? cidx : a.indices + e0;
  const float* vx = csr_smem ? cval : (has_vals ? a.values + e0 : nullptr);
  __syncthreads();

  // Gram work split: `parts` threads per entry, `per_pass` entries per pass
  const int parts = max(1, PT_THREADS / nE), per_pass = PT_THREADS / parts;
  const int passes = (nE + per_pass - 1) / per_pass;  // <= PT_MAX_PASSES for k <= 32
  // small partial tables are reduced redundantly by every CTA (one grid
  // barrier less per step); large ones by one warp per entry
  const bool redundant_reduce = (int64_t)nb * nE <= PT_REDUNDANT_MAX;
  // term lanes: a row is S nonzero slots x k columns; a warp takes RW rows
  const int S = a.slots, LR = S * k, RW = 32 / LR;
  const int lg = lane / LR, lrem = lane - lg * LR, lc = lrem % k, ls = lrem / k;
  const bool active = lg < RW;
  const int rows_per_pass = (PT_THREADS / 32) * RW;

  float* X = a.V;
  float* sX = sXa;   // own rows of X (resident mode)
  float* sXn = sXb;  // next generation
  const uint32_t tag0 = *reinterpret_cast<volatile uint32_t*>(a.epoch);

#ifdef PT_PROFILE
  uint64_t pt_t[64];
  const char* pt_name[64];
  int pt_n = 0;
  if (tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(pt_t[pt_n]));
  pt_name[pt_n++] = "start";
#endif
  for (int step = 0; step < a.steps; ++step) {
    // ---- M = p(L) X: RW rows per warp, S slots x k columns per row ---------
    // term 0 gathers X (float, written before the last grid barrier); term
    // t >= 1 gathers the tagged output of term t-1; the final term writes M
    // (own rows only: smem when resident, else the float buffer Mb)
    float* M = a.Mb;
    for (int t = 0; t < a.nterms; ++t) {
      const bool final = (t == a.nterms - 1);
      const unsigned long long* lin = (t & 1) ? a.L0 : a.L1;   // output of term t-1
      unsigned long long* lout = (t & 1) ? a.L1 : a.L0;
      const uint32_t want = tag0 + (uint32_t)(step * a.nterms + t);      // tag of term t-1
      const uint32_t mine = want + 1u;
      const float sc = (t == 0) ? a.w0 : 1.f;
      const float al = a.alpha[t], be = a.beta[t] * sc, ga = a.gamma[t] * sc;
      for (int lr0 = warp * RW; lr0 < nr; lr0 += rows_per_pass) {
        const int lr = min(lr0 + lg, nr - 1);  // idle groups re-read the last row
        const bool own = active && (lr0 + lg < nr);
        const int r = r0 + lr;
        const int rb = rp[lr] - rbase, re = rp[lr + 1] - rbase;
        const float dg = (float)(re - rb - 1);
        const int64_t i = (int64_t)r * k + lc;
        const bool lead = (ls == 0 && own);
        // own-row operands issued before the gathers (independent loads);
        // the own row of a tagged block was written by this very thread
        float wself = 0.f;
        if (lead && ga != 0.f)
          wself = (t == 0) ? (resident ? sX[lr * k + lc] : __ldcg(X + i))
                           : __uint_as_float((uint32_t)ld_ll(lin + i));
        const float xv = (lead && (al != 0.f || final))
                             ? (resident ? sX[lr * k + lc] : __ldcg(X + i)) : 0.f;
        float acc = 0.f;
        if (active) {
          // all of a lane's gathers (up to 8) in flight at once, predicated
          for (int base = rb + ls; base < re; base += 8 * S) {
            int c[8];
            float v[8], x[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const int p = base + j * S;
              c[j] = (p < re) ? ix[p] : -1;
            }
            if (t == 0) {
#pragma unroll
              for (int j = 0; j < 8; ++j)
                x[j] = (c[j] < 0) ? 0.f : __ldcg(X + (int64_t)c[j] * k + lc);
            } else {
              unsigned long long q[8];
#pragma unroll
              for (int j = 0; j < 8; ++j)
                q[j] = (c[j] < 0) ? 0ull : ld_ll(lin + (int64_t)c[j] * k + lc);
              // re-poll every stale word of the batch in the same round (one
              // L2 round trip per round, not one per stale word)
              for (uint32_t spins = 0;; ++spins) {
                bool ready = true;
#pragma unroll
                for (int j = 0; j < 8; ++j)
                  ready &= (c[j] < 0) || ((uint32_t)(q[j] >> 32) == want);
                if (ready) break;
                // a word already carrying a LATER generation of this buffer
                // means its owner overwrote it before this reader consumed
                // it: the two-buffer invariant broke (flag bit 4, raised)
                bool ahead = false;
#pragma unroll
                for (int j = 0; j < 8; ++j)
                  ahead |= (c[j] >= 0) && ((int32_t)((uint32_t)(q[j] >> 32) - want) > 0);
                if (ahead) {
                  atomicOr(a.flag, 4);
                  break;
                }
                if (spins > LL_SPIN_LIMIT) {
                  atomicOr(a.flag, 2);
                  break;
                }
#pragma unroll
                for (int j = 0; j < 8; ++j)
                  if (c[j] >= 0 && (uint32_t)(q[j] >> 32) != want)
                    q[j] = ld_ll(lin + (int64_t)c[j] * k + lc);
              }
#pragma unroll
              for (int j = 0; j < 8; ++j) x[j] = (c[j] < 0) ? 0.f : __uint_as_float((uint32_t)q[j]);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const int p = base + j * S;
              v[j] = (c[j] < 0) ? 0.f : (has_vals ? vx[p] : (c[j] == r ? dg : -1.f));
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) acc = fmaf(v[j], x[j], acc);
          }
        }
        float tot = acc;  // slots folded in fixed order
        for (int s2 = 1; s2 < S; ++s2) {
          const float o = __shfl_sync(0xffffffffu, acc, lg * LR + s2 * k + lc);
          if (ls == 0) tot += o;
        }
        if (lead) {
          float o = be * tot;
          if (al != 0.f) o = fmaf(al, xv, o);
          if (ga != 0.f) o = fmaf(ga, wself, o);
          if (final) {
            o = fmaf(a.lamf, xv, a.sfin * o);
            if (resident)
              sM[lr * k + lc] = o;  // M is only read back by this CTA
            else
              M[i] = o;
          } else {
            st_ll(lout + i, o, mine);
          }
        }
      }
      PT_MARK("term");
    }
    if (a.nterms == 0) {
      for (int64_t i = i0 + tid; i < i1; i += PT_THREADS) {
        const float o = (a.lamf + a.sfin * a.w0) * (resident ? sX[i - i0] : __ldcg(X + i));
        if (resident)
          sM[i - i0] = o;
        else
          M[i] = o;
      }
    }
    float* Xn = (X == a.V) ? a.XB : a.V;  // X' goes to the other float buffer
    __syncthreads();                      // own rows of M complete

    if constexpr (OJA) {
      // W = X + eta M over the own rows, in place of M (smem or Mb)
      float* Wb = resident ? sM : M;
      float* W1b = resident ? sXn : Xn;
      const int64_t wo = resident ? 0 : i0;  // element offset of own row 0
      for (int i = tid; i < nr * k; i += PT_THREADS) {
        const float xv = resident ? sX[i] : __ldcg(X + i0 + i);
        const float mv = resident ? sM[i] : __ldcg(M + i0 + i);
        Wb[wo + i] = fmaf(eta_f, mv, xv);
      }
      __syncthreads();
      const int nSo = k * (k + 1) / 2;
      const int parts_o = max(1, PT_THREADS / nSo), per_pass_o = PT_THREADS / parts_o;
      const int passes_o = (nSo + per_pass_o - 1) / per_pass_o;
      const bool redundant_o = (int64_t)nb * nSo <= PT_REDUNDANT_MAX;
      for (int cq = 0; cq < 2; ++cq) {
        const float* Bsrc = cq == 0 ? Wb : W1b;   // block whose Gram is taken
        float* Bdst = cq == 0 ? W1b : Wb;         // block times R^{-1}
        // Gram partial of the own rows (upper triangle, fixed order)
        double acc[PT_MAX_PASSES];
#pragma unroll
        for (int q = 0; q < PT_MAX_PASSES; ++q) acc[q] = 0.0;
        for (int pass = 0; pass < passes_o; ++pass) {
          const int e = pass * per_pass_o + tid / parts_o, q = tid % parts_o;
          double sum = 0.0;
          if (tid < per_pass_o * parts_o && e < nSo) {
            int ca, cb;
            entry_cols(e, k, nSo, 0, ca, cb);
            for (int r = q; r < nr; r += parts_o) {
              const float pa = resident ? Bsrc[r * k + ca] : __ldcg(Bsrc + wo + r * k + ca);
              const float pb = resident ? Bsrc[r * k + cb] : __ldcg(Bsrc + wo + r * k + cb);
              sum += (double)pa * (double)pb;
            }
          }
          red[tid] = sum;
          __syncthreads();
          if (tid < per_pass_o) {
            double t2 = 0.0;
            for (int qq = 0; qq < parts_o; ++qq) t2 += red[tid * parts_o + qq];
            acc[pass] += t2;
          }
          __syncthreads();
        }
        for (int pass = 0; pass < passes_o; ++pass) {
          const int e = pass * per_pass_o + tid;
          if (tid < per_pass_o && e < nSo) a.partials[(size_t)b * nSo + e] = acc[pass];
        }
        grid.sync();
        // sum the partials in CTA order into Gs (symmetric S)
        if (redundant_o) {
          for (int e = tid; e < nSo; e += PT_THREADS) {
            double sum = 0.0;
            for (int q = 0; q < nb; ++q) sum += __ldcg(a.partials + (size_t)q * nSo + e);
            put_gram(Gs, e, k, nSo, 0, sum);
          }
        } else {
          const int gw = b * (PT_THREADS / 32) + warp;
          const int nwarps = nb * (PT_THREADS / 32);
          for (int e = gw; e < nSo; e += nwarps) {
            double sum = 0.0;
            for (int q = lane; q < nb; q += 32) sum += __ldcg(a.partials + (size_t)q * nSo + e);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, off);
            if (lane == 0) a.G[e] = sum;
          }
          grid.sync();
          for (int e = tid; e < nSo; e += PT_THREADS) put_gram(Gs, e, k, nSo, 0, __ldcg(a.G + e));
        }
        __syncthreads();
        if (cta_chol_inverse<PT_THREADS>(k, Gs, Ad, Acoef) && b == 0 && tid == 0)
          atomicExch(a.flag, 1);
        // rows times R^{-1} (upper): Bdst[r][c] = sum_{q <= c} Bsrc[r][q] T[q][c]
        for (int i = tid; i < nr * k; i += PT_THREADS) {
          const int r = i / k, c = i - r * k;
          float o = 0.f;
          for (int q = 0; q <= c; ++q) {
            const float bv = resident ? Bsrc[r * k + q] : __ldcg(Bsrc + wo + r * k + q);
            o = fmaf(bv, Acoef[q * k + c], o);
          }
          Bdst[wo + i] = o;
        }
        __syncthreads();
        if (cq == 0) grid.sync();  // the partials buffer is reused by pass 2
      }
      // X' = Wb (own rows) -> Xn (global) and the resident copy
      for (int i = tid; i < nr * k; i += PT_THREADS) {
        const float o = resident ? Wb[i] : __ldcg(Wb + wo + i);
        Xn[i0 + i] = o;
        if (resident) sXn[i] = o;
      }
    } else {
    // ---- Gram partials over own rows (fp64 accumulation, fixed order) ------
    {
      double acc[PT_MAX_PASSES];
#pragma unroll
      for (int q = 0; q < PT_MAX_PASSES; ++q) acc[q] = 0.0;
      const int chunk = resident ? max(nr, 1) : stage_rows;
      float* qX = resident ? sX : sXa;
      float* qM = resident ? sM : sXa + (size_t)stage_rows * k;
      for (int rr = 0; rr < nr; rr += chunk) {
        const int nrr = min(chunk, nr - rr);
        if (!resident) {
          for (int i = tid; i < nrr * k; i += PT_THREADS) {
            qX[i] = __ldcg(X + i0 + (int64_t)rr * k + i);
            qM[i] = __ldcg(M + i0 + (int64_t)rr * k + i);
          }
          __syncthreads();
        }
        for (int pass = 0; pass < passes; ++pass) {
          const int e = pass * per_pass + tid / parts, q = tid % parts;
          double s = 0.0;
          if (tid < per_pass * parts && e < nE) {
            int ca, cb;
            entry_cols(e, k, nS, nC, ca, cb);
            const float* P = (e < nS + nC) ? qX : qM;
            const float* R = (e < nS) ? qX : qM;
            for (int r = q; r < nrr; r += parts) s += (double)P[r * k + ca] * (double)R[r * k + cb];
          }
          red[tid] = s;
          __syncthreads();
          if (tid < per_pass) {
            double t2 = 0.0;
            for (int qq = 0; qq < parts; ++qq) t2 += red[tid * parts + qq];
            acc[pass] += t2;
          }
          __syncthreads();
        }
      }
      for (int pass = 0; pass < passes; ++pass) {
        const int e = pass * per_pass + tid;
        if (tid < per_pass && e < nE) a.partials[(size_t)b * nE + e] = acc[pass];
      }
    }
    PT_MARK("gram");
    grid.sync();
    PT_MARK("gram-sync");

    // ---- reduce the per-CTA partials (fixed order) --------------------------
    if (redundant_reduce) {  // 8 lanes per entry, all of a lane's loads in flight
      const int sub = lane & 7;
      for (int e0 = warp * 4; e0 < nE; e0 += (PT_THREADS / 32) * 4) {
        const int e = e0 + (lane >> 3);
        double s = 0.0;
        if (e < nE) {
#pragma unroll 4
          for (int q = sub; q < nb; q += 8) s += __ldcg(a.partials + (size_t)q * nE + e);
        }
        s += __shfl_down_sync(0xffffffffu, s, 4, 8);
        s += __shfl_down_sync(0xffffffffu, s, 2, 8);
        s += __shfl_down_sync(0xffffffffu, s, 1, 8);
        if (sub == 0 && e < nE) put_gram(Gs, e, k, nS, nC, s);
      }
    } else {
      const int gw = b * (PT_THREADS / 32) + warp;
      const int nwarps = nb * (PT_THREADS / 32);
      for (int e = gw; e < nE; e += nwarps) {
        double s = 0.0;
        for (int q = lane; q < nb; q += 32) s += __ldcg(a.partials + (size_t)q * nE + e);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
        if (lane == 0) a.G[e] = s;
      }
      grid.sync();
      for (int e = tid; e < nE; e += PT_THREADS) put_gram(Gs, e, k, nS, nC, __ldcg(a.G + e));
    }
    __syncthreads();
    PT_MARK("reduce");

    // ---- coefficients (every CTA, fp64; solvers.py:121-144 in Gram form) ---
    const double* Sg = Gs;
    const double* Cg = Gs + k * k;
    const double eta = a.eta;
    if (tid < k) {  // column i of A: -eta C[r,i] above, 1 - eta d_i on the diagonal
      const int i = tid;
      double d = Cg[i * k + i];
      for (int j = 0; j < i; ++j) d -= Sg[i * k + j] * Cg[j * k + i];
      for (int r = 0; r < k; ++r)
        Ad[r * k + i] = (r < i) ? -eta * Cg[r * k + i] : (r == i ? 1.0 - eta * d : 0.0);
    }
    __syncthreads();
    // norm terms T[bb,i] = A[bb,i] (sum_{r<=i} S[bb,r] A[r,i] + 2 eta C[bb,i]), bb <= i
    for (int q = tid; q < PT_MAX_K * PT_MAX_K; q += PT_THREADS) {
      const int tb = q / PT_MAX_K, ti = q % PT_MAX_K;
      double tval = 0.0;
      if (tb < k && ti < k && tb <= ti) {
        double sa = 0.0;
        for (int r = 0; r <= ti; ++r) sa += Sg[tb * k + r] * Ad[r * k + ti];
        tval = Ad[tb * k + ti] * (sa + 2.0 * eta * Cg[tb * k + ti]);
      }
      Tn[q] = tval;
    }
    __syncthreads();
    if (tid < k) {
      const int i = tid;
      double nrm2 = eta * eta * Gs[2 * k * k + i];
      for (int bb = 0; bb <= i; ++bb) nrm2 += Tn[bb * PT_MAX_K + i];
      for (int r = 0; r < k; ++r) Acoef[r * k + i] = (float)Ad[r * k + i];
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
      float acc = 0.f, m;
      if (resident) {
        const float* xr = sX + (r - r0) * k;
        for (int q = 0; q <= c; ++q) acc = fmaf(xr[q], Acoef[q * k + c], acc);
        m = sM[i - i0];
      } else {
        const float* xr = X + (int64_t)r * k;
        for (int q = 0; q <= c; ++q) acc = fmaf(__ldcg(xr + q), Acoef[q * k + c], acc);
        m = __ldcg(M + i);
      }
      const float o = fmaf(eta_f, m, acc) * scale[c];
      Xn[i] = o;
      if (resident) sXn[i - i0] = o;
    }
    }
    X = Xn;
    {
      float* tmp = sX;
      sX = sXn;
      sXn = tmp;
    }
    PT_MARK("coef+upd");
    grid.sync();
    PT_MARK("upd-sync");
  }
  if (X != a.V)
    for (int64_t i = i0 + tid; i < i1; i += PT_THREADS)
      a.V[i] = resident ? sX[i - i0] : __ldcg(X + i);
  // every CTA read the tag base before its first grid barrier
  if (b == 0 && tid == 0) *a.epoch = tag0 + (uint32_t)(a.steps * a.nterms);
#ifdef PT_PROFILE
  if (b == 0 && tid == 0)
    for (int q = 2; q < pt_n; ++q)
      printf("pt %-10s %7.3f us\n", pt_name[q], (pt_t[q] - pt_t[q - 1]) * 1e-3);
#endif
}

}  // namespace
}  // namespace sped

using namespace sped;

// Workspace: [XB f32 n*k][Mb f32 n*k][L0 u64 n*k][L1 u64 n*k][partials, G
// f64 (sms+1)*nE][epoch u32].  Zero it once before the first launch (tags
// start at 1); keep it across launches (the tag base lives in it).
static void persistent_layout(int32_t n, int32_t k, size_t* l0_off, size_t* part_off,
                              size_t* epoch_off, size_t* total) {
  const size_t nk = (size_t)n * k;
  const size_t nE = (size_t)k * (k + 1) / 2 + (size_t)k * k + k;
  size_t off = 2 * nk * sizeof(float);
  off = (off + 255) & ~size_t(255);
  *l0_off = off;
  off += 2 * nk * sizeof(unsigned long long);
  off = (off + 255) & ~size_t(255);
  *part_off = off;
  off += ((size_t)num_sms() + 1) * nE * sizeof(double);
  off = (off + 255) & ~size_t(255);
  *epoch_off = off;
  *total = off + 256;
}

extern "C" int sped_persistent_workspace_bytes(int32_t n, int32_t k, int64_t* bytes) {
  SPED_CHECK_ARG(n >= 1 && k >= 1 && bytes, "bad persistent workspace arguments");
  size_t l0, part, ep, total;
  persistent_layout(n, k, &l0, &part, &ep, &total);
  *bytes = (int64_t)total;
  return SPED_OK;
}

static int persistent_run(int32_t n, int32_t k, int64_t nnz, const int32_t* indptr,
                          const int32_t* indices, const float* values, int32_t n_terms,
                          const double* alpha, const double* beta, const double* gamma,
                          double w0_scale, double lam_f, double s_final, double eta,
                          int32_t steps, float* V, int32_t* flag, void* workspace,
                          int64_t workspace_bytes, sped_stream_t stream, bool oja) {
  SPED_CHECK_ARG(n >= 1 && k >= 1 && nnz >= 0 && V && flag && indptr && indices && workspace &&
                     steps >= 0,
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
  // 512-thread CTAs (116 registers, no spills; the 1024-thread variant is
  // capped at 64 registers and spilled the tagged gathers: config 2 96 vs
  // 76 us/step)
  const double avg = (double)nnz / n;
  int slots = (int)std::ceil(avg / 8.0);  // ~8 gathers in flight per lane
  slots = std::max(1, std::min(slots, 32 / k));
  const int rw = 32 / (slots * k);
  const int sms = num_sms();
  constexpr int nt = PT_NT;
  const void* fn = oja ? (const void*)persistent_mueg_kernel<PT_NT, true>
                       : (const void*)persistent_mueg_kernel<PT_NT, false>;
  static PerDeviceOnce attr;  // per device: function attributes are per context
  {
    const int rc_ = attr([&]() -> int {
      SPED_CUDA(cudaFuncSetAttribute(persistent_mueg_kernel<PT_NT, false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, PT_DYN_BYTES));
      SPED_CUDA(cudaFuncSetAttribute(persistent_mueg_kernel<PT_NT, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, PT_DYN_BYTES));
      return SPED_OK;
    });
    if (rc_ != SPED_OK) return rc_;
  }
  int per_sm = 0;
  SPED_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, nt, PT_DYN_BYTES));
  if (per_sm < 1) {
    set_error("persistent solver kernel cannot be resident");
    return SPED_ERR_CUDA;
  }
  // one CTA per SM, but no more CTAs than it takes to give each warp a row group
  const int64_t rows_per_cta = (int64_t)(nt / 32) * rw;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(sms, (n + rows_per_cta - 1) / rows_per_cta));
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
  a.slots = slots;
  a.V = V;
  char* ws = static_cast<char*>(workspace);
  size_t l0_off, part_off, epoch_off, total;
  persistent_layout(n, k, &l0_off, &part_off, &epoch_off, &total);
  a.XB = reinterpret_cast<float*>(ws);
  a.Mb = a.XB + (size_t)n * k;
  a.L0 = reinterpret_cast<unsigned long long*>(ws + l0_off);
  a.L1 = a.L0 + (size_t)n * k;
  a.partials = reinterpret_cast<double*>(ws + part_off);
  a.G = a.partials + (size_t)grid * nE;
  a.epoch = reinterpret_cast<uint32_t*>(ws + epoch_off);
  a.flag = flag;
  void* args[] = {&a};
  SPED_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(nt), args, PT_DYN_BYTES,
                                        as_stream(stream)));
  return SPED_OK;
}

extern "C" int sped_persistent_mueg(int32_t n, int32_t k, int64_t nnz, const int32_t* indptr,
                                    const int32_t* indices, const float* values, int32_t n_terms,
                                    const double* alpha, const double* beta, const double* gamma,
                                    double w0_scale, double lam_f, double s_final, double eta,
                                    int32_t steps, float* V, int32_t* flag, void* workspace,
                                    int64_t workspace_bytes, sped_stream_t stream) {
  return persistent_run(n, k, nnz, indptr, indices, values, n_terms, alpha, beta, gamma, w0_scale,
                        lam_f, s_final, eta, steps, V, flag, workspace, workspace_bytes, stream,
                        false);
}

extern "C" int sped_persistent_oja(int32_t n, int32_t k, int64_t nnz, const int32_t* indptr,
                                   const int32_t* indices, const float* values, int32_t n_terms,
                                   const double* alpha, const double* beta, const double* gamma,
                                   double w0_scale, double lam_f, double s_final, double eta,
                                   int32_t steps, float* V, int32_t* flag, void* workspace,
                                   int64_t workspace_bytes, sped_stream_t stream) {
  return persistent_run(n, k, nnz, indptr, indices, values, n_terms, alpha, beta, gamma, w0_scale,
                        lam_f, s_final, eta, steps, V, flag, workspace, workspace_bytes, stream,
                        true);
}
