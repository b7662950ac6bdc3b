// K3: edge-minibatch sampled-Laplacian apply fused into the polynomial
// recurrence.  Replaces the identity stochastic oracle of
// make_stochastic_oracle (solvers.py:166-178):
//     batch = rng.integers(0, m, B)                          (host / K4)
//     diff  = (x[u_b] - x[v_b]) * w_b
//     est[u_b] += diff ; est[v_b] -= diff                    (np.add.at)
//     return lam* x - (m/B) est
// and, per term, the restated composition of SURVEY 8c(1) (term t uses the
// t-th minibatch of the same PCG64 stream).
//
// Deterministic formulation (no float atomics): the sampled estimate of row r
//     est_r = sum_{b : r endpoint of e_b} w_b (w_r - w_{other end of e_b})
// is formed from SORTED RECORDS.  Per term, one thread per sampled edge writes
// a (row, neighbour, weight) record for each endpoint the call owns (its CSR
// positions `epos` say where the entries live; a row shard marks the others
// -1), a stable radix sort groups the records by row keeping sample order,
// and a warp-per-row sweep folds each row's records in that order, gathers
// the sampled neighbours' rows and applies the recurrence epilogue.  Rows
// without records only run the epilogue.  (The first version histogrammed
// the batch into an nnz-sized array and scanned all nnz positions per term;
// config 3s: 0.41 ms/term.)

#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <initializer_list>

#include "sped_common.cuh"

namespace sped {
namespace {

// one record per owned endpoint of each sampled edge: key = row, value =
// (float weight bits << 32) | neighbour column (the entry's CSR column: the
// node id, or the [own | halo] index of a row shard); unowned -> key n.
// Records of several terms at once (total = terms * Bt): term t's keys are
// offset by t * (n + 1).
__global__ void records_kernel(int64_t B, int64_t Bt, int64_t n, const int32_t* __restrict__ batch,
                               const int32_t* __restrict__ epos, const int32_t* __restrict__ erow,
                               const int32_t* __restrict__ indices,
                               const float* __restrict__ edge_w, int32_t* __restrict__ keys,
                               uint64_t* __restrict__ vals) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int64_t e = batch[b];
  SPED_DCHECK(e >= 0, DBG_EDGE_OOB);
  const float we = edge_w ? edge_w[e] : 1.0f;
  const int32_t p0 = epos[2 * e], p1 = epos[2 * e + 1];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int32_t p = s ? p1 : p0;
    int32_t row = (int32_t)n;
    uint64_t val = 0;
    if (p >= 0) {
      // the entry's row is the column of its partner entry (whole graph), or
      // the shard's row table
      row = erow ? erow[2 * e + s] : indices[s ? p0 : p1];
      SPED_DCHECK(row >= 0 && row < n, DBG_EDGE_OOB);
      val = ((uint64_t)__float_as_uint(we) << 32) | (uint32_t)indices[p];
    }
    keys[2 * b + s] = row + (int32_t)((b / Bt) * (n + 1));
    vals[2 * b + s] = val;
  }
}

// start[i] = first sorted record with row >= i (i in [0, n])
__global__ void row_starts_kernel(int64_t R, int64_t n, const int32_t* __restrict__ key,
                                  int32_t* __restrict__ start) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t > R) return;
  const int64_t lo = (t == 0) ? -1 : (int64_t)key[t - 1];
  const int64_t hi = (t == R) ? n : min((int64_t)key[t], n);
  for (int64_t i = lo + 1; i <= hi; ++i) start[i] = (int32_t)t;
}

struct BatchArgs {
  int64_t n;
  int32_t k;   // slab width
  int64_t ld;
  const int32_t* start;  // n+1 record runs
  const uint64_t* rec;   // sorted records
  const float* x;
  const float* win;
  float* wout;
  float alpha, beta, gamma, lamf, sfin;  // beta already includes m/B
  int flags;   // bit0 alpha, bit1 gamma, bit2 final, bit3 lamf
  int spare_per_sm;  // resident blocks per SM left free (the concurrent sort)
};

template <int LPR, int CPL, bool VEC>
struct Slab {
  static constexpr int W = VEC ? 4 : 1;  // floats per access
  float v[CPL][W];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int q = 0; q < CPL; ++q)
#pragma unroll
      for (int i = 0; i < W; ++i) v[q][i] = 0.f;
  }
  __device__ __forceinline__ static int col0(int q, int cl) { return (q * LPR + cl) * W; }
  __device__ __forceinline__ void load(const float* base, int cl, int k, bool gather) {
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      const int c = col0(q, cl);
      if (VEC) {
        float4 t = gather ? ld_gather_f4(base + c) : ld_stream_f4(base + c);
        v[q][0] = t.x; v[q][1] = t.y; v[q][2] = t.z; v[q][3] = t.w;
      } else {
        v[q][0] = (c < k) ? (gather ? ld_gather_f32(base + c) : ld_stream_f32(base + c)) : 0.f;
      }
    }
  }
  __device__ __forceinline__ void fma(float a, const Slab& o) {
#pragma unroll
    for (int q = 0; q < CPL; ++q)
#pragma unroll
      for (int i = 0; i < W; ++i) v[q][i] = fmaf(a, o.v[q][i], v[q][i]);
  }
  __device__ __forceinline__ void fold_xor(int off) {
#pragma unroll
    for (int q = 0; q < CPL; ++q)
#pragma unroll
      for (int i = 0; i < W; ++i) v[q][i] += __shfl_xor_sync(0xffffffffu, v[q][i], off);
  }
};

// One warp per row (grid-stride, resident grid, the next row's record run
// prefetched).  The row's records are read 32 at a time in sorted (= sample)
// order; SUB lane groups gather the sampled neighbours' rows.
template <int LPR, int CPL, bool VEC>
__global__ void __launch_bounds__(256) batch_row_kernel(const BatchArgs a) {
  constexpr int SUB = 32 / LPR;
  using S = Slab<LPR, CPL, VEC>;
  const int lane = threadIdx.x & 31;
  const int sub = lane / LPR;
  const int cl = lane % LPR;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= a.n) return;
  const bool need_x = (a.flags & 1) || ((a.flags & 4) && (a.flags & 8));
  int32_t hb = __ldg(a.start + row), he = __ldg(a.start + row + 1);
  for (; row < a.n; row += nwarps) {
    const int64_t nrow = row + nwarps;
    int32_t nb = 0, ne = 0;
    if (nrow < a.n) {
      nb = __ldg(a.start + nrow);
      ne = __ldg(a.start + nrow + 1);
    }
    S wr, xr, acc;
    wr.load(a.win + row * a.ld, cl, a.k, true);
    if (need_x) xr.load(a.x + row * a.ld, cl, a.k, false); else xr.zero();
    acc.zero();
    float hsum = 0.f;  // sum of the row's record weights (the h*w_r part)
    for (int32_t p0 = hb; p0 < he; p0 += 32) {
      const int32_t p = p0 + lane;
      float h = 0.f;
      int32_t col = 0;
      if (p < he) {
        const uint64_t r = __ldg(reinterpret_cast<const unsigned long long*>(a.rec) + p);
        col = (int32_t)(uint32_t)r;
        h = __uint_as_float((uint32_t)(r >> 32));
      }
      hsum += h;
      const int cnt = min(32, he - p0);
      for (int j0 = 0; j0 < cnt; j0 += SUB) {
        const int j = j0 + sub;
        const int32_t c = __shfl_sync(0xffffffffu, col, j & 31);
        const float hh = __shfl_sync(0xffffffffu, h, j & 31);
        if (j < cnt) {
          S g;
          g.load(a.win + (int64_t)c * a.ld, cl, a.k, true);
          acc.fma(-hh, g);
        }
      }
    }
    // fold: nonzero-parallel groups, and the row-sum of h across all lanes
#pragma unroll
    for (int off = LPR; off < 32; off <<= 1) acc.fold_xor(off);
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) hsum += __shfl_xor_sync(0xffffffffu, hsum, off);
    if (sub == 0) {
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
#pragma unroll
        for (int i = 0; i < S::W; ++i) {
          const float est = fmaf(hsum, wr.v[q][i], acc.v[q][i]);
          float r = a.beta * est;
          if (a.flags & 1) r = fmaf(a.alpha, xr.v[q][i], r);
          if (a.flags & 2) r = fmaf(a.gamma, wr.v[q][i], r);
          if (a.flags & 4) {
            r *= a.sfin;
            if (a.flags & 8) r = fmaf(a.lamf, xr.v[q][i], r);
          }
          acc.v[q][i] = r;
        }
        const int c = S::col0(q, cl);
        float* dst = a.wout + row * a.ld + c;
        if (VEC) {
          st_stream_f4(dst, make_float4(acc.v[q][0], acc.v[q][1], acc.v[q][2], acc.v[q][3]));
        } else if (c < a.k) {
          dst[0] = acc.v[q][0];
        }
      }
    }
    hb = nb;
    he = ne;
  }
}

// Aligned slabs (k % 4 == 0, 16-B rows): G = k/4 lanes per row, one float4
// column slice per lane, 32/G rows per warp.  Every lane of a group reads the
// row's records itself (the group's lanes load the same 8-B word: one
// broadcast request), so there are no shuffles and no fold: per record one
// broadcast load, one 16-B gather and 4 FMAs per lane; U records are in
// flight per group.  Records are folded in sorted (= sample) order, so the
// result is deterministic.  (The warp-per-row kernel below spent most of its
// issue slots on shuffles and folds: config 3s has ~2 records per row.)
// G <= 16: U = 2 records in flight and 8 resident blocks (32 registers);
// G = 32 (k = 128, one row per warp): U = 4 at the natural register count
// (config 3s 0.33 -> 0.23 ms/term, 5s 1.26 -> 1.17 ms/term against the
// warp-per-row kernel; re-measured in profiles/r02_ab_sto_group.log)
template <int G, int U, int MINB>
__global__ void __launch_bounds__(256, MINB) batch_group_kernel(const BatchArgs a) {
  constexpr int RPW = 32 / G;
  const int lane = threadIdx.x & 31;
  const int c = 4 * (lane % G);
  const int64_t ngroups = (int64_t)gridDim.x * (blockDim.x >> 5) * RPW;
  const bool need_x = (a.flags & 1) || ((a.flags & 4) && (a.flags & 8));
  const unsigned long long* rec = reinterpret_cast<const unsigned long long*>(a.rec);
  const char* wlb = reinterpret_cast<const char*>(a.win + c);  // the lane's column slice
  const uint32_t ldb = (uint32_t)a.ld * 4u;                    // row stride in bytes (< 2^32)
  for (int64_t row = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * RPW + lane / G;
       row < a.n; row += ngroups) {
    const int32_t b = __ldg(a.start + row), e = __ldg(a.start + row + 1);
    const float4 wr = ld_gather_f4(a.win + row * a.ld + c);
    const float4 xr = need_x ? ld_stream_f4(a.x + row * a.ld + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    float hsum = 0.f;
    for (int32_t p = b; p < e; p += U) {
      unsigned long long r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) r[u] = (p + u < e) ? __ldg(rec + p + u) : 0ull;
      float4 g[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        g[u] = (p + u < e) ? ld_gather_f4(reinterpret_cast<const float*>(
                                 wlb + (uint64_t)(uint32_t)r[u] * ldb))  // one IMAD.WIDE.U32
                           : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float h = __uint_as_float((uint32_t)(r[u] >> 32));  // 0 for padding
        hsum += h;
        acc = f4_fma(-h, g[u], acc);
      }
    }
    float o[4] = {acc.x, acc.y, acc.z, acc.w};
    const float wv[4] = {wr.x, wr.y, wr.z, wr.w};
    const float xv[4] = {xr.x, xr.y, xr.z, xr.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float r = a.beta * fmaf(hsum, wv[i], o[i]);
      if (a.flags & 1) r = fmaf(a.alpha, xv[i], r);
      if (a.flags & 2) r = fmaf(a.gamma, wv[i], r);
      if (a.flags & 4) {
        r *= a.sfin;
        if (a.flags & 8) r = fmaf(a.lamf, xv[i], r);
      }
      o[i] = r;
    }
    st_stream_f4(a.wout + row * a.ld + c, make_float4(o[0], o[1], o[2], o[3]));
  }
}

#ifndef STO_U
#define STO_U 2      // records in flight per group (G <= 16)
#endif
#ifndef STO_MINB
#define STO_MINB 8   // resident blocks (G <= 16)
#endif
template <int G>
void launch_groups(const BatchArgs& a, cudaStream_t s) {
  constexpr int U = G == 32 ? 4 : STO_U;
  constexpr int MINB = G == 32 ? 1 : STO_MINB;
  static PerDeviceOnce once;
  static int per_sm[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  once([&]() -> int {
    int v = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, batch_group_kernel<G, U, MINB>, 256, 0);
    per_sm[dev & 63] = v < 1 ? 1 : v;
    return SPED_OK;
  });
  const int64_t rows_per_block = 8 * (32 / G);
  const int64_t blocks = std::min<int64_t>(
      (a.n + rows_per_block - 1) / rows_per_block,
      (int64_t)num_sms() * std::max(1, per_sm[dev & 63] - a.spare_per_sm));
  batch_group_kernel<G, U, MINB><<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, s>>>(a);
}

template <int LPR, int CPL, bool VEC>
void launch_rows(const BatchArgs& a, cudaStream_t s) {
  // grid = resident capacity (per device); warps stride over rows
  static PerDeviceOnce once;
  static int per_sm[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  once([&]() -> int {
    int v = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, batch_row_kernel<LPR, CPL, VEC>, 256, 0);
    per_sm[dev & 63] = v < 1 ? 1 : v;
    return SPED_OK;
  });
  const int64_t blocks = std::min<int64_t>(
      (a.n + 7) / 8, (int64_t)num_sms() * std::max(1, per_sm[dev & 63] - a.spare_per_sm));
  batch_row_kernel<LPR, CPL, VEC><<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, s>>>(a);
}

#ifndef STO_FORCE_ROWS
#define STO_FORCE_ROWS 0  // A/B builds only: the warp-per-row sweep for every slab
#endif
int launch_batch_slab(const BatchArgs& a, bool aligned, cudaStream_t s) {
  const int k = a.k;
  if (!STO_FORCE_ROWS && aligned && k % 4 == 0) {
    switch (k) {
      case 4: launch_groups<1>(a, s); break;
      case 8: launch_groups<2>(a, s); break;
      case 16: launch_groups<4>(a, s); break;
      case 32: launch_groups<8>(a, s); break;
      case 64: launch_groups<16>(a, s); break;
      case 128: launch_groups<32>(a, s); break;
      default: aligned = false;
    }
    if (aligned) {
      SPED_LAUNCH_CHECK();
      return SPED_OK;
    }
  }
  if (k <= 1) launch_rows<1, 1, false>(a, s);
  else if (k <= 2) launch_rows<2, 1, false>(a, s);
  else if (k <= 4) launch_rows<4, 1, false>(a, s);
  else if (k <= 8) launch_rows<8, 1, false>(a, s);
  else if (k <= 16) launch_rows<16, 1, false>(a, s);
  else if (k <= 32) launch_rows<32, 1, false>(a, s);
  else if (k <= 64) launch_rows<32, 2, false>(a, s);
  else if (k <= 96) launch_rows<32, 3, false>(a, s);
  else launch_rows<32, 4, false>(a, s);
  SPED_LAUNCH_CHECK();
  return SPED_OK;
}

size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

struct BatchWs {
  int32_t *kin, *kout, *start;
  uint64_t *vin, *vout;
  void* tmp;
  size_t tmp_bytes, bytes;
};

// T terms' records (T > 1: one sort for all of them)
BatchWs batch_ws_layout(char* base, int64_t n, int64_t B, int64_t T = 1) {
  BatchWs w{};
  const int64_t R = 2 * B * T;
  size_t off = 0;
  auto take = [&](size_t b) {
    char* p = base ? base + off : nullptr;
    off += align256(b);
    return p;
  };
  w.kin = (int32_t*)take(sizeof(int32_t) * R);
  w.kout = (int32_t*)take(sizeof(int32_t) * R);
  w.vin = (uint64_t*)take(sizeof(uint64_t) * R);
  w.vout = (uint64_t*)take(sizeof(uint64_t) * R);
  w.start = (int32_t*)take(sizeof(int32_t) * (T * (n + 1) + 4));  // <= 4 sort groups
  size_t t = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t, (int32_t*)nullptr, (int32_t*)nullptr,
                                  (uint64_t*)nullptr, (uint64_t*)nullptr, (int)R);
  w.tmp_bytes = t;
  w.tmp = take(t);
  w.bytes = off + 256;
  return w;
}

}  // namespace

int launch_axpby(int64_t count, double a, const float* x, double b, const float* y, float* out,
                 cudaStream_t s);

// Per-device side stream for the record/sort stage (created once; the
// stochastic oracle is single-threaded by contract, it carries its RNG).
static cudaStream_t batch_side_stream() {
  static cudaStream_t st[16] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return nullptr;
  if (!st[dev] && cudaStreamCreateWithFlags(&st[dev], cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    st[dev] = nullptr;
  }
  return st[dev];
}

}  // namespace sped

using namespace sped;

// two record / sort sets: term t+1's records are built and sorted (side
// stream) while term t's row sweep runs
extern "C" int64_t sped_edge_batch_workspace_bytes(int64_t n, int64_t B) {
  return 2 * (int64_t)align256(batch_ws_layout(nullptr, n, std::max<int64_t>(B, 1)).bytes) + 256;
}

// all terms' records sorted at once (one bandwidth-bound sort instead of
// n_terms latency-bound ones) when the keys fit; else the per-term size
static bool all_terms_fit(int64_t n, int64_t B, int64_t T) {
  return T > 1 && 2 * B * T < INT32_MAX && T * (n + 1) < INT32_MAX;
}
extern "C" int64_t sped_edge_batch_workspace_bytes_terms(int64_t n, int64_t B, int32_t n_terms) {
  const int64_t per = sped_edge_batch_workspace_bytes(n, B);
  B = std::max<int64_t>(B, 1);
  if (!all_terms_fit(n, B, n_terms)) return per;
  return std::max<int64_t>(per, (int64_t)batch_ws_layout(nullptr, n, B, n_terms).bytes + 256);
}

// Edge-minibatch apply with an explicit estimator scale (m/B of the global
// batch).  B == 0 (a row shard owning no endpoint of this term's samples):
// every estimate is 0 and only the term epilogues run.
static int edge_batch_apply(int64_t n, int32_t k, int64_t m, const int32_t* indices,
                            const float* edge_w, const int32_t* epos, const int32_t* erow,
                            const int32_t* batch, int64_t B, double scale, void* workspace,
                            int64_t workspace_bytes, const float* x, const float* w_init,
                            float* w_a, float* w_b, float* out, int32_t n_terms,
                            const double* alpha, const double* beta, const double* gamma,
                            double w0_scale, double lam_f, double s_final, sped_stream_t stream);

extern "C" int sped_edge_batch_poly_apply(int64_t n, int32_t k, int64_t m, const int32_t* indices,
                                          const float* edge_w, const int32_t* epos,
                                          const int32_t* erow, const int32_t* batch, int64_t B,
                                          void* workspace, int64_t workspace_bytes,
                                          const float* x, const float* w_init, float* w_a,
                                          float* w_b, float* out, int32_t n_terms,
                                          const double* alpha, const double* beta,
                                          const double* gamma, double w0_scale, double lam_f,
                                          double s_final, sped_stream_t stream) {
  SPED_CHECK_ARG(n >= 0 && k >= 1 && k < (1 << 30) && m >= 0 && B >= 1, "bad sizes");
  return edge_batch_apply(n, k, m, indices, edge_w, epos, erow, batch, B, (double)m / (double)B,
                          workspace, workspace_bytes, x, w_init, w_a, w_b, out, n_terms, alpha,
                          beta, gamma, w0_scale, lam_f, s_final, stream);
}

extern "C" int sped_edge_batch_poly_apply_scaled(
    int64_t n, int32_t k, int64_t m, const int32_t* indices, const float* edge_w,
    const int32_t* epos, const int32_t* erow, const int32_t* batch, int64_t B, double scale,
    void* workspace, int64_t workspace_bytes, const float* x, const float* w_init, float* w_a,
    float* w_b, float* out, int32_t n_terms, const double* alpha, const double* beta,
    const double* gamma, double w0_scale, double lam_f, double s_final, sped_stream_t stream) {
  SPED_CHECK_ARG(n >= 0 && k >= 1 && k < (1 << 30) && m >= 0 && B >= 0, "bad sizes");
  SPED_CHECK_ARG(B == 0 || n_terms <= 1, "a compacted shard batch carries one term");
  return edge_batch_apply(n, k, m, indices, edge_w, epos, erow, batch, B, scale, workspace,
                          workspace_bytes, x, w_init, w_a, w_b, out, n_terms, alpha, beta, gamma,
                          w0_scale, lam_f, s_final, stream);
}

static int edge_batch_apply(int64_t n, int32_t k, int64_t m, const int32_t* indices,
                            const float* edge_w, const int32_t* epos, const int32_t* erow,
                            const int32_t* batch, int64_t B, double scale, void* workspace,
                            int64_t workspace_bytes, const float* x, const float* w_init,
                            float* w_a, float* w_b, float* out, int32_t n_terms,
                            const double* alpha, const double* beta, const double* gamma,
                            double w0_scale, double lam_f, double s_final, sped_stream_t stream) {
  SPED_CHECK_ARG(n_terms >= 0 && (n_terms == 0 || (alpha && beta && gamma)), "bad schedule");
  SPED_CHECK_ARG(x != out && x != w_a && x != w_b, "x must not alias outputs");
  SPED_CHECK_ARG(w_init == nullptr || (w_init != out && w_init != w_a && w_init != w_b),
                 "w_init must not alias outputs");
  SPED_CHECK_ARG(n < INT32_MAX && 2 * B < INT32_MAX, "problem too large");
  if (n == 0) return SPED_OK;
  cudaStream_t s = as_stream(stream);
  if (n_terms == 0) return launch_axpby(n * k, lam_f + s_final * w0_scale, x, 0.0, nullptr, out, s);
  SPED_CHECK_ARG(workspace && (B == 0 || (m > 0 && indices && epos && batch)),
                 "null graph/batch array");
  char* base = (char*)(((uintptr_t)workspace + 255) & ~uintptr_t(255));
  BatchWs wsv[2];
  wsv[0] = batch_ws_layout(base, n, std::max<int64_t>(B, 1));
  wsv[1] = batch_ws_layout(base + align256(wsv[0].bytes), n, std::max<int64_t>(B, 1));
  SPED_CHECK_ARG(workspace_bytes >= (int64_t)(2 * align256(wsv[0].bytes)),
                 "edge batch workspace too small");
  const int32_t slabs = (k + 127) / 128;
  auto sweep = [&](int32_t t, const int32_t* start, const uint64_t* rec, const float* cur,
                   float* dst, int spare) -> int {
    const bool final = (t == n_terms - 1);
    const double sc = (t == 0) ? w0_scale : 1.0;
    for (int32_t sl = 0; sl < slabs; ++sl) {
      const int32_t c0 = sl * 128;
      BatchArgs a;
      a.n = n;
      a.k = min(128, k - c0);
      a.ld = k;
      a.start = start;
      a.rec = rec;
      a.x = x + c0;
      a.win = cur + c0;
      a.wout = dst + c0;
      a.alpha = (float)alpha[t];
      // est is built from the term input w_t = sc * (stored input)
      a.beta = (float)(beta[t] * scale * sc);
      a.gamma = (float)(gamma[t] * sc);
      a.lamf = (float)lam_f;
      a.sfin = (float)s_final;
      a.flags = (alpha[t] != 0.0 ? 1 : 0) | (gamma[t] != 0.0 ? 2 : 0) | (final ? 4 : 0) |
                (lam_f != 0.0 ? 8 : 0);
      a.spare_per_sm = spare;
      const bool aligned = (k % 4 == 0) &&
                           ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(cur) |
                             reinterpret_cast<uintptr_t>(dst)) % 16 == 0);
      int rc = launch_batch_slab(a, aligned, s);
      if (rc != SPED_OK) return rc;
    }
    return SPED_OK;
  };
  if (B == 0) {
    // no sampled endpoint in this shard: empty runs, epilogue only
    SPED_CUDA(cudaMemsetAsync(wsv[0].start, 0, sizeof(int32_t) * (n + 1), s));
    const float* cur = w_init ? w_init : x;
    for (int32_t t = 0; t < n_terms; ++t) {
      float* dst = (t == n_terms - 1) ? out : ((t & 1) == 0 ? w_a : w_b);
      SPED_CHECK_ARG(dst != nullptr, "scratch buffer for term %d is NULL", t);
      int rc = sweep(t, wsv[0].start, wsv[0].vout, cur, dst, 0);
      if (rc != SPED_OK) return rc;
      cur = dst;
    }
    return SPED_OK;
  }
  static const bool all_env = [] {
    const char* e = getenv("SPED_STO_ALLTERMS");
    return !(e && e[0] == '0');
  }();
  if (all_env && all_terms_fit(n, B, n_terms)) {
    BatchWs wa = batch_ws_layout(base, n, B, n_terms);
    if (workspace_bytes >= (int64_t)wa.bytes) {
      // every term's records in one launch, one stable sort by (term, row)
      // -- a row's records keep sample order, as in the per-term sort -- and
      // the run starts of all terms; then the row sweeps
      // Terms are split into G equal groups (one sort each) when that drops
      // the key width to one fewer 8-bit onesweep pass and each group still
      // holds >= 2^22 records (bandwidth-bound); SPED_STO_SPLIT=0: one group.
      static const bool split_env = [] {
        const char* e = getenv("SPED_STO_SPLIT");
        return !(e && e[0] == '0');
      }();
      auto key_bits = [&](int64_t terms) {
        int eb = 1;
        while (eb < 31 && ((int64_t)1 << eb) < terms * (n + 1)) ++eb;  // keys in [0, T(n+1))
        return eb;
      };
      int32_t G = 1;
      if (split_env) {
        const int passes1 = (key_bits(n_terms) + 7) / 8;
        for (int32_t g = 2; g <= 4 && g <= n_terms; ++g) {
          const int64_t tg = (n_terms + g - 1) / g;
          if ((key_bits(tg) + 7) / 8 < passes1 && 2 * B * tg >= (int64_t(1) << 22)) {
            G = g;
            break;
          }
        }
      }
      const int32_t tper = (n_terms + G - 1) / G;
      for (int32_t t0 = 0; t0 < n_terms; t0 += tper) {
        const int32_t tn = min(tper, n_terms - t0);
        const int64_t off = 2 * B * t0, RT = 2 * B * tn, keys = (int64_t)tn * (n + 1);
        records_kernel<<<grid_for(B * tn, 256), 256, 0, s>>>(
            B * tn, B, n, batch + (int64_t)t0 * B, epos, erow, indices, edge_w, wa.kin + off,
            wa.vin + off);
        SPED_LAUNCH_CHECK();
        size_t tb = wa.tmp_bytes;
        SPED_CUDA(cub::DeviceRadixSort::SortPairs(wa.tmp, tb, wa.kin + off, wa.kout + off,
                                                  wa.vin + off, wa.vout + off, (int)RT, 0,
                                                  key_bits(tn), s));
        row_starts_kernel<<<grid_for(RT + 1, 256), 256, 0, s>>>(
            RT, keys, wa.kout + off, wa.start + (int64_t)t0 * (n + 1) + (t0 / tper));
        SPED_LAUNCH_CHECK();
      }
      const float* cur = w_init ? w_init : x;
      for (int32_t t = 0; t < n_terms; ++t) {
        float* dst = (t == n_terms - 1) ? out : ((t & 1) == 0 ? w_a : w_b);
        SPED_CHECK_ARG(dst != nullptr, "scratch buffer for term %d is NULL", t);
        // group g's run starts follow the previous groups' (one extra end
        // entry per group); positions are relative to the group's records
        const int32_t g = t / tper;
        int rc = sweep(t, wa.start + (int64_t)t * (n + 1) + g, wa.vout + 2 * B * (g * tper), cur,
                       dst, 0);
        if (rc != SPED_OK) return rc;
        cur = dst;
      }
      return SPED_OK;
    }
  }
  const int64_t R = 2 * B;
  int end_bit = 1;
  while (end_bit < 31 && ((int64_t)1 << end_bit) <= n) ++end_bit;  // keys in [0, n]
  // Pipeline: the records + stable sort + run starts of term t+1 (side
  // stream, double-buffered workspace) overlap the row sweep of term t; the
  // sweep fills the SMs (SPED_STO_SPARE=j leaves j block slots per SM free
  // for the side stream; 1, 2, 4 measured slower).  SPED_STO_OVERLAP=0
  // runs everything in order on `s`.  Same kernels, same order of summation:
  // the result does not depend on the overlap.
  static const bool overlap_env = [] {
    const char* e = getenv("SPED_STO_OVERLAP");
    return !(e && e[0] == '0');
  }();
  static const int spare_env = [] {
    const char* e = getenv("SPED_STO_SPARE");
    return e ? atoi(e) : 0;
  }();
  cudaStream_t s2 = (overlap_env && n_terms > 1) ? batch_side_stream() : nullptr;
  const bool overlap = s2 != nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ready[2] = {nullptr, nullptr},
              freed[2] = {nullptr, nullptr};
  if (overlap) {
    for (cudaEvent_t* e : {&ev_fork, &ev_join, &ready[0], &ready[1], &freed[0], &freed[1]})
      SPED_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    SPED_CUDA(cudaEventRecord(ev_fork, s));
    SPED_CUDA(cudaStreamWaitEvent(s2, ev_fork, 0));
  }
  cudaStream_t sp = overlap ? s2 : s;  // the record/sort stream
  auto prep = [&](int32_t t) -> int {
    BatchWs& w = wsv[t & 1];
    if (overlap && t >= 2) SPED_CUDA(cudaStreamWaitEvent(sp, freed[t & 1], 0));
    records_kernel<<<grid_for(B, 256), 256, 0, sp>>>(B, B, n, batch + (int64_t)t * B, epos, erow,
                                                     indices, edge_w, w.kin, w.vin);
    SPED_LAUNCH_CHECK();
    size_t tb = w.tmp_bytes;
    // stable: a row's records keep sample order -> fixed summation order
    SPED_CUDA(cub::DeviceRadixSort::SortPairs(w.tmp, tb, w.kin, w.kout, w.vin, w.vout, (int)R, 0,
                                              end_bit, sp));
    row_starts_kernel<<<grid_for(R + 1, 256), 256, 0, sp>>>(R, n, w.kout, w.start);
    SPED_LAUNCH_CHECK();
    if (overlap) SPED_CUDA(cudaEventRecord(ready[t & 1], sp));
    return SPED_OK;
  };
  int rc0 = prep(0);
  if (rc0 != SPED_OK) return rc0;
  const float* cur = w_init ? w_init : x;
  for (int32_t t = 0; t < n_terms; ++t) {
    const bool final = (t == n_terms - 1);
    float* dst = final ? out : ((t & 1) == 0 ? w_a : w_b);
    SPED_CHECK_ARG(dst != nullptr, "scratch buffer for term %d is NULL", t);
    if (t + 1 < n_terms) {
      if (overlap) {
        int rc = prep(t + 1);
        if (rc != SPED_OK) return rc;
      }
    }
    if (overlap) SPED_CUDA(cudaStreamWaitEvent(s, ready[t & 1], 0));
    const BatchWs& ws = wsv[t & 1];
    int rc = sweep(t, ws.start, ws.vout, cur, dst, (overlap && !final) ? spare_env : 0);
    if (rc != SPED_OK) return rc;
    if (overlap) SPED_CUDA(cudaEventRecord(freed[t & 1], s));
    if (!overlap && t + 1 < n_terms) {
      int rc = prep(t + 1);
      if (rc != SPED_OK) return rc;
    }
    cur = dst;
  }
  if (overlap) {
    SPED_CUDA(cudaEventRecord(ev_join, sp));
    SPED_CUDA(cudaStreamWaitEvent(s, ev_join, 0));
    for (cudaEvent_t e : {ev_fork, ev_join, ready[0], ready[1], freed[0], freed[1]})
      cudaEventDestroy(e);  // released once the recorded work completes
  }
  return SPED_OK;
}

extern "C" unsigned int sped_debug_take_edge_batch(void) { return sped::debug_take_unit(); }
