// K9: walk-based polynomial estimator on the device (walks.py:175-341),
// walks bit-identical to the reference's.
//
// The reference samples walks on the EDGE INCIDENCE graph (graph.py:326-342:
// edge e is adjacent to every edge sharing an endpoint, itself included; the
// incident list is sorted by edge id) from numpy Philox streams keyed by
// SeedSequence((seed, chunk)) (walks.py:196-198), 8192 walks per chunk.  Here
// one thread runs one walk:
//   * draw d of a chunk (walk i, step j: d = j*count + i, the order numpy's
//     vectorised sampler consumes its stream in) is word d%4 of the
//     Philox4x64-10 block with counter d/4 + 1 -- numpy increments the counter
//     before each block -- turned into a double as (x >> 11) * 2^-53;
//   * the incidence list is never materialised (it has sum_i deg_i^2 entries):
//     node x's incident edge ids in increasing order are its v == x run (in
//     the stable sort by v) followed by its u == x run (a contiguous id range,
//     the edge list being lexsorted), so the pick-th element of the sorted
//     union of the lists at the edge's two endpoints (the edge itself once) is
//     a k-th-of-two-sorted-arrays binary search;
//   * the walk's prefix contributions coeffs[i] * chain_i / p_i (signs and
//     log magnitudes accumulated as in walks.py:207-222) are summed per walk
//     and emitted as two (node, value) records at the first edge's endpoints;
//     the records are reduced by a stable sort + per-run sequential sums, so the result
//     is deterministic.
// Values are fp64 like the reference; agreement is to fp64 rounding (the
// walks themselves are identical).

#include <cub/cub.cuh>

#include <cmath>

#include "sped_common.cuh"

namespace sped {
namespace {

constexpr int WALK_CHUNK = 8192;  // walks.py:45
constexpr int WALK_MAX_ELL = 64;

__device__ __forceinline__ uint64_t mulhi64(uint64_t a, uint64_t b) { return __umul64hi(a, b); }

// Philox4x64-10 (Random123 constants), the block for `ctr` under `key`.
__device__ __forceinline__ void philox4x64(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3,
                                           uint64_t k0, uint64_t k1, uint64_t out[4]) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t hi0 = mulhi64(M0, c0), lo0 = M0 * c0;
    const uint64_t hi1 = mulhi64(M1, c2), lo1 = M1 * c2;
    const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += W0;
    k1 += W1;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

// numpy Generator(Philox).random() value number d of a fresh stream
__device__ __forceinline__ double philox_uniform(uint64_t k0, uint64_t k1, uint64_t d) {
  uint64_t o[4];
  philox4x64(d / 4 + 1, 0, 0, 0, k0, k1, o);
  const uint64_t x = o[d % 4];
  return (double)(x >> 11) * (1.0 / 9007199254740992.0);
}

struct WalkIndex {
  int64_t n, m;
  const int64_t* u;
  const int64_t* v;
  const double* w;
  const int32_t* up_start;  // n+1: edges with u == x are ids [up_start[x], up_start[x+1])
  const int32_t* lo_start;  // n+1: positions of the v == x run in sorted_e
  const int32_t* sorted_e;  // m: edge ids stably sorted by v
};

// t-th smallest incident edge id of node x
__device__ __forceinline__ int64_t inc_at(const WalkIndex& g, int64_t x, int64_t t) {
  const int64_t lo0 = g.lo_start[x], lo_len = g.lo_start[x + 1] - lo0;
  return t < lo_len ? (int64_t)g.sorted_e[lo0 + t] : (int64_t)g.up_start[x] + (t - lo_len);
}
__device__ __forceinline__ int64_t inc_len(const WalkIndex& g, int64_t x) {
  return (g.lo_start[x + 1] - g.lo_start[x]) + (g.up_start[x + 1] - g.up_start[x]);
}

// q-th smallest (0-based) of the multiset union of node a's and node b's lists
__device__ int64_t kth_of_two(const WalkIndex& g, int64_t a, int64_t na, int64_t b, int64_t nb,
                              int64_t q) {
  int64_t lo = max((int64_t)0, q + 1 - nb), hi = min(q + 1, na);
  while (lo < hi) {  // i = elements taken from a's list among the first q+1
    const int64_t i = (lo + hi) >> 1, j = q + 1 - i;
    if (i < na && j > 0 && inc_at(g, b, j - 1) > inc_at(g, a, i))
      lo = i + 1;
    else
      hi = i;
  }
  const int64_t i = lo, j = q + 1 - i;
  const int64_t va = i > 0 ? inc_at(g, a, i - 1) : -1;
  const int64_t vb = j > 0 ? inc_at(g, b, j - 1) : -1;
  return va > vb ? va : vb;
}

// position of edge e in node x's list (x = v_e: inside the v == x run)
__device__ __forceinline__ int64_t pos_in_lo_run(const WalkIndex& g, int64_t x, int64_t e) {
  int64_t lo = g.lo_start[x], hi = g.lo_start[x + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)g.sorted_e[mid] < e)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo - g.lo_start[x];
}

// pick-th element of edge e's incident list (graph.py:326-342 order)
__device__ __forceinline__ int64_t incident_pick(const WalkIndex& g, int64_t e, int64_t pick) {
  const int64_t a = g.u[e], b = g.v[e];
  const int64_t na = inc_len(g, a), nb = inc_len(g, b);
  const int64_t ia = (g.lo_start[a + 1] - g.lo_start[a]) + (e - g.up_start[a]);
  const int64_t ib = pos_in_lo_run(g, b, e);
  const int64_t first_e = ia + ib;  // e occupies merged positions first_e, first_e + 1
  const int64_t q = pick <= first_e ? pick : pick + 1;
  return kth_of_two(g, a, na, b, nb, q);
}

__device__ __forceinline__ double alpha_pair(const WalkIndex& g, int64_t e1, int64_t e2) {
  const int64_t u1 = g.u[e1], v1 = g.v[e1], u2 = g.u[e2], v2 = g.v[e2];
  return (double)((u1 == u2) + (v1 == v2) - (u1 == v2) - (v1 == u2));
}

struct WalkArgs {
  WalkIndex g;
  int32_t k, ell, mode;  // mode 0 importance, 1 rejection
  double coeffs[WALK_MAX_ELL + 1];
  double log_m, lpmin;
  int64_t walks, n_chunks;
  const uint64_t* keys;  // [k][n_chunks][2]
  const double* x;       // n x k
  int32_t* rec_key;      // 2 * walks * k
  double* rec_val;
};

__global__ void walk_kernel(const WalkArgs a) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t per_col = a.walks;
  if (t >= per_col * a.k) return;
  const int col = (int)(t / per_col);
  const int64_t wi = t - (int64_t)col * per_col;
  const int64_t chunk = wi / WALK_CHUNK, i = wi - chunk * WALK_CHUNK;
  const int64_t count = min((int64_t)WALK_CHUNK, a.walks - chunk * WALK_CHUNK);
  const uint64_t k0 = a.keys[2 * ((int64_t)col * a.n_chunks + chunk)];
  const uint64_t k1 = a.keys[2 * ((int64_t)col * a.n_chunks + chunk) + 1];
  const WalkIndex& g = a.g;
  const double* x = a.x;
  const int K = a.k;

  int64_t e = (int64_t)(philox_uniform(k0, k1, (uint64_t)i) * (double)g.m);
  const int64_t e0 = e;
  double log_p = -a.log_m;  // log p of the full walk (rejection test)
  double deg_cum = 0.0;     // sum of log deg over the edges before the current one
  double lw_cum = log(g.w[e]), la_cum = 0.0, sgn = 1.0;
  double total = 0.0;
  for (int s = 1; s <= a.ell; ++s) {
    // prefix of length s ends at edge e
    if (a.mode == 0 && a.coeffs[s] != 0.0) {
      const double lp = -a.log_m - deg_cum;
      const double logmag = (s == 1) ? lw_cum : lw_cum + la_cum;
      const double coef = a.coeffs[s] * sgn * exp(logmag - lp);
      total += coef * (x[g.u[e] * K + col] - x[g.v[e] * K + col]);
    }
    if (s == a.ell) break;
    const int64_t deg = inc_len(g, g.u[e]) + inc_len(g, g.v[e]) - 1;
    const double r = philox_uniform(k0, k1, (uint64_t)(s * count + i));
    const int64_t pick = (int64_t)(r * (double)deg);
    const int64_t nx = incident_pick(g, e, pick);
    const double ld = log((double)deg);
    log_p -= ld;
    deg_cum += ld;
    const double al = alpha_pair(g, e, nx);
    sgn *= (al > 0.0) ? 1.0 : ((al < 0.0) ? -1.0 : 0.0);
    la_cum += log(fabs(al));
    lw_cum += log(g.w[nx]);
    e = nx;
  }
  if (a.mode == 1) {
    const double r = philox_uniform(k0, k1, (uint64_t)(a.ell * count + i));
    if (r < exp(a.lpmin - log_p)) {
      const double logmag = (a.ell == 1) ? lw_cum : lw_cum + la_cum;
      const double coef = a.coeffs[a.ell] * sgn * exp(logmag);
      total = coef * (x[g.u[e] * K + col] - x[g.v[e] * K + col]);
    } else {
      total = 0.0;
    }
  }
  const int64_t r0 = 2 * t;
  a.rec_key[r0] = (int32_t)(col * g.n + g.u[e0]);
  a.rec_val[r0] = total;
  a.rec_key[r0 + 1] = (int32_t)(col * g.n + g.v[e0]);
  a.rec_val[r0 + 1] = -total;
}

// Sum each run of equal sorted keys in sorted (= walk) order, one thread per
// run, and scatter it to total[node][col].  (cub::DeviceReduce::ReduceByKey
// combined the partial sums of runs spanning tiles in a timing-dependent
// grouping -- decoupled look-back -- so fp64 results differed in the last
// bit between calls.)
__global__ void run_sums_kernel(int64_t count, const int32_t* __restrict__ keys,
                                const double* __restrict__ vals, int64_t n, int32_t k,
                                double* __restrict__ total) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= count) return;
  const int32_t key = keys[i];
  if (i > 0 && keys[i - 1] == key) return;
  double s = 0.0;
  for (int64_t j = i; j < count && keys[j] == key; ++j) s += vals[j];
  const int64_t col = key / n, node = key - col * n;
  total[node * k + col] = s;
}

__global__ void finish_kernel(int64_t nk, double c0, double scale, const double* __restrict__ x,
                              const double* __restrict__ total, double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < nk) out[i] = c0 * x[i] + total[i] * scale;
}

__global__ void walk_index_kernel(int64_t m, const int64_t* __restrict__ v, int32_t* vkey,
                                  int32_t* eval) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m) return;
  vkey[e] = (int32_t)v[e];
  eval[e] = (int32_t)e;
}

template <typename K>
__global__ void walk_run_starts(int64_t m, int64_t n, const K* __restrict__ key,
                                int32_t* __restrict__ start) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t > m) return;
  const int64_t lo = (t == 0) ? -1 : (int64_t)key[t - 1];
  const int64_t hi = (t == m) ? n : (int64_t)key[t];
  for (int64_t i = lo + 1; i <= hi; ++i) start[i] = (int32_t)t;
}

size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

}  // namespace
}  // namespace sped

using namespace sped;

extern "C" int64_t sped_walk_index_workspace_bytes(int64_t n, int64_t m) {
  (void)n;
  const int mm = (int)std::max<int64_t>(m, 1);
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, (int32_t*)nullptr, (int32_t*)nullptr,
                                  (int32_t*)nullptr, (int32_t*)nullptr, mm);
  return (int64_t)(3 * align256(sizeof(int32_t) * mm) + align256(tmp) + 256);
}

extern "C" int sped_walk_index_build(int64_t n, int64_t m, const int64_t* u, const int64_t* v,
                                     int32_t* up_start, int32_t* lo_start, int32_t* sorted_e,
                                     void* workspace, int64_t workspace_bytes,
                                     sped_stream_t stream) {
  SPED_CHECK_ARG(n >= 1 && m >= 1 && u && v && up_start && lo_start && sorted_e && workspace,
                 "bad walk index arguments");
  SPED_CHECK_ARG(n < INT32_MAX && m < INT32_MAX, "graph too large");
  SPED_CHECK_ARG(workspace_bytes >= sped_walk_index_workspace_bytes(n, m), "workspace too small");
  cudaStream_t s = as_stream(stream);
  char* ws = (char*)(((uintptr_t)workspace + 255) & ~uintptr_t(255));
  int32_t* vkey = (int32_t*)ws;
  int32_t* eval = (int32_t*)(ws + align256(sizeof(int32_t) * m));
  int32_t* vsorted = (int32_t*)(ws + 2 * align256(sizeof(int32_t) * m));
  void* tmpb = ws + 3 * align256(sizeof(int32_t) * m);
  size_t tmp = 0;
  SPED_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, vkey, vsorted, eval, sorted_e, (int)m));
  walk_index_kernel<<<grid_for(m, 256), 256, 0, s>>>(m, v, vkey, eval);
  SPED_LAUNCH_CHECK();
  int end_bit = 1;
  while (end_bit < 31 && ((int64_t)1 << end_bit) < n) ++end_bit;
  // stable: equal v keep increasing edge id
  SPED_CUDA(cub::DeviceRadixSort::SortPairs(tmpb, tmp, vkey, vsorted, eval, sorted_e, (int)m, 0,
                                            end_bit, s));
  walk_run_starts<int64_t><<<grid_for(m + 1, 256), 256, 0, s>>>(m, n, u, up_start);
  walk_run_starts<int32_t><<<grid_for(m + 1, 256), 256, 0, s>>>(m, n, vsorted, lo_start);
  SPED_LAUNCH_CHECK();
  return SPED_OK;
}

namespace sped {
namespace {
struct WalkWs {
  int32_t *key_in, *key_out;
  double *val_in, *val_out, *total;
  void* tmp;
  size_t tmp_bytes;
  size_t bytes;
};

WalkWs walk_ws_layout(char* base, int64_t n, int32_t k, int64_t walks) {
  WalkWs w{};
  const int64_t R = 2 * walks * (int64_t)k;
  size_t off = 0;
  auto take = [&](size_t b) {
    char* p = base ? base + off : nullptr;
    off += align256(b);
    return p;
  };
  w.key_in = (int32_t*)take(sizeof(int32_t) * R);
  w.key_out = (int32_t*)take(sizeof(int32_t) * R);
  w.val_in = (double*)take(sizeof(double) * R);
  w.val_out = (double*)take(sizeof(double) * R);
  w.total = (double*)take(sizeof(double) * n * k);
  size_t t1 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t1, (int32_t*)nullptr, (int32_t*)nullptr,
                                  (double*)nullptr, (double*)nullptr, (int)R);
  w.tmp_bytes = t1;
  w.tmp = take(w.tmp_bytes);
  w.bytes = off + 256;
  return w;
}
}  // namespace
}  // namespace sped

extern "C" int64_t sped_walk_workspace_bytes(int64_t n, int32_t k, int64_t walks) {
  return (int64_t)walk_ws_layout(nullptr, n, k, walks).bytes;
}

extern "C" int sped_walk_poly_estimate(int64_t n, int64_t m, int32_t k, const int64_t* u,
                                       const int64_t* v, const double* w,
                                       const int32_t* up_start, const int32_t* lo_start,
                                       const int32_t* sorted_e, int32_t ell, const double* coeffs,
                                       int32_t mode, int64_t deg_star_inc, int64_t walks,
                                       const uint64_t* keys, const double* x, double* out,
                                       void* workspace, int64_t workspace_bytes,
                                       sped_stream_t stream) {
  SPED_CHECK_ARG(n >= 1 && m >= 1 && k >= 1 && walks >= 1 && ell >= 1 && ell <= WALK_MAX_ELL,
                 "bad walk estimate sizes");
  SPED_CHECK_ARG(u && v && w && up_start && lo_start && sorted_e && coeffs && keys && x && out &&
                     workspace,
                 "null walk estimate array");
  SPED_CHECK_ARG(mode == 0 || mode == 1, "mode must be 0 (importance) or 1 (rejection)");
  SPED_CHECK_ARG(n * (int64_t)k < INT32_MAX && 2 * walks * (int64_t)k < INT32_MAX,
                 "walk estimate too large");
  SPED_CHECK_ARG(mode == 0 || deg_star_inc >= 1, "rejection needs deg_star_inc >= 1");
  cudaStream_t s = as_stream(stream);
  char* base = (char*)(((uintptr_t)workspace + 255) & ~uintptr_t(255));
  WalkWs ws = walk_ws_layout(base, n, k, walks);
  SPED_CHECK_ARG(workspace_bytes >= (int64_t)ws.bytes, "walk workspace too small");
  WalkArgs a;
  a.g = WalkIndex{n, m, u, v, w, up_start, lo_start, sorted_e};
  a.k = k;
  a.ell = ell;
  a.mode = mode;
  for (int i = 0; i <= ell; ++i) a.coeffs[i] = coeffs[i];
  a.log_m = std::log((double)m);
  a.lpmin = (mode == 1) ? -(double)ell * std::log((double)deg_star_inc) - std::log((double)m) : 0.0;
  a.walks = walks;
  a.n_chunks = (walks + WALK_CHUNK - 1) / WALK_CHUNK;
  a.keys = keys;
  a.x = x;
  a.rec_key = ws.key_in;
  a.rec_val = ws.val_in;
  const int64_t threads = walks * (int64_t)k;
  walk_kernel<<<grid_for(threads, 128), 128, 0, s>>>(a);
  SPED_LAUNCH_CHECK();
  const int R = (int)(2 * threads);
  int end_bit = 1;
  while (end_bit < 31 && ((int64_t)1 << end_bit) < n * (int64_t)k) ++end_bit;
  size_t tb = ws.tmp_bytes;
  // stable sort by (column, node): records of one node stay in walk order
  SPED_CUDA(cub::DeviceRadixSort::SortPairs(ws.tmp, tb, ws.key_in, ws.key_out, ws.val_in,
                                            ws.val_out, R, 0, end_bit, s));
  SPED_CUDA(cudaMemsetAsync(ws.total, 0, sizeof(double) * n * k, s));
  run_sums_kernel<<<grid_for(R, 256), 256, 0, s>>>(R, ws.key_out, ws.val_out, n, k, ws.total);
  SPED_LAUNCH_CHECK();
  // importance: coeffs[0] x + total / N; rejection: total / (N p_min)
  const double scale = (mode == 0) ? 1.0 / (double)walks
                                   : 1.0 / ((double)walks * std::exp(a.lpmin));
  finish_kernel<<<grid_for(n * k, 256), 256, 0, s>>>(n * (int64_t)k, mode == 0 ? coeffs[0] : 0.0,
                                                     scale, x, ws.total, out);
  SPED_LAUNCH_CHECK();
  return SPED_OK;
}
