// Laplacian CSR construction on the device (replaces
// LaplacianOperator.__post_init__, graph.py:182-199, and Graph.degrees,
// graph.py:118-122).
//
// Input: the canonical edge list (u < v, lexsorted, unique) produced by
// Graph.__post_init__ (graph.py:64-88).  Output: the scipy CSR layout
// (sorted columns, explicit diagonal, isolated rows empty) with values equal
// to fp32(scipy fp64 value):
//   * off-diagonal  -w_e                              (graph.py:189-191)
//   * diagonal      sum of w over incident edges, folded in scipy's
//                   coo->csr input order: the (u,u) block entries in edge
//                   order, then the (v,v) block entries in edge order
//                   (graph.py:189-192; exact for unweighted graphs and for
//                   weighted rows with <= 8 incident edges, where libstdc++'s
//                   std::sort in csr_sort_indices is an insertion sort)
//   * normalized    fl(fl(dinv_i * L_ij) * dinv_j), dinv = 1/sqrt(deg)
//                   (graph.py:193-198, (D L) D evaluated left to right)
// degrees reproduce np.bincount(u,w) + np.bincount(v,w) bit for bit.
//
// Layout choices (B200): entry-parallel, no atomics.  The upper-triangle
// entries of row i are the edges u_e == i (a contiguous run of the lexsorted
// edge list), the lower-triangle entries the edges v_e == i in a stable radix
// sort by v (equal v keep increasing u = edge order), so every entry's CSR
// position is known in closed form and one thread per entry writes it
// (coalesced).  Only the weighted diagonal (and weighted degree) is a
// sequential per-row fold, which bit-exactness requires; unit weights make it
// the integer count.

#include <cub/cub.cuh>

#include "sped_common.cuh"

namespace sped {
namespace {

__global__ void unit_check_kernel(int64_t m, const double* __restrict__ w, int32_t* nonunit) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  bool bad = false;
  for (; e < m; e += stride) bad |= (w[e] != 1.0);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nonunit, 1);
}

__global__ void keys_kernel(int64_t m, const int64_t* __restrict__ v, int32_t* vkey, int32_t* eval) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m) return;
  vkey[e] = (int32_t)v[e];
  eval[e] = (int32_t)e;
}

// start[i] = first index whose key >= i, for a key array sorted ascending
// (start[n] = m).  Thread t covers the rows in (key[t-1], key[t]].
template <typename K>
__global__ void run_starts_kernel(int64_t m, int64_t n, const K* __restrict__ key,
                                  int32_t* __restrict__ start) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t > m) return;
  const int64_t lo = (t == 0) ? -1 : (int64_t)key[t - 1];
  const int64_t hi = (t == m) ? n : (int64_t)key[t];
  for (int64_t i = lo + 1; i <= hi; ++i) start[i] = (int32_t)t;
}

__global__ void rowlen_kernel(int64_t n, const int32_t* __restrict__ up_start,
                              const int32_t* __restrict__ lo_start, int32_t* rowlen) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > n) return;
  if (i == n) {
    rowlen[n] = 0;
    return;
  }
  int32_t d = (up_start[i + 1] - up_start[i]) + (lo_start[i + 1] - lo_start[i]);
  rowlen[i] = d + (d > 0 ? 1 : 0);
}

__global__ void count_zero_kernel(int64_t n, const double* __restrict__ d, int32_t* flag) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n && d[i] == 0.0) atomicExch(flag, 1);
}

// np.bincount(u, w) + np.bincount(v, w): per bin a sequential fold in edge
// order; with unit weights that is the exact integer count
__global__ void degree_kernel(int64_t n, const int32_t* __restrict__ up_start,
                              const int32_t* __restrict__ lo_start,
                              const int32_t* __restrict__ sorted_e,
                              const double* __restrict__ w, const int32_t* __restrict__ nonunit,
                              int normalized, double* __restrict__ degrees,
                              double* __restrict__ dinv, int32_t* zero_flag) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double d;
  if (*nonunit) {
    double su = 0.0;
    for (int32_t e = up_start[i]; e < up_start[i + 1]; ++e) su += w[e];
    double sv = 0.0;
    for (int32_t j = lo_start[i]; j < lo_start[i + 1]; ++j) sv += w[sorted_e[j]];
    d = su + sv;
  } else {
    d = (double)((up_start[i + 1] - up_start[i]) + (lo_start[i + 1] - lo_start[i]));
  }
  degrees[i] = d;
  if (normalized) {
    if (d == 0.0) {
      atomicExch(zero_flag, 1);
      dinv[i] = 0.0;
    } else {
      dinv[i] = 1.0 / sqrt(d);
    }
  }
}

// lower-triangle entries: sorted position j -> edge e with v_e = i, column u_e
__global__ void fill_lower_kernel(int64_t m, const int64_t* __restrict__ u,
                                  const int32_t* __restrict__ sorted_v,
                                  const int32_t* __restrict__ sorted_e,
                                  const double* __restrict__ w,
                                  const int32_t* __restrict__ lo_start,
                                  const int32_t* __restrict__ indptr,
                                  const double* __restrict__ dinv, int normalized,
                                  int32_t* __restrict__ indices, float* __restrict__ values,
                                  int32_t* __restrict__ epos) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= m) return;
  const int32_t i = sorted_v[j];
  const int32_t e = sorted_e[j];
  const int32_t c = (int32_t)u[e];
  const int32_t p = indptr[i] + ((int32_t)j - lo_start[i]);
  SPED_DCHECK(p >= indptr[i] && p < indptr[i + 1], DBG_CSR_POS);
  indices[p] = c;
  if (values) {
    double val = -w[e];
    if (normalized) val = (dinv[i] * val) * dinv[c];
    values[p] = (float)val;
  }
  epos[2 * (int64_t)e + 1] = p;
}

// upper-triangle entries: edge e (lexsorted, u_e = i), column v_e, placed
// after row i's lower entries and its diagonal
__global__ void fill_upper_kernel(int64_t m, const int64_t* __restrict__ u,
                                  const int64_t* __restrict__ v, const double* __restrict__ w,
                                  const int32_t* __restrict__ up_start,
                                  const int32_t* __restrict__ lo_start,
                                  const int32_t* __restrict__ indptr,
                                  const double* __restrict__ dinv, int normalized,
                                  int32_t* __restrict__ indices, float* __restrict__ values,
                                  int32_t* __restrict__ epos) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m) return;
  const int32_t i = (int32_t)u[e];
  const int32_t c = (int32_t)v[e];
  const int32_t p =
      indptr[i] + (lo_start[i + 1] - lo_start[i]) + 1 + ((int32_t)e - up_start[i]);
  SPED_DCHECK(p >= indptr[i] && p < indptr[i + 1], DBG_CSR_POS);
  indices[p] = c;
  if (values) {
    double val = -w[e];
    if (normalized) val = (dinv[i] * val) * dinv[c];
    values[p] = (float)val;
  }
  epos[2 * (int64_t)e] = p;
}

// diagonal: scipy's duplicate fold in coo input order -- the (u,u) block in
// edge order, then the (v,v) block in edge order (graph.py:189-192)
__global__ void fill_diag_kernel(int64_t n, const double* __restrict__ w,
                                 const int32_t* __restrict__ up_start,
                                 const int32_t* __restrict__ lo_start,
                                 const int32_t* __restrict__ sorted_e,
                                 const int32_t* __restrict__ indptr,
                                 const double* __restrict__ dinv,
                                 const int32_t* __restrict__ nonunit, int normalized,
                                 int32_t* __restrict__ indices, float* __restrict__ values) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t up0 = up_start[i], up1 = up_start[i + 1];
  const int32_t lo0 = lo_start[i], lo1 = lo_start[i + 1];
  if (up1 == up0 && lo1 == lo0) return;  // isolated row: empty
  const int32_t p = indptr[i] + (lo1 - lo0);
  indices[p] = (int32_t)i;
  if (!values) return;
  double acc;
  if (*nonunit) {
    acc = 0.0;
    bool first = true;
    for (int32_t e = up0; e < up1; ++e) {
      acc = first ? w[e] : acc + w[e];
      first = false;
    }
    for (int32_t j = lo0; j < lo1; ++j) {
      const double x = w[sorted_e[j]];
      acc = first ? x : acc + x;
      first = false;
    }
  } else {
    acc = (double)((up1 - up0) + (lo1 - lo0));
  }
  if (normalized) acc = (dinv[i] * acc) * dinv[i];
  values[p] = (float)acc;
}

struct AsyncBuf {
  void* p = nullptr;
  cudaStream_t s;
  explicit AsyncBuf(cudaStream_t st) : s(st) {}
  cudaError_t alloc(size_t bytes) { return cudaMallocAsync(&p, bytes ? bytes : 16, s); }
  ~AsyncBuf() {
    if (p) cudaFreeAsync(p, s);
  }
};

}  // namespace
}  // namespace sped

using namespace sped;

extern "C" int sped_laplacian_build(int64_t n, int64_t m, const int64_t* u, const int64_t* v,
                                    const double* w, int normalized, int store_values,
                                    int32_t* indptr, int32_t* indices, float* values,
                                    double* degrees, int32_t* epos, int64_t* nnz_out,
                                    sped_stream_t stream) {
  SPED_CHECK_ARG(n >= 0 && m >= 0, "negative size");
  SPED_CHECK_ARG(n < (int64_t)INT32_MAX && 2 * m + n < (int64_t)INT32_MAX,
                 "graph too large for int32 CSR (n=%lld, m=%lld)", (long long)n, (long long)m);
  SPED_CHECK_ARG(indptr && nnz_out, "null output");
  cudaStream_t s = as_stream(stream);
  if (n == 0) {
    SPED_CUDA(cudaMemsetAsync(indptr, 0, sizeof(int32_t), s));
    SPED_CUDA(cudaStreamSynchronize(s));
    *nnz_out = 0;
    return SPED_OK;
  }
  SPED_CHECK_ARG(m == 0 || (u && v && w && indices && epos && degrees), "null edge/output array");
  SPED_CHECK_ARG(!store_values || values, "values requested but NULL");

  AsyncBuf b_len(s), b_up(s), b_lo(s), b_keys(s), b_vals(s), b_keys2(s), b_vals2(s), b_dinv(s),
      b_flag(s), b_tmp(s);
  SPED_CUDA(b_len.alloc(sizeof(int32_t) * (n + 1)));
  SPED_CUDA(b_up.alloc(sizeof(int32_t) * (n + 1)));
  SPED_CUDA(b_lo.alloc(sizeof(int32_t) * (n + 1)));
  SPED_CUDA(b_keys.alloc(sizeof(int32_t) * m));
  SPED_CUDA(b_vals.alloc(sizeof(int32_t) * m));
  SPED_CUDA(b_keys2.alloc(sizeof(int32_t) * m));
  SPED_CUDA(b_vals2.alloc(sizeof(int32_t) * m));
  SPED_CUDA(b_dinv.alloc(sizeof(double) * n));
  SPED_CUDA(b_flag.alloc(sizeof(int32_t) * 2));  // [zero degree, non-unit weights]
  SPED_CUDA(cudaMemsetAsync(b_flag.p, 0, sizeof(int32_t) * 2, s));
  int32_t* zero_flag_d = (int32_t*)b_flag.p;
  int32_t* nonunit_d = zero_flag_d + 1;

  int32_t* rowlen = (int32_t*)b_len.p;
  int32_t* up_start = (int32_t*)b_up.p;
  int32_t* lo_start = (int32_t*)b_lo.p;
  int32_t* keys = (int32_t*)b_keys.p;
  int32_t* vals = (int32_t*)b_vals.p;
  int32_t* sorted_v = (int32_t*)b_keys2.p;
  int32_t* sorted_e = (int32_t*)b_vals2.p;

  size_t tmp_scan = 0, tmp_sort = 0;
  SPED_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_scan, rowlen, indptr, (int)(n + 1), s));
  int end_bit = 1;
  while (end_bit < 31 && ((int64_t)1 << end_bit) < n) ++end_bit;
  if (m > 0) {
    SPED_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_sort, keys, sorted_v, vals, sorted_e,
                                              (int)m, 0, end_bit, s));
  }
  SPED_CUDA(b_tmp.alloc(tmp_scan > tmp_sort ? tmp_scan : tmp_sort));
  if (m > 0) {
    unit_check_kernel<<<grid_for(m, 256, num_sms() * 8), 256, 0, s>>>(m, w, nonunit_d);
    keys_kernel<<<grid_for(m, 256), 256, 0, s>>>(m, v, keys, vals);
    SPED_LAUNCH_CHECK();
    // stable: equal v keep increasing edge (= u) order, scipy's transpose order
    size_t sb = tmp_sort;
    SPED_CUDA(cub::DeviceRadixSort::SortPairs(b_tmp.p, sb, keys, sorted_v, vals, sorted_e, (int)m,
                                              0, end_bit, s));
  }
  run_starts_kernel<int64_t><<<grid_for(m + 1, 256), 256, 0, s>>>(m, n, u, up_start);
  run_starts_kernel<int32_t><<<grid_for(m + 1, 256), 256, 0, s>>>(m, n, sorted_v, lo_start);
  rowlen_kernel<<<grid_for(n + 1, 256), 256, 0, s>>>(n, up_start, lo_start, rowlen);
  SPED_LAUNCH_CHECK();
  size_t tmp_bytes = tmp_scan;
  SPED_CUDA(cub::DeviceScan::ExclusiveSum(b_tmp.p, tmp_bytes, rowlen, indptr, (int)(n + 1), s));

  degree_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, up_start, lo_start, sorted_e, w, nonunit_d,
                                                   normalized, degrees, (double*)b_dinv.p,
                                                   zero_flag_d);
  SPED_LAUNCH_CHECK();
  int32_t zero_flag = 0;
  SPED_CUDA(cudaMemcpyAsync(&zero_flag, zero_flag_d, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SPED_CUDA(cudaStreamSynchronize(s));
  if (normalized && zero_flag) {
    set_error("normalized Laplacian requires all degrees > 0");
    return SPED_ERR_ZERO_DEGREE;
  }
  const double* dinv = (const double*)b_dinv.p;
  float* vout = store_values ? values : nullptr;
  if (m > 0) {
    fill_lower_kernel<<<grid_for(m, 256), 256, 0, s>>>(m, u, sorted_v, sorted_e, w, lo_start,
                                                         indptr, dinv, normalized, indices, vout,
                                                         epos);
    fill_upper_kernel<<<grid_for(m, 256), 256, 0, s>>>(m, u, v, w, up_start, lo_start, indptr,
                                                         dinv, normalized, indices, vout, epos);
  }
  fill_diag_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, w, up_start, lo_start, sorted_e, indptr,
                                                      dinv, nonunit_d, normalized, indices, vout);
  SPED_LAUNCH_CHECK();
  int32_t nnz = 0;
  SPED_CUDA(cudaMemcpyAsync(&nnz, indptr + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SPED_CUDA(cudaStreamSynchronize(s));
  *nnz_out = nnz;
  return SPED_OK;
}

// ---------------------------------------------------------------------------
// long-row plan

namespace sped {
namespace {
__global__ void plan_count_kernel(int64_t n, const int32_t* __restrict__ indptr, int32_t thresh,
                                  int32_t chunk, int32_t* __restrict__ nch) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > n) return;
  if (i == n) {
    nch[n] = 0;
    return;
  }
  int32_t len = indptr[i + 1] - indptr[i];
  nch[i] = len > thresh ? (len + chunk - 1) / chunk : 0;
}
__global__ void plan_fill_kernel(int64_t n, const int32_t* __restrict__ indptr, int32_t thresh,
                                 int32_t chunk, const int32_t* __restrict__ off,
                                 int32_t* __restrict__ desc) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t b = indptr[i], e = indptr[i + 1];
  if (e - b <= thresh) return;
  int32_t c0 = off[i];
  int32_t c = c0;
  for (int32_t p = b; p < e; p += chunk, ++c) {
    desc[4 * (int64_t)c + 0] = (int32_t)i;
    desc[4 * (int64_t)c + 1] = p;
    desc[4 * (int64_t)c + 2] = min(e, p + chunk);
    desc[4 * (int64_t)c + 3] = c0;
  }
}
__global__ void count_long_rows(int64_t n, const int32_t* __restrict__ nch, int32_t* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n && nch[i] > 0) atomicAdd(out, 1);
}
}  // namespace
}  // namespace sped

extern "C" int64_t sped_spmm_plan_max_chunks(int64_t n, int64_t nnz, int32_t long_threshold,
                                             int32_t chunk_len) {
  if (long_threshold < 1 || chunk_len < 1) return 0;
  (void)n;
  return nnz / chunk_len + nnz / (long_threshold + 1) + 1;
}

extern "C" int sped_spmm_plan(int64_t n, const int32_t* indptr, int32_t long_threshold,
                              int32_t chunk_len, int32_t* chunk_desc, int64_t max_chunks,
                              int64_t* n_chunks_out, int64_t* n_long_rows_out,
                              sped_stream_t stream) {
  SPED_CHECK_ARG(long_threshold >= 1 && chunk_len >= 1, "bad plan parameters");
  SPED_CHECK_ARG(n_chunks_out && n_long_rows_out, "null output");
  cudaStream_t s = as_stream(stream);
  *n_chunks_out = 0;
  *n_long_rows_out = 0;
  if (n == 0) return SPED_OK;
  AsyncBuf b_nch(s), b_off(s), b_tmp(s), b_cnt(s);
  SPED_CUDA(b_nch.alloc(sizeof(int32_t) * (n + 1)));
  SPED_CUDA(b_off.alloc(sizeof(int32_t) * (n + 1)));
  SPED_CUDA(b_cnt.alloc(sizeof(int32_t)));
  SPED_CUDA(cudaMemsetAsync(b_cnt.p, 0, sizeof(int32_t), s));
  int32_t* nch = (int32_t*)b_nch.p;
  int32_t* off = (int32_t*)b_off.p;
  plan_count_kernel<<<grid_for(n + 1, 256), 256, 0, s>>>(n, indptr, long_threshold, chunk_len, nch);
  SPED_LAUNCH_CHECK();
  size_t tmp = 0;
  SPED_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, nch, off, (int)(n + 1), s));
  SPED_CUDA(b_tmp.alloc(tmp));
  SPED_CUDA(cub::DeviceScan::ExclusiveSum(b_tmp.p, tmp, nch, off, (int)(n + 1), s));
  count_long_rows<<<grid_for(n, 256), 256, 0, s>>>(n, nch, (int32_t*)b_cnt.p);
  SPED_LAUNCH_CHECK();
  int32_t total = 0, nlong = 0;
  SPED_CUDA(cudaMemcpyAsync(&total, off + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SPED_CUDA(cudaMemcpyAsync(&nlong, b_cnt.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SPED_CUDA(cudaStreamSynchronize(s));
  SPED_CHECK_ARG(total <= max_chunks, "plan needs %d chunks > capacity %lld", total,
                 (long long)max_chunks);
  if (total > 0) {
    SPED_CHECK_ARG(chunk_desc != nullptr, "null chunk_desc");
    plan_fill_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, indptr, long_threshold, chunk_len, off,
                                                        chunk_desc);
    SPED_LAUNCH_CHECK();
  }
  *n_chunks_out = total;
  *n_long_rows_out = nlong;
  return SPED_OK;
}

// ---------------------------------------------------------------------------
// Degree-descending node order (locality for power-law graphs) and edge
// relabelling.  Hubs get the smallest ids, so the most-gathered rows of every
// block form one contiguous prefix that the SpMM keeps L2-resident
// (a persisting-L2 window over the prefix); rows also come sorted by
// length, which lets the SpMM pick a lanes-per-row width per row range.

namespace sped {
namespace {
__global__ void rowlen_key_kernel(int64_t n, const int32_t* __restrict__ indptr,
                                  int32_t* __restrict__ key, int32_t* __restrict__ ids) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  key[i] = indptr[i + 1] - indptr[i];
  ids[i] = (int32_t)i;
}
__global__ void invert_perm_kernel(int64_t n, const int32_t* __restrict__ perm,
                                   int32_t* __restrict__ iperm) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) iperm[perm[i]] = (int32_t)i;
}
__global__ void relabel_key_kernel(int64_t m, int64_t n, const int64_t* __restrict__ u,
                                   const int64_t* __restrict__ v,
                                   const int32_t* __restrict__ iperm,
                                   unsigned long long* __restrict__ key, int32_t* __restrict__ ids) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m) return;
  const int64_t a = iperm[u[e]], b = iperm[v[e]];
  const int64_t lo = a < b ? a : b, hi = a < b ? b : a;
  key[e] = (unsigned long long)(lo * n + hi);
  ids[e] = (int32_t)e;
}
__global__ void relabel_gather_kernel(int64_t m, int64_t n, const unsigned long long* __restrict__ key,
                                      const int32_t* __restrict__ ids, const double* __restrict__ w,
                                      int64_t* __restrict__ u2, int64_t* __restrict__ v2,
                                      double* __restrict__ w2) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m) return;
  const unsigned long long kk = key[e];
  u2[e] = (int64_t)(kk / (unsigned long long)n);
  v2[e] = (int64_t)(kk % (unsigned long long)n);
  w2[e] = w[ids[e]];
}
}  // namespace
}  // namespace sped

extern "C" int sped_degree_order(int64_t n, const int32_t* indptr, int32_t* perm, int32_t* iperm,
                                 sped_stream_t stream) {
  SPED_CHECK_ARG(n >= 0 && n < INT32_MAX, "bad n");
  if (n == 0) return SPED_OK;
  SPED_CHECK_ARG(indptr && perm && iperm, "null array");
  cudaStream_t s = as_stream(stream);
  AsyncBuf b_key(s), b_key2(s), b_ids(s), b_tmp(s);
  SPED_CUDA(b_key.alloc(sizeof(int32_t) * n));
  SPED_CUDA(b_key2.alloc(sizeof(int32_t) * n));
  SPED_CUDA(b_ids.alloc(sizeof(int32_t) * n));
  rowlen_key_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, indptr, (int32_t*)b_key.p, (int32_t*)b_ids.p);
  SPED_LAUNCH_CHECK();
  size_t tmp = 0;
  SPED_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp, (int32_t*)b_key.p,
                                                      (int32_t*)b_key2.p, (int32_t*)b_ids.p, perm,
                                                      (int)n, 0, 32, s));
  SPED_CUDA(b_tmp.alloc(tmp));
  SPED_CUDA(cub::DeviceRadixSort::SortPairsDescending(b_tmp.p, tmp, (int32_t*)b_key.p,
                                                      (int32_t*)b_key2.p, (int32_t*)b_ids.p, perm,
                                                      (int)n, 0, 32, s));
  invert_perm_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, perm, iperm);
  SPED_LAUNCH_CHECK();
  return SPED_OK;
}

extern "C" int sped_relabel_edges(int64_t n, int64_t m, const int64_t* u, const int64_t* v,
                                  const double* w, const int32_t* iperm, int64_t* u2, int64_t* v2,
                                  double* w2, int32_t* edge_map, sped_stream_t stream) {
  SPED_CHECK_ARG(n >= 0 && m >= 0 && m < INT32_MAX, "bad sizes");
  if (m == 0) return SPED_OK;
  SPED_CHECK_ARG(u && v && w && iperm && u2 && v2 && w2 && edge_map, "null array");
  cudaStream_t s = as_stream(stream);
  AsyncBuf b_key(s), b_key2(s), b_ids(s), b_tmp(s);
  SPED_CUDA(b_key.alloc(sizeof(unsigned long long) * m));
  SPED_CUDA(b_key2.alloc(sizeof(unsigned long long) * m));
  SPED_CUDA(b_ids.alloc(sizeof(int32_t) * m));
  relabel_key_kernel<<<grid_for(m, 256), 256, 0, s>>>(m, n, u, v, iperm,
                                                        (unsigned long long*)b_key.p,
                                                        (int32_t*)b_ids.p);
  SPED_LAUNCH_CHECK();
  int end_bit = 1;
  const unsigned long long maxkey = (unsigned long long)n * (unsigned long long)n;
  while (end_bit < 64 && (1ULL << end_bit) < maxkey) ++end_bit;
  size_t tmp = 0;
  SPED_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, (unsigned long long*)b_key.p,
                                            (unsigned long long*)b_key2.p, (int32_t*)b_ids.p,
                                            edge_map, (int)m, 0, end_bit, s));
  SPED_CUDA(b_tmp.alloc(tmp));
  SPED_CUDA(cub::DeviceRadixSort::SortPairs(b_tmp.p, tmp, (unsigned long long*)b_key.p,
                                            (unsigned long long*)b_key2.p, (int32_t*)b_ids.p,
                                            edge_map, (int)m, 0, end_bit, s));
  relabel_gather_kernel<<<grid_for(m, 256), 256, 0, s>>>(m, n, (unsigned long long*)b_key2.p,
                                                           edge_map, w, u2, v2, w2);
  SPED_LAUNCH_CHECK();
  return SPED_OK;
}

// ---------------------------------------------------------------------------
// Graph canonicalisation on the device (Graph.__post_init__, graph.py:64-88):
// drop zero-weight edges, validate (negative weights, self loops, endpoint
// range, duplicate unordered pairs -- the reference's checks and order of
// precedence), orient u < v and sort lexicographically by (u, v).  The key
// lo*n + hi is unique per unordered pair, so an integer radix sort gives the
// reference's lexsort order bit for bit.  Dropped / invalid edges get a
// sentinel key that sorts after every valid one.

namespace sped {
namespace {
enum CanonStatus : int { CS_NEG = 1, CS_SELF = 2, CS_RANGE = 4, CS_DUP = 8 };

__global__ void canon_key_kernel(int64_t m, int64_t n, const int64_t* __restrict__ u,
                                 const int64_t* __restrict__ v, const double* __restrict__ w,
                                 unsigned long long sentinel, unsigned long long* __restrict__ key,
                                 int32_t* __restrict__ ids, int32_t* __restrict__ keep,
                                 int* __restrict__ status) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m) return;
  const double we = w[e];
  const int64_t a = u[e], b = v[e];
  int st = 0;
  bool kept = false;
  if (we < 0.0) {
    st |= CS_NEG;
  } else if (we > 0.0) {
    if (a == b) st |= CS_SELF;
    if (a < 0 || a >= n || b < 0 || b >= n) st |= CS_RANGE;
    kept = (st == 0);
  }
  if (st) atomicOr(status, st);
  const int64_t lo = a < b ? a : b, hi = a < b ? b : a;
  key[e] = kept ? (unsigned long long)(lo * n + hi) : sentinel;
  ids[e] = (int32_t)e;
  keep[e] = (we > 0.0) ? 1 : 0;  // the reference drops w == 0 before its checks
}

__global__ void canon_gather_kernel(int64_t mk, int64_t n, const unsigned long long* __restrict__ key,
                                    const int32_t* __restrict__ ids, const double* __restrict__ w,
                                    int64_t* __restrict__ u2, int64_t* __restrict__ v2,
                                    double* __restrict__ w2, int* __restrict__ status) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= mk) return;
  const unsigned long long kk = key[e];
  if (e > 0 && key[e - 1] == kk) atomicOr(status, CS_DUP);
  u2[e] = (int64_t)(kk / (unsigned long long)n);
  v2[e] = (int64_t)(kk % (unsigned long long)n);
  w2[e] = w[ids[e]];
}
}  // namespace
}  // namespace sped

extern "C" int sped_canonicalize_edges(int64_t n, int64_t m, const int64_t* u, const int64_t* v,
                                       const double* w, int64_t* u2, int64_t* v2, double* w2,
                                       int64_t* m_out, int32_t* status_out,
                                       sped_stream_t stream) {
  SPED_CHECK_ARG(n >= 0 && m >= 0 && m < INT32_MAX, "bad sizes");
  SPED_CHECK_ARG(m_out && status_out, "null output");
  SPED_CHECK_ARG((double)n * (double)n < 9.2e18, "node count too large for 64-bit pair keys");
  *m_out = 0;
  *status_out = 0;
  if (m == 0) return SPED_OK;
  SPED_CHECK_ARG(u && v && w && u2 && v2 && w2, "null array");
  cudaStream_t s = as_stream(stream);
  AsyncBuf b_key(s), b_key2(s), b_ids(s), b_ids2(s), b_keep(s), b_cnt(s), b_tmp(s), b_tmp2(s);
  SPED_CUDA(b_key.alloc(sizeof(unsigned long long) * m));
  SPED_CUDA(b_key2.alloc(sizeof(unsigned long long) * m));
  SPED_CUDA(b_ids.alloc(sizeof(int32_t) * m));
  SPED_CUDA(b_ids2.alloc(sizeof(int32_t) * m));
  SPED_CUDA(b_keep.alloc(sizeof(int32_t) * m));
  SPED_CUDA(b_cnt.alloc(sizeof(int64_t) + sizeof(int)));
  int64_t* d_cnt = (int64_t*)b_cnt.p;
  int* d_status = (int*)(d_cnt + 1);
  SPED_CUDA(cudaMemsetAsync(d_status, 0, sizeof(int), s));
  // 2^end_bit > n*n: every valid key < n*n - n, the sentinel 2^end_bit - 1
  int end_bit = 1;
  const unsigned long long nn = (unsigned long long)n * (unsigned long long)n;
  while (end_bit < 64 && (1ULL << end_bit) <= nn) ++end_bit;
  const unsigned long long sentinel = (end_bit >= 64) ? ~0ULL : ((1ULL << end_bit) - 1ULL);
  canon_key_kernel<<<grid_for(m, 256), 256, 0, s>>>(m, n, u, v, w, sentinel,
                                                      (unsigned long long*)b_key.p,
                                                      (int32_t*)b_ids.p, (int32_t*)b_keep.p,
                                                      d_status);
  SPED_LAUNCH_CHECK();
  size_t t1 = 0, t2 = 0;
  SPED_CUDA(cub::DeviceReduce::Sum(nullptr, t2, (int32_t*)b_keep.p, d_cnt, (int)m, s));
  SPED_CUDA(b_tmp2.alloc(t2));
  SPED_CUDA(cub::DeviceReduce::Sum(b_tmp2.p, t2, (int32_t*)b_keep.p, d_cnt, (int)m, s));
  SPED_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t1, (unsigned long long*)b_key.p,
                                            (unsigned long long*)b_key2.p, (int32_t*)b_ids.p,
                                            (int32_t*)b_ids2.p, (int)m, 0, end_bit, s));
  SPED_CUDA(b_tmp.alloc(t1));
  SPED_CUDA(cub::DeviceRadixSort::SortPairs(b_tmp.p, t1, (unsigned long long*)b_key.p,
                                            (unsigned long long*)b_key2.p, (int32_t*)b_ids.p,
                                            (int32_t*)b_ids2.p, (int)m, 0, end_bit, s));
  int64_t mk = 0;
  int st = 0;
  SPED_CUDA(cudaMemcpyAsync(&mk, d_cnt, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SPED_CUDA(cudaMemcpyAsync(&st, d_status, sizeof(int), cudaMemcpyDeviceToHost, s));
  SPED_CUDA(cudaStreamSynchronize(s));
  if (st == 0 && mk > 0) {
    canon_gather_kernel<<<grid_for(mk, 256), 256, 0, s>>>(mk, n, (unsigned long long*)b_key2.p,
                                                            (int32_t*)b_ids2.p, w, u2, v2, w2,
                                                            d_status);
    SPED_LAUNCH_CHECK();
    SPED_CUDA(cudaMemcpyAsync(&st, d_status, sizeof(int), cudaMemcpyDeviceToHost, s));
    SPED_CUDA(cudaStreamSynchronize(s));
  }
  *m_out = mk;
  *status_out = st;
  return SPED_OK;
}

// ---------------------------------------------------------------------------
// Row-range build for one row shard: rows [b, e) of the same
// CSR, from the edges incident to those rows only.  Input: any lexsorted
// subsequence of the canonical edge list that contains every edge with an
// endpoint in [b, e) (other edges are ignored), so a rank never holds the
// whole graph.  The entries of row i are built exactly as in
// sped_laplacian_build (lower run by a stable sort on v, diagonal, upper run
// = the contiguous u-run of the lexsorted list), so the shard rows are
// bit-identical to rows [b, e) of the full build.  Normalized values need
// d^-1/2 of the halo columns too: the caller passes every node's degree
// (the all-gather of the shards' own degrees).

namespace sped {
namespace {
__device__ __forceinline__ int64_t clamp_row(int64_t x, int64_t b, int64_t nr) {
  const int64_t r = x - b;
  return r < 0 ? -1 : (r > nr ? nr : r);
}

// up_start[i] = first edge whose u - b >= i, i in [0, nr]
__global__ void range_up_starts_kernel(int64_t m, int64_t nr, int64_t b,
                                       const int64_t* __restrict__ u, int32_t* __restrict__ start) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t > m) return;
  const int64_t lo = (t == 0) ? -1 : clamp_row(u[t - 1], b, nr);
  const int64_t hi = (t == m) ? nr : clamp_row(u[t], b, nr);
  for (int64_t i = lo + 1; i <= hi; ++i) start[i] = (int32_t)t;
}

// lower-run sort keys: local row of v (nr = not in this shard)
__global__ void range_keys_kernel(int64_t m, int64_t nr, int64_t b, const int64_t* __restrict__ v,
                                  int32_t* __restrict__ vkey, int32_t* __restrict__ eval) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m) return;
  const int64_t r = v[e] - b;
  vkey[e] = (r >= 0 && r < nr) ? (int32_t)r : (int32_t)nr;
  eval[e] = (int32_t)e;
}

__device__ __forceinline__ double dinv_of(const double* deg, int64_t c) { return 1.0 / sqrt(deg[c]); }

__global__ void range_degree_kernel(int64_t nr, const int32_t* __restrict__ up_start,
                                    const int32_t* __restrict__ lo_start,
                                    const int32_t* __restrict__ sorted_e,
                                    const double* __restrict__ w, const int32_t* __restrict__ nonunit,
                                    double* __restrict__ degrees) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nr) return;
  double d;
  if (*nonunit) {
    double su = 0.0;
    for (int32_t e = up_start[i]; e < up_start[i + 1]; ++e) su += w[e];
    double sv = 0.0;
    for (int32_t j = lo_start[i]; j < lo_start[i + 1]; ++j) sv += w[sorted_e[j]];
    d = su + sv;
  } else {
    d = (double)((up_start[i + 1] - up_start[i]) + (lo_start[i + 1] - lo_start[i]));
  }
  degrees[i] = d;
}

__global__ void range_fill_lower_kernel(int64_t n_lo, int64_t b, const int64_t* __restrict__ u,
                                        const int32_t* __restrict__ sorted_v,
                                        const int32_t* __restrict__ sorted_e,
                                        const double* __restrict__ w,
                                        const int32_t* __restrict__ lo_start,
                                        const int32_t* __restrict__ indptr,
                                        const double* __restrict__ col_deg, int normalized,
                                        int32_t* __restrict__ indices, float* __restrict__ values,
                                        int32_t* __restrict__ epos) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n_lo) return;
  const int32_t i = sorted_v[j];  // local row
  const int32_t e = sorted_e[j];
  const int64_t c = u[e];
  const int32_t p = indptr[i] + ((int32_t)j - lo_start[i]);
  SPED_DCHECK(p >= indptr[i] && p < indptr[i + 1], DBG_CSR_POS);
  indices[p] = (int32_t)c;
  if (values) {
    double val = -w[e];
    if (normalized) val = (dinv_of(col_deg, b + i) * val) * dinv_of(col_deg, c);
    values[p] = (float)val;
  }
  epos[2 * (int64_t)e + 1] = p;
}

__global__ void range_fill_upper_kernel(int64_t e0, int64_t e1, int64_t b,
                                        const int64_t* __restrict__ u, const int64_t* __restrict__ v,
                                        const double* __restrict__ w,
                                        const int32_t* __restrict__ up_start,
                                        const int32_t* __restrict__ lo_start,
                                        const int32_t* __restrict__ indptr,
                                        const double* __restrict__ col_deg, int normalized,
                                        int32_t* __restrict__ indices, float* __restrict__ values,
                                        int32_t* __restrict__ epos) {
  const int64_t e = e0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= e1) return;
  const int32_t i = (int32_t)(u[e] - b);
  const int64_t c = v[e];
  const int32_t p = indptr[i] + (lo_start[i + 1] - lo_start[i]) + 1 + ((int32_t)e - up_start[i]);
  SPED_DCHECK(p >= indptr[i] && p < indptr[i + 1], DBG_CSR_POS);
  indices[p] = (int32_t)c;
  if (values) {
    double val = -w[e];
    if (normalized) val = (dinv_of(col_deg, b + i) * val) * dinv_of(col_deg, c);
    values[p] = (float)val;
  }
  epos[2 * e] = p;
}

__global__ void range_fill_diag_kernel(int64_t nr, int64_t b, const double* __restrict__ w,
                                       const int32_t* __restrict__ up_start,
                                       const int32_t* __restrict__ lo_start,
                                       const int32_t* __restrict__ sorted_e,
                                       const int32_t* __restrict__ indptr,
                                       const double* __restrict__ col_deg,
                                       const int32_t* __restrict__ nonunit, int normalized,
                                       int32_t* __restrict__ indices, float* __restrict__ values) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nr) return;
  const int32_t up0 = up_start[i], up1 = up_start[i + 1];
  const int32_t lo0 = lo_start[i], lo1 = lo_start[i + 1];
  if (up1 == up0 && lo1 == lo0) return;
  const int32_t p = indptr[i] + (lo1 - lo0);
  indices[p] = (int32_t)(b + i);
  if (!values) return;
  double acc;
  if (*nonunit) {
    acc = 0.0;
    bool first = true;
    for (int32_t e = up0; e < up1; ++e) {
      acc = first ? w[e] : acc + w[e];
      first = false;
    }
    for (int32_t j = lo0; j < lo1; ++j) {
      const double x = w[sorted_e[j]];
      acc = first ? x : acc + x;
      first = false;
    }
  } else {
    acc = (double)((up1 - up0) + (lo1 - lo0));
  }
  if (normalized) {
    const double di = dinv_of(col_deg, b + i);
    acc = (di * acc) * di;
  }
  values[p] = (float)acc;
}
}  // namespace
}  // namespace sped

extern "C" int sped_laplacian_build_rows(int64_t n, int64_t row_begin, int64_t row_end, int64_t m,
                                         const int64_t* u, const int64_t* v, const double* w,
                                         const double* col_degrees, int normalized,
                                         int store_values, int32_t* indptr, int32_t* indices,
                                         float* values, double* degrees, int32_t* epos,
                                         int64_t* nnz_out, sped_stream_t stream) {
  SPED_CHECK_ARG(n >= 0 && m >= 0 && row_begin >= 0 && row_begin <= row_end && row_end <= n,
                 "bad row range [%lld, %lld) of n=%lld", (long long)row_begin, (long long)row_end,
                 (long long)n);
  const int64_t nr = row_end - row_begin;
  SPED_CHECK_ARG(n < (int64_t)INT32_MAX && 2 * m + nr < (int64_t)INT32_MAX,
                 "shard too large for int32 CSR (rows=%lld, m=%lld)", (long long)nr, (long long)m);
  SPED_CHECK_ARG(indptr && nnz_out, "null output");
  SPED_CHECK_ARG(!normalized || !store_values || col_degrees,
                 "normalized values need every node's degree (col_degrees)");
  cudaStream_t s = as_stream(stream);
  *nnz_out = 0;
  if (nr == 0) {
    SPED_CUDA(cudaMemsetAsync(indptr, 0, sizeof(int32_t), s));
    if (m > 0 && epos) SPED_CUDA(cudaMemsetAsync(epos, 0xFF, sizeof(int32_t) * 2 * m, s));
    SPED_CUDA(cudaStreamSynchronize(s));
    return SPED_OK;
  }
  SPED_CHECK_ARG(m == 0 || (u && v && w && indices && epos && degrees), "null edge/output array");
  SPED_CHECK_ARG(!store_values || values, "values requested but NULL");
  SPED_CHECK_ARG(degrees, "null degrees");

  AsyncBuf b_len(s), b_up(s), b_lo(s), b_keys(s), b_vals(s), b_keys2(s), b_vals2(s), b_flag(s),
      b_tmp(s);
  SPED_CUDA(b_len.alloc(sizeof(int32_t) * (nr + 1)));
  SPED_CUDA(b_up.alloc(sizeof(int32_t) * (nr + 1)));
  SPED_CUDA(b_lo.alloc(sizeof(int32_t) * (nr + 1)));
  SPED_CUDA(b_keys.alloc(sizeof(int32_t) * m));
  SPED_CUDA(b_vals.alloc(sizeof(int32_t) * m));
  SPED_CUDA(b_keys2.alloc(sizeof(int32_t) * m));
  SPED_CUDA(b_vals2.alloc(sizeof(int32_t) * m));
  SPED_CUDA(b_flag.alloc(sizeof(int32_t)));
  SPED_CUDA(cudaMemsetAsync(b_flag.p, 0, sizeof(int32_t), s));
  int32_t* nonunit_d = (int32_t*)b_flag.p;
  int32_t* rowlen = (int32_t*)b_len.p;
  int32_t* up_start = (int32_t*)b_up.p;
  int32_t* lo_start = (int32_t*)b_lo.p;
  int32_t* keys = (int32_t*)b_keys.p;
  int32_t* vals = (int32_t*)b_vals.p;
  int32_t* sorted_v = (int32_t*)b_keys2.p;
  int32_t* sorted_e = (int32_t*)b_vals2.p;

  size_t tmp_scan = 0, tmp_sort = 0;
  SPED_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_scan, rowlen, indptr, (int)(nr + 1), s));
  int end_bit = 1;
  while (end_bit < 31 && ((int64_t)1 << end_bit) <= nr) ++end_bit;  // keys in [0, nr]
  if (m > 0)
    SPED_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_sort, keys, sorted_v, vals, sorted_e,
                                              (int)m, 0, end_bit, s));
  SPED_CUDA(b_tmp.alloc(tmp_scan > tmp_sort ? tmp_scan : tmp_sort));
  if (m > 0) {
    SPED_CUDA(cudaMemsetAsync(epos, 0xFF, sizeof(int32_t) * 2 * m, s));  // -1: row not in shard
    unit_check_kernel<<<grid_for(m, 256, num_sms() * 8), 256, 0, s>>>(m, w, nonunit_d);
    range_keys_kernel<<<grid_for(m, 256), 256, 0, s>>>(m, nr, row_begin, v, keys, vals);
    SPED_LAUNCH_CHECK();
    size_t sb = tmp_sort;
    SPED_CUDA(cub::DeviceRadixSort::SortPairs(b_tmp.p, sb, keys, sorted_v, vals, sorted_e, (int)m,
                                              0, end_bit, s));
  }
  range_up_starts_kernel<<<grid_for(m + 1, 256), 256, 0, s>>>(m, nr, row_begin, u, up_start);
  run_starts_kernel<int32_t><<<grid_for(m + 1, 256), 256, 0, s>>>(m, nr, sorted_v, lo_start);
  rowlen_kernel<<<grid_for(nr + 1, 256), 256, 0, s>>>(nr, up_start, lo_start, rowlen);
  SPED_LAUNCH_CHECK();
  size_t tmp_bytes = tmp_scan;
  SPED_CUDA(cub::DeviceScan::ExclusiveSum(b_tmp.p, tmp_bytes, rowlen, indptr, (int)(nr + 1), s));
  range_degree_kernel<<<grid_for(nr, 256), 256, 0, s>>>(nr, up_start, lo_start, sorted_e, w,
                                                          nonunit_d, degrees);
  SPED_LAUNCH_CHECK();
  int32_t bounds[3] = {0, 0, 0};  // up_start[0], up_start[nr], lo_start[nr]
  SPED_CUDA(cudaMemcpyAsync(&bounds[0], up_start, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SPED_CUDA(cudaMemcpyAsync(&bounds[1], up_start + nr, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SPED_CUDA(cudaMemcpyAsync(&bounds[2], lo_start + nr, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SPED_CUDA(cudaStreamSynchronize(s));
  if (normalized) {
    // the shard's own rows: a zero degree is the reference's ValueError
    // (graph.py:187-188); callers check the gathered degree vector globally
    AsyncBuf b_z(s);
    SPED_CUDA(b_z.alloc(sizeof(int32_t)));
    SPED_CUDA(cudaMemsetAsync(b_z.p, 0, sizeof(int32_t), s));
    count_zero_kernel<<<grid_for(nr, 256), 256, 0, s>>>(nr, degrees, (int32_t*)b_z.p);
    SPED_LAUNCH_CHECK();
    int32_t z = 0;
    SPED_CUDA(cudaMemcpyAsync(&z, b_z.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SPED_CUDA(cudaStreamSynchronize(s));
    if (z) {
      set_error("normalized Laplacian requires all degrees > 0");
      return SPED_ERR_ZERO_DEGREE;
    }
  }
  float* vout = store_values ? values : nullptr;
  const int64_t n_lo = bounds[2];
  if (n_lo > 0)
    range_fill_lower_kernel<<<grid_for(n_lo, 256), 256, 0, s>>>(
        n_lo, row_begin, u, sorted_v, sorted_e, w, lo_start, indptr, col_degrees, normalized,
        indices, vout, epos);
  if (bounds[1] > bounds[0])
    range_fill_upper_kernel<<<grid_for(bounds[1] - bounds[0], 256), 256, 0, s>>>(
        bounds[0], bounds[1], row_begin, u, v, w, up_start, lo_start, indptr, col_degrees,
        normalized, indices, vout, epos);
  range_fill_diag_kernel<<<grid_for(nr, 256), 256, 0, s>>>(nr, row_begin, w, up_start, lo_start,
                                                             sorted_e, indptr, col_degrees,
                                                             nonunit_d, normalized, indices, vout);
  SPED_LAUNCH_CHECK();
  int32_t nnz = 0;
  SPED_CUDA(cudaMemcpyAsync(&nnz, indptr + nr, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SPED_CUDA(cudaStreamSynchronize(s));
  *nnz_out = nnz;
  return SPED_OK;
}

extern "C" unsigned int sped_debug_take_csr(void) { return sped::debug_take_unit(); }
