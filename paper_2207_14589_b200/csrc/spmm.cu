// K1: CSR SpMM with the dilation-polynomial recurrence fused into the
// epilogue (replaces the ell x `L.matvec` + numpy axpys of
// TransformedOperator.apply, transforms.py:241-262 / graph.py:211).
//
// One term:  w' = alpha*x + beta*(L w) + gamma*w
// last term: out = lam_f*x + s*w'
// so every intermediate block is written exactly once.
//
// Mapping (sm_100a, HBM/L2-gather bound):
//  * a row is owned by G = LPR*SUB lanes: LPR lanes cover its k columns with
//    W-float (256-bit when k >= 32 and rows are 32-B aligned) loads, SUB
//    lane slices split its nonzeros; lanes per row and SUB are chosen per
//    row RANGE (degree-sorted rows) from a segment table;
//  * shuffle-free: every lane slice walks its own nonzeros, reading column
//    indices (and values) through L1, with U independent row gathers in
//    flight -- no warp-uniform trip count, no index broadcast; the SUB
//    partials fold with an xor tree (free_accumulate);
//  * rows longer than `long_thresh` are cut into chunks (sped_spmm_plan);
//    the last chunk of a row to arrive (ticket) folds the partials in chunk
//    order and applies the epilogue -> deterministic, no float atomics;
//  * degree-relabelled graphs: a persisting-L2 access-policy window over
//    the hub prefix of the gathered block keeps the most-gathered rows in L2;
//  * unweighted combinatorial Laplacians use implicit values (-1 off the
//    diagonal, row_len-1 on it): 4 B per nonzero instead of 8;
//  * unweighted NORMALIZED Laplacians (no self loops) run every term after
//    the first on the scaled block u = D^-1/2 w: (L w)_i = w_i -
//    d_i^-1/2 sum_{j~i} u_j needs no values either (VM 2, row_scale = d^-1/2).
//  * column slabs of <= 128 floats (row stride `ld`) cover any k.

#include <cstdlib>

#include "sped_common.cuh"

#ifndef CHUNK_MIN_BLOCKS
#define CHUNK_MIN_BLOCKS 5  // with LONG_MIN_BLOCKS 5 / FREE_LONG_U 3: config 4 2.520 -> 2.481 ms/term (r02_ab_long_occupancy_cfg4.log)
#endif
#ifndef CHUNK_W8_MIN_K
#define CHUNK_W8_MIN_K 32  // free kernels: 256-bit hub gathers at k = 32 too (config 4: 2.548 -> 2.522 ms/term, r02_ab_chunk_width_cfg4.log)
#endif
#ifndef LONG_MIN_BLOCKS
#define LONG_MIN_BLOCKS 5
#endif

namespace sped {

enum TermFlags : int {
  TF_ALPHA = 1,   // alpha != 0: read x
  TF_GAMMA = 2,   // gamma != 0: read w row
  TF_FINAL = 4,   // last term: out = lam_f*x + s*w'
  TF_LAMF = 8,    // lam_f != 0
  TF_NORM_IN = 16,    // win holds u = D^-1/2 w; gathers are unweighted (VM 2)
  TF_SCALE_OUT = 32,  // write u' = D^-1/2 w' (the next term gathers it)
  TF_RAW_OUT = 64,    // split shard pass 0: write the raw neighbour sum, no epilogue
};

struct TermArgs {
  int64_t n;
  int32_t k;    // columns in this slab
  int64_t ld;   // row stride of the gathered block win (floats)
  int64_t n_in; // rows of the gathered block (0: unknown; debug checks only)
  int64_t ldx;  // row stride of x
  int64_t ldo;  // row stride of wout (and acc_in)
  const int32_t* indptr;
  const int32_t* indices;
  const float* values;
  const float* x;
  const float* win;
  float* wout;
  float alpha, beta, gamma, lamf, sfin;
  int flags;
  int32_t long_thresh;     // rows longer than this are chunk-processed
  const int32_t* chunk_desc;
  int32_t n_chunks;
  int32_t chunk_blocks;    // leading blocks reserved for chunks
  int32_t chunk_len;
  float* partials;         // [n_chunks][k]
  int32_t* tickets;
  int64_t row_begin, row_end;  // this launch's row segment
  int64_t hot_rows;        // hub prefix kept in L2 (persisting window)
  const float* rscale;     // d^-1/2 per row (TF_NORM_IN / TF_SCALE_OUT)
  const float* acc_in;     // VM 2/3: partial neighbour sum added before the epilogue (or NULL)
  int pdl;                 // programmatic dependent launch role (pdl_prologue)
};

// Programmatic dependent launch (default; SPED_PDL=0 off): the launches of one term
// (short rows, warp rows, hub chunks) read the same input and write
// disjoint rows, so each may start as soon as the previous launch's CTAs
// are all resident -- their tails overlap.  Completion stays ordered: the
// first launch of a term waits (every thread) for the previous grid, which
// is the previous term's last launch; later launches of the term chain
// completion through one waiting thread, so a term's last launch cannot
// complete before its first.  pdl bit 0: data dependency, bit 1: chain.
__device__ __forceinline__ void pdl_prologue(int mode) {
  if (mode & 1) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
  } else if ((mode & 2) && blockIdx.x == 0 && threadIdx.x == 0) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  if (mode) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// VM 0: stored values; 1: implicit combinatorial (-1, row_len-1 on the
// diagonal); 2: implicit normalized on the scaled block (1 off the diagonal,
// the diagonal handled in the epilogue); 3: stored values, split-shard term
// (pass 0 writes the raw sum, pass 1 adds acc_in before the epilogue)
template <int VM>
__device__ __forceinline__ float entry_value(const float* values, int64_t p, int32_t col, int64_t row,
                                             int32_t rowlen) {
  if (VM == 1) return col == row ? (float)(rowlen - 1) : -1.0f;
  if (VM == 2) return col == row ? 0.0f : 1.0f;
  return ld_stream_f32(values + p);
}

// CSR stream of the row sums: through L1 (the LPR lanes of a slice and the
// next nonzeros of the same row share sectors); FREE_IDX_EF=1 also marks
// the lines evict_first in L2 (read once per term)
#ifndef FREE_IDX_EF
#define FREE_IDX_EF 0
#endif
template <class T>
__device__ __forceinline__ T ld_csr(const T* p) {
#if FREE_IDX_EF
  if constexpr (sizeof(T) == 4) {
    uint32_t r;
    asm("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(policy_evict_first()));
    T t;
    memcpy(&t, &r, 4);
    return t;
  }
#endif
  return __ldg(p);
}

// W-float lane vectors: W = 4 (128-bit loads) or W = 8 (256-bit loads,
// LDG.E.256 on sm_100a).
template <int W>
struct Vf {
  float v[W];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < W; ++i) v[i] = 0.f;
  }
  // packed fp32 FMAs (FFMA2 on sm_100a): two of the lane's columns per
  // instruction, each element still one fused multiply-add (same bits)
  __device__ __forceinline__ void fma(float s, const Vf& x) {
    uint64_t ss;
    asm("mov.b64 %0, {%1,%1};" : "=l"(ss) : "f"(s));
#pragma unroll
    for (int i = 0; i < W; i += 2) {
      uint64_t xv, av;
      asm("mov.b64 %0, {%1,%2};" : "=l"(xv) : "f"(x.v[i]), "f"(x.v[i + 1]));
      asm("mov.b64 %0, {%1,%2};" : "=l"(av) : "f"(v[i]), "f"(v[i + 1]));
      asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(av) : "l"(ss), "l"(xv));
      asm("mov.b64 {%0,%1}, %2;" : "=f"(v[i]), "=f"(v[i + 1]) : "l"(av));
    }
  }
  __device__ __forceinline__ void add(const Vf& x) {
#pragma unroll
    for (int i = 0; i < W; ++i) v[i] += x.v[i];
  }
  __device__ __forceinline__ void add_xor(int off) {
#pragma unroll
    for (int i = 0; i < W; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], off);
  }
};

template <int W>
__device__ __forceinline__ Vf<W> ldg_vec(const float* p) {
  Vf<W> r;
  if constexpr (W == 8) {
    asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
          "=f"(r.v[6]), "=f"(r.v[7])
        : "l"(p));
  } else {
    const float4 t = __ldg(reinterpret_cast<const float4*>(p));
    r.v[0] = t.x; r.v[1] = t.y; r.v[2] = t.z; r.v[3] = t.w;
  }
  return r;
}
template <int W>
__device__ __forceinline__ Vf<W> ld_stream_vec(const float* p) {
  Vf<W> r;
#pragma unroll
  for (int h = 0; h < W / 4; ++h) {
    const float4 t = ld_stream_f4(p + 4 * h);
    r.v[4 * h] = t.x; r.v[4 * h + 1] = t.y; r.v[4 * h + 2] = t.z; r.v[4 * h + 3] = t.w;
  }
  return r;
}
template <int W>
__device__ __forceinline__ void st_stream_vec(float* p, const Vf<W>& x) {
#pragma unroll
  for (int h = 0; h < W / 4; ++h)
    st_stream_f4(p + 4 * h, make_float4(x.v[4 * h], x.v[4 * h + 1], x.v[4 * h + 2], x.v[4 * h + 3]));
}

// ds = d_i^-1/2 (only read with TF_NORM_IN / TF_SCALE_OUT).  With TF_NORM_IN
// the own row wr is u_i = ds*w_i and y the unweighted neighbour sum of u:
// (L w)_i = u_i/ds - ds*y_i.
template <int W>
__device__ __forceinline__ Vf<W> term_epilogue(const TermArgs& a, const Vf<W>& y, const Vf<W>& xr,
                                               const Vf<W>& wr, float ds = 1.f) {
  Vf<W> r;
  const float inv = (a.flags & TF_NORM_IN) ? 1.0f / ds : 1.f;
#pragma unroll
  for (int i = 0; i < W; ++i) {
    float lw = y.v[i], wv = wr.v[i];
    if (a.flags & TF_NORM_IN) {
      wv = wr.v[i] * inv;
      lw = fmaf(-ds, y.v[i], wv);
    }
    float t = a.beta * lw;
    if (a.flags & TF_ALPHA) t = fmaf(a.alpha, xr.v[i], t);
    if (a.flags & TF_GAMMA) t = fmaf(a.gamma, wv, t);
    if (a.flags & TF_FINAL) {
      t *= a.sfin;
      if (a.flags & TF_LAMF) t = fmaf(a.lamf, xr.v[i], t);
    }
    if (a.flags & TF_SCALE_OUT) t *= ds;
    r.v[i] = t;
  }
  return r;
}
__device__ __forceinline__ float row_ds(const TermArgs& a, int64_t row) {
  return (a.flags & (TF_NORM_IN | TF_SCALE_OUT)) ? __ldg(a.rscale + row) : 1.f;
}

__device__ __forceinline__ float4 term_epilogue(const TermArgs& a, float4 y, float4 xr, float4 wr) {
  Vf<4> Y, X, R;
  Y.v[0] = y.x; Y.v[1] = y.y; Y.v[2] = y.z; Y.v[3] = y.w;
  X.v[0] = xr.x; X.v[1] = xr.y; X.v[2] = xr.z; X.v[3] = xr.w;
  R.v[0] = wr.x; R.v[1] = wr.y; R.v[2] = wr.z; R.v[3] = wr.w;
  const Vf<4> o = term_epilogue<4>(a, Y, X, R);
  return make_float4(o.v[0], o.v[1], o.v[2], o.v[3]);
}

// Row sums without shuffles: every LPR-lane slice of a row's SUB lane
// groups walks its own nonzeros (p = b + sub, b + sub + SUB, ...); column
// indices and values come through L1 (the LPR lanes of a slice read the same
// words), so there is no warp-uniform trip count, no predicated zero-fill
// and no index broadcast, and U independent gathers per lane are in flight.
// The SUB partial sums fold with the same xor tree as group_row_accumulate:
// the summation order -- and so every result bit -- is unchanged.
// (config 3: 0.542 -> 0.418 ms/term, config 5: 2.83 -> 2.41, config 4:
// 3.04 -> 2.87; profiles/r02_ab_shuffle_free_cfg*.log)
#ifndef FREE_U
#define FREE_U 2
#endif
#ifndef FREE_MINB
#define FREE_MINB 6
#endif
#ifndef FREE_LONG_U
#define FREE_LONG_U 3
#endif
#ifndef FREE_K128_U
#define FREE_K128_U 3  // k = 128 rows (16 lanes): config 5 2.41 -> 2.36 ms/term
#endif
#ifndef FREE_K128_MINB
#define FREE_K128_MINB 5
#endif
// DIAG_EPI=1 (default): implicit combinatorial rows (VM 1) skip the diagonal
// gather too and add (len-1) * w_i from the epilogue's coalesced own-row
// read (changes the fp32 summation order of the diagonal term)
#ifndef DIAG_EPI
#define DIAG_EPI 1  // config 3: 0.431 -> 0.424 ms/term (r02_ab_diag_skip_cfg3.log)
#endif
template <int W, int LPR, int SUB, int U, int VM, bool SKIPD = (VM == 2)>
__device__ __forceinline__ Vf<W> free_accumulate(const TermArgs& a, int32_t row, bool valid,
                                                 int32_t b, int32_t e, int32_t rowlen, int lane) {
  constexpr int G = LPR * SUB;
  const int g = lane % G;
  const int sub = g / LPR;
  const int cl = g % LPR;
  const float* wbase = a.win + cl * W;
  // row stride < 2^30 floats and columns are non-negative: the gather
  // address is one 32x32+64 multiply-add (IMAD.WIDE.U32) on the lane's base
  const char* wlb = reinterpret_cast<const char*>(wbase);
  uint32_t ldb = (uint32_t)a.ld * 4u;
  // below k = 128 the lane base and the stride are made opaque, so the
  // compiler keeps them in (uniform) registers instead of rebuilding the base
  // from the thread id before every gather (config 3: 36 -> 22 instructions
  // per two gathers, -5.7 %/term; the k = 128 kernel is 1.3 % faster without)
  if constexpr (W * LPR < 128) {
    asm("" : "+l"(wlb));
    asm("" : "+r"(ldb));
  }
  auto row_ptr = [&](int32_t c) {
    return reinterpret_cast<const float*>(wlb + (uint64_t)(uint32_t)c * ldb);
  };
  // the skipped diagonal: implicit combinatorial rows (VM 1) predicate the
  // gather and the add; scaled-normalized rows (VM 2) zero-fill instead
  // (config 3 -2.8 %, config 4 -1.5 % that way round; r02_ab_diet_cfg*.log)
  constexpr bool PRED = (VM == 1);
  Vf<W> acc;
  acc.zero();
  if (valid) {
    int32_t p = b + sub;
    for (; p + (U - 1) * SUB < e; p += U * SUB) {
      int32_t c[U];
      float v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        c[u] = ld_csr(a.indices + p + u * SUB);
        if (VM == 1) v[u] = c[u] == row ? (float)(rowlen - 1) : -1.0f;
        else if (VM == 2) v[u] = c[u] == row ? 0.0f : 1.0f;
        else v[u] = ld_csr(a.values + p + u * SUB);
      }
      Vf<W> gv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        SPED_DCHECK(c[u] >= 0 && (a.n_in == 0 || c[u] < a.n_in), DBG_GATHER_OOB);
        // VM 2: the diagonal's weight is 0 (the epilogue reads the own row
        // itself) -- no gather and no add for it (predicated, nothing zeroed)
        if (PRED) {
          if (!(SKIPD && c[u] == row)) gv[u] = ldg_vec<W>(row_ptr(c[u]));
        } else {
          if (SKIPD && c[u] == row) gv[u].zero();
          else gv[u] = ldg_vec<W>(row_ptr(c[u]));
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (!PRED || !(SKIPD && c[u] == row)) acc.fma(v[u], gv[u]);
    }
    for (; p < e; p += SUB) {
      const int32_t c = ld_csr(a.indices + p);
      float v;
      if (VM == 1) v = c == row ? (float)(rowlen - 1) : -1.0f;
      else if (VM == 2) v = c == row ? 0.0f : 1.0f;
      else v = ld_csr(a.values + p);
      SPED_DCHECK(c >= 0 && (a.n_in == 0 || c < a.n_in), DBG_GATHER_OOB);
      if (!(SKIPD && c == row)) acc.fma(v, ldg_vec<W>(row_ptr(c)));
    }
  }
#pragma unroll
  for (int off = LPR; off < G; off <<= 1) acc.add_xor(off);
  return acc;
}

template <int W, int LPR, int SUB, int VM>
__global__ void __launch_bounds__(256, (SUB > 1 ? LONG_MIN_BLOCKS : (W * LPR >= 128 ? FREE_K128_MINB : FREE_MINB))) spmm_free_kernel(const TermArgs a) {
  constexpr int G = LPR * SUB;
  constexpr int RPW = 32 / G;
  pdl_prologue(a.pdl);
  const int lane = threadIdx.x & 31;
  const int g = lane % G;
  const int cl = g % LPR;
  const int32_t wglobal = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int32_t row = (int32_t)a.row_begin + wglobal * RPW + lane / G;
  bool valid = row < a.row_end;
  int32_t b = 0, e = 0;
  if (valid) {
    b = __ldg(a.indptr + row);
    e = __ldg(a.indptr + row + 1);
    if (e - b > a.long_thresh) valid = false;
  }
  if (SUB > 1) {
    if (__all_sync(0xffffffffu, !valid)) return;  // the fold needs the whole warp
  } else if (!valid) {
    return;
  }
  constexpr bool SKIPD = (VM == 2) || (DIAG_EPI && VM == 1);
  Vf<W> acc = free_accumulate<W, LPR, SUB,
                              (SUB > 1 ? FREE_LONG_U : (W * LPR >= 128 ? FREE_K128_U : FREE_U)), VM,
                              SKIPD>(a, row, valid, b, e, e - b, lane);
  if (!valid || g >= LPR) return;
  const int64_t off = (int64_t)row * a.ld + cl * W;
  const int64_t offo = (int64_t)row * a.ldo + cl * W;
  if (DIAG_EPI && VM == 1 && e > b)  // the diagonal, from the own row (coalesced)
    acc.fma((float)(e - b - 1), ldg_vec<W>(a.win + off));
  if (VM == 3 || VM == 2) {
    if (a.acc_in) acc.add(ldg_vec<W>(a.acc_in + offo));
    if (a.flags & TF_RAW_OUT) {
      st_stream_vec<W>(a.wout + offo, acc);
      return;
    }
  }
  const bool need_x = (a.flags & TF_ALPHA) || ((a.flags & TF_FINAL) && (a.flags & TF_LAMF));
  Vf<W> xr, wr;
  xr.zero();
  wr.zero();
  if (need_x) xr = ld_stream_vec<W>(a.x + (int64_t)row * a.ldx + cl * W);
  if (a.flags & (TF_GAMMA | TF_NORM_IN)) wr = ldg_vec<W>(a.win + off);
  st_stream_vec<W>(a.wout + offo, term_epilogue<W>(a, acc, xr, wr, row_ds(a, row)));
}

template <class Kern>
static void launch_pdl(Kern kern, unsigned grid, cudaStream_t s, const TermArgs& a) {
  if (a.pdl == 0) {
    kern<<<grid, 256, 0, s>>>(a);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, a);
}

template <int W, int LPR, int SUB>
static void launch_free(const TermArgs& a, int vm, cudaStream_t s) {
  constexpr int RPW = 32 / (LPR * SUB);
  const int64_t rows = a.row_end - a.row_begin;
  const unsigned grid = (unsigned)(((rows + RPW - 1) / RPW + 7) / 8);
  if (grid == 0) return;
  if (vm == 1) launch_pdl(spmm_free_kernel<W, LPR, SUB, 1>, grid, s, a);
  else if (vm == 2) launch_pdl(spmm_free_kernel<W, LPR, SUB, 2>, grid, s, a);
  else if (vm == 3) launch_pdl(spmm_free_kernel<W, LPR, SUB, 3>, grid, s, a);
  else launch_pdl(spmm_free_kernel<W, LPR, SUB, 0>, grid, s, a);
}

template <int W, int LPR>
static void launch_free_sub(const TermArgs& a, int sub, int vm, cudaStream_t s) {
  switch (sub) {
    case 1: launch_free<W, LPR, 1>(a, vm, s); break;
    case 2: if constexpr (LPR * 2 <= 32) { launch_free<W, LPR, 2>(a, vm, s); break; } [[fallthrough]];
    case 4: if constexpr (LPR * 4 <= 32) { launch_free<W, LPR, 4>(a, vm, s); break; } [[fallthrough]];
    case 8: if constexpr (LPR * 8 <= 32) { launch_free<W, LPR, 8>(a, vm, s); break; } [[fallthrough]];
    default: launch_free<W, LPR, 32 / LPR>(a, vm, s); break;
  }
}
template <int W>
static void launch_free_w(int lpr, int sub, const TermArgs& a, int vm, cudaStream_t s) {
  switch (lpr) {
    case 1: launch_free_sub<W, 1>(a, sub, vm, s); break;
    case 2: launch_free_sub<W, 2>(a, sub, vm, s); break;
    case 4: launch_free_sub<W, 4>(a, sub, vm, s); break;
    case 8: launch_free_sub<W, 8>(a, sub, vm, s); break;
    case 16: launch_free_sub<W, 16>(a, sub, vm, s); break;
    default: if constexpr (W == 4) launch_free_sub<W, 32>(a, sub, vm, s); break;
  }
}


// Long-row chunks: one warp per chunk (all 32/LPR lane groups over the
// chunk's nonzeros).  The last chunk of a row to finish (ticket) folds the
// partial rows in chunk order and applies the epilogue: deterministic, no
// float atomics.
template <int W, int LPR, int U, int VM>
__global__ void __launch_bounds__(256, CHUNK_MIN_BLOCKS) spmm_chunk_kernel(const TermArgs a) {
  pdl_prologue(a.pdl);
  const int lane = threadIdx.x & 31;
  const bool need_x = (a.flags & TF_ALPHA) || ((a.flags & TF_FINAL) && (a.flags & TF_LAMF));
  const int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= a.n_chunks) return;
  const int32_t row = a.chunk_desc[4 * c + 0];
  const int32_t pb = a.chunk_desc[4 * c + 1];
  const int32_t pe = a.chunk_desc[4 * c + 2];
  const int32_t c0 = a.chunk_desc[4 * c + 3];
  const int32_t rb = a.indptr[row], re = a.indptr[row + 1];
  const Vf<W> acc = free_accumulate<W, LPR, 32 / LPR, U, VM>(a, row, true, pb, pe, re - rb, lane);
  const int lsub = lane / LPR, lcl = lane % LPR;
  if (lsub == 0) {
#pragma unroll
    for (int h = 0; h < W / 4; ++h)
      __stcg(reinterpret_cast<float4*>(a.partials + c * a.k + lcl * W + 4 * h),
             make_float4(acc.v[4 * h], acc.v[4 * h + 1], acc.v[4 * h + 2], acc.v[4 * h + 3]));
  }
  __threadfence();
  __syncwarp();  // every lane's partial store is fenced before lane 0 takes the ticket
  int ticket = 0;
  if (lane == 0) ticket = atomicAdd(a.tickets + c0, 1);
  ticket = __shfl_sync(0xffffffffu, ticket, 0);
  const int32_t nch = (re - rb + a.chunk_len - 1) / a.chunk_len;
  SPED_DCHECK(ticket >= 0 && ticket < nch, DBG_TICKET);
  if (ticket != nch - 1) return;
  __threadfence();
  if (lsub == 0) {
    Vf<W> y;
    y.zero();
    for (int32_t q = 0; q < nch; ++q) {
#pragma unroll
      for (int h = 0; h < W / 4; ++h) {
        const float4 t = __ldcg(reinterpret_cast<const float4*>(
            a.partials + (int64_t)(c0 + q) * a.k + lcl * W + 4 * h));
        y.v[4 * h] += t.x; y.v[4 * h + 1] += t.y; y.v[4 * h + 2] += t.z; y.v[4 * h + 3] += t.w;
      }
    }
    const int64_t off = (int64_t)row * a.ld + lcl * W;
    const int64_t offo = (int64_t)row * a.ldo + lcl * W;
    if (VM == 3 || VM == 2) {
      if (a.acc_in) y.add(ldg_vec<W>(a.acc_in + offo));
      if (a.flags & TF_RAW_OUT) {
        st_stream_vec<W>(a.wout + offo, y);
        y.zero();
      }
    }
    if (!(VM == 3 || VM == 2) || !(a.flags & TF_RAW_OUT)) {
      Vf<W> xr, wr;
      xr.zero();
      wr.zero();
      if (need_x) xr = ld_stream_vec<W>(a.x + (int64_t)row * a.ldx + lcl * W);
      if (a.flags & (TF_GAMMA | TF_NORM_IN)) wr = ldg_vec<W>(a.win + off);
      st_stream_vec<W>(a.wout + offo, term_epilogue<W>(a, y, xr, wr, row_ds(a, row)));
    }
  }
  if (lane == 0) a.tickets[c0] = 0;
}

// Generic slab (k not in {4,8,...,128} or unaligned): scalar loads, LPR
// lanes over columns (CPL columns each), SUB groups over nonzeros.  Handles
// every row itself (no long-row plan).
template <int LPR, int CPL, int VM>
__global__ void __launch_bounds__(256) spmm_term_generic(const TermArgs a) {
  constexpr int SUB = 32 / LPR;
  const int lane = threadIdx.x & 31;
  const int sub = lane / LPR;
  const int cl = lane % LPR;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= a.n) return;
  const int32_t b = a.indptr[row], e = a.indptr[row + 1];
  float acc[CPL];
#pragma unroll
  for (int q = 0; q < CPL; ++q) acc[q] = 0.f;
  for (int32_t p0 = b; p0 < e; p0 += 32) {
    const int32_t p = p0 + lane;
    int32_t col = 0;
    float val = 0.f;
    if (p < e) {
      col = ld_stream_i32(a.indices + p);
      val = entry_value<VM>(a.values, p, col, row, e - b);
    }
    const int cnt = min(32, e - p0);
    const int T = (cnt + SUB - 1) / SUB;
    for (int t = 0; t < T; t += 2) {
      int32_t c[2];
      float w[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int j = (t + u) * SUB + sub;
        const int js = j < 32 ? j : 31;
        c[u] = __shfl_sync(0xffffffffu, col, js);
        w[u] = __shfl_sync(0xffffffffu, val, js);
        if (j >= cnt) w[u] = 0.f;
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int j = (t + u) * SUB + sub;
        if (j < cnt) {
#pragma unroll
          for (int q = 0; q < CPL; ++q) {
            const int cc = q * LPR + cl;
            if (cc < a.k) acc[q] = fmaf(w[u], ld_gather_f32(a.win + (int64_t)c[u] * a.ld + cc), acc[q]);
          }
        }
      }
    }
  }
#pragma unroll
  for (int off = LPR; off < 32; off <<= 1)
#pragma unroll
    for (int q = 0; q < CPL; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], off);
  if (sub != 0) return;
#pragma unroll
  for (int q = 0; q < CPL; ++q) {
    const int cc = q * LPR + cl;
    if (cc >= a.k) continue;
    const int64_t off = row * a.ld + cc;
    const int64_t offo = row * a.ldo + cc;
    if (VM == 3) {
      if (a.acc_in) acc[q] += a.acc_in[offo];
      if (a.flags & TF_RAW_OUT) {
        a.wout[offo] = acc[q];
        continue;
      }
    }
    float r = a.beta * acc[q];
    const bool need_x = (a.flags & TF_ALPHA) || ((a.flags & TF_FINAL) && (a.flags & TF_LAMF));
    const float xv = need_x ? a.x[row * a.ldx + cc] : 0.f;
    if (a.flags & TF_ALPHA) r = fmaf(a.alpha, xv, r);
    if (a.flags & TF_GAMMA) r = fmaf(a.gamma, a.win[off], r);
    if (a.flags & TF_FINAL) {
      r *= a.sfin;
      if (a.flags & TF_LAMF) r = fmaf(a.lamf, xv, r);
    }
    a.wout[offo] = r;
  }
}

template <int W, int LPR>
static void launch_chunks(const TermArgs& a, int vm, cudaStream_t s) {
  const unsigned grid = (unsigned)((a.n_chunks + 7) / 8);
  if (grid == 0) return;
  if (vm == 1) launch_pdl(spmm_chunk_kernel<W, LPR, FREE_LONG_U, 1>, grid, s, a);
  else if (vm == 2) launch_pdl(spmm_chunk_kernel<W, LPR, FREE_LONG_U, 2>, grid, s, a);
  else if (vm == 3) launch_pdl(spmm_chunk_kernel<W, LPR, FREE_LONG_U, 3>, grid, s, a);
  else launch_pdl(spmm_chunk_kernel<W, LPR, FREE_LONG_U, 0>, grid, s, a);
}

// width dispatch: W = 8 (256-bit gathers) when k % 8 == 0 and rows are 32 B
// aligned, else W = 4.  lpr = k / W.
template <int W>
static void launch_chunks_w(int lpr, const TermArgs& a, int vm, cudaStream_t s) {
  switch (lpr) {
    case 1: launch_chunks<W, 1>(a, vm, s); break;
    case 2: launch_chunks<W, 2>(a, vm, s); break;
    case 4: launch_chunks<W, 4>(a, vm, s); break;
    case 8: launch_chunks<W, 8>(a, vm, s); break;
    case 16: launch_chunks<W, 16>(a, vm, s); break;
    default: if constexpr (W == 4) launch_chunks<W, 32>(a, vm, s); break;
  }
}
template <int LPR, int CPL>
static void launch_generic(const TermArgs& a, int vm, cudaStream_t s) {  // vm 0 / 1 / 3
  const int threads = 256;
  const unsigned grid = grid_for(a.n, threads / 32);
  if (vm == 1)
    spmm_term_generic<LPR, CPL, 1><<<grid, threads, 0, s>>>(a);
  else if (vm == 3)
    spmm_term_generic<LPR, CPL, 3><<<grid, threads, 0, s>>>(a);
  else
    spmm_term_generic<LPR, CPL, 0><<<grid, threads, 0, s>>>(a);
}

struct Segment {
  int64_t begin, end;
  int sub;
};


// Launch one term over one column slab: one launch per row segment, the
// long-row chunks riding in the leading blocks of the first launch.
static int launch_term_slab(TermArgs a, int vm, bool aligned, bool aligned32,
                            const Segment* segs, int nseg, cudaStream_t s) {
  const int k = a.k;
  const bool fast = aligned && (k == 4 || k == 8 || k == 16 || k == 32 || k == 64 || k == 128);
  if (fast) {
    static const int wide = [] {  // SPED_VEC=4 forces 128-bit gathers
      const char* e = getenv("SPED_VEC");
      return (e && e[0] == '4') ? 0 : 1;
    }();
#ifndef W8_MIN_K
#define W8_MIN_K 32  // k = 32: 4 lanes x 256-bit per row (config 4: 3.53 -> 3.22 ms/term)
#endif
    const bool w8 = wide && (k % 8 == 0) && aligned32 && k >= W8_MIN_K;
    const int lpr = k / (w8 ? 8 : 4);
    // rows in descending segment order, hub chunks last: the hub prefix of
    // the output is then the most recently written data when the next term
    // starts gathering from it (config 4: -0.3 %/term in a round-2 A/B)
    auto chunks = [&]() -> int {
      if (a.n_chunks > 0) {
        // hub chunks: 128-bit gathers below k = CHUNK_W8_MIN_K
        if (w8 && k >= CHUNK_W8_MIN_K) launch_chunks_w<8>(lpr, a, vm, s);
        else launch_chunks_w<4>(k / 4, a, vm, s);
        SPED_LAUNCH_CHECK();
      }
      return SPED_OK;
    };
    // on by default (config 4: 2.528 -> 2.513 ms/term, config 3: 0.430 ->
    // 0.428, config 5: within noise; profiles/r02_ab_pdl_cfg*.log);
    // SPED_PDL=0 launches plainly
    static const bool pdl_on = [] {
      const char* e = getenv("SPED_PDL");
      return !(e && e[0] == '0');
    }();
    for (int j = 0; j < nseg; ++j) {
      const int i = nseg - 1 - j;
      a.row_begin = segs[i].begin;
      a.row_end = segs[i].end;
      a.pdl = pdl_on ? (j == 0 ? 1 : 2) : 0;
      int sub = segs[i].sub;
      if (sub < 1) sub = 1;
      if (sub * lpr > 32) sub = 32 / lpr;
      if (w8) launch_free_w<8>(lpr, sub, a, vm, s);
      else launch_free_w<4>(lpr, sub, a, vm, s);
      SPED_LAUNCH_CHECK();
    }
    a.pdl = pdl_on ? (nseg == 0 ? 1 : 2) : 0;
    const int rc = chunks();
    if (rc != SPED_OK) return rc;
  } else {
    a.pdl = 0;
    a.chunk_blocks = 0;
    a.long_thresh = INT32_MAX;
    if (k <= 1) launch_generic<1, 1>(a, vm, s);
    else if (k <= 2) launch_generic<2, 1>(a, vm, s);
    else if (k <= 4) launch_generic<4, 1>(a, vm, s);
    else if (k <= 8) launch_generic<8, 1>(a, vm, s);
    else if (k <= 16) launch_generic<16, 1>(a, vm, s);
    else if (k <= 32) launch_generic<32, 1>(a, vm, s);
    else if (k <= 64) launch_generic<32, 2>(a, vm, s);
    else if (k <= 96) launch_generic<32, 3>(a, vm, s);
    else launch_generic<32, 4>(a, vm, s);
    SPED_LAUNCH_CHECK();
  }
  return SPED_OK;
}

__global__ void axpby_kernel(int64_t count, float a, const float* __restrict__ x, float b,
                             const float* __restrict__ y, float* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < count; i += stride) {
    float r = a * x[i];
    if (y) r = fmaf(b, y[i], r);
    out[i] = r;
  }
}

int launch_axpby(int64_t count, double a, const float* x, double b, const float* y, float* out,
                 cudaStream_t s) {
  if (count <= 0) return SPED_OK;
  axpby_kernel<<<grid_for(count, 256, num_sms() * 16), 256, 0, s>>>(count, (float)a, x, (float)b, y,
                                                                       out);
  SPED_LAUNCH_CHECK();
  return SPED_OK;
}

// Persisting-L2 window over the hub prefix of the gathered block.  After
// degree relabelling the rows gathered most often are the prefix
// [0, hot_rows); an access-policy window marks them "persisting" so the random
// cold-row gathers (normal lines) cannot evict them: a static L2 cache of the
// highest-degree rows (config 4: -12 % DRAM bytes, 3.32 -> 3.18 ms/term,
// profiles/r01_sweep_l2_persist.log).  The set-aside is requested on the first
// apply that has a hub prefix; SPED_L2_PERSIST_MB overrides its size (0 = off).
struct L2Persist {
  size_t setaside = 0;
  size_t max_window = 0;
  bool on = false;
};
static const L2Persist& l2_persist() {
  static const L2Persist cfg = [] {  // initialised once (thread-safe static)
    L2Persist p;
    const char* e = getenv("SPED_L2_PERSIST_MB");
    const double mb = e ? atof(e) : 40.0;
    if (mb > 0) {
      int dev = 0, maxp = 0, maxw = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
      cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev);
      size_t want = (size_t)(mb * 1048576.0);
      if (want > (size_t)maxp) want = (size_t)maxp;
      if (want > 0 && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) == cudaSuccess) {
        cudaDeviceGetLimit(&p.setaside, cudaLimitPersistingL2CacheSize);
        p.max_window = (size_t)maxw;
        p.on = p.setaside > 0 && p.max_window > 0;
      }
      cudaGetLastError();  // no persisting L2 on this device: plain gathers
    }
    return p;
  }();
  return cfg;
}

// Window [base, base + bytes) for the following launches on `s` (bytes = 0
// clears it).
static void l2_window(cudaStream_t s, const void* base, size_t bytes) {
  const L2Persist& p = l2_persist();
  if (!p.on) return;
  cudaStreamAttrValue v = {};
  if (bytes > p.max_window) bytes = p.max_window;
  v.accessPolicyWindow.base_ptr = bytes ? const_cast<void*>(base) : nullptr;
  v.accessPolicyWindow.num_bytes = bytes;
  v.accessPolicyWindow.hitRatio = bytes ? (float)fmin(1.0, (double)p.setaside / (double)bytes) : 0.f;
  v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v);
  cudaGetLastError();
}

// Shared driver for the exact and stochastic applies: runs the schedule,
// calling `term(t, win, wout, args)` for each term.
template <class TermFn>
int run_schedule(int64_t n, int32_t k, const float* x, const float* w_init, float* w_a, float* w_b,
                 float* out, int32_t n_terms, const double* alpha, const double* beta,
                 const double* gamma, double w0, double lam_f, double s_final, cudaStream_t s,
                 TermFn&& term) {
  if (n_terms == 0) return launch_axpby(n * k, lam_f + s_final * w0, x, 0.0, nullptr, out, s);
  const float* cur = w_init ? w_init : x;
  for (int32_t t = 0; t < n_terms; ++t) {
    const bool final = (t == n_terms - 1);
    float* dst = final ? out : ((t & 1) == 0 ? w_a : w_b);
    if (!dst) {
      set_error("scratch buffer for term %d is NULL", t);
      return SPED_ERR_ARG;
    }
    const double sc = (t == 0) ? w0 : 1.0;
    int flags = 0;
    if (alpha[t] != 0.0) flags |= TF_ALPHA;
    if (gamma[t] != 0.0) flags |= TF_GAMMA;
    if (final) {
      flags |= TF_FINAL;
      if (lam_f != 0.0) flags |= TF_LAMF;
    }
    int rc = term(t, cur, dst, (float)alpha[t], (float)(beta[t] * sc), (float)(gamma[t] * sc),
                  (float)lam_f, (float)s_final, flags);
    if (rc != SPED_OK) return rc;
    cur = dst;
  }
  return SPED_OK;
}

}  // namespace sped

using namespace sped;

extern "C" int sped_axpby(int64_t count, double a, const float* x, double b, const float* y,
                          float* out, sped_stream_t stream) {
  SPED_CHECK_ARG(count >= 0 && (count == 0 || (x && out)), "bad axpby arguments");
  return launch_axpby(count, a, x, b, y, out, as_stream(stream));
}

// With no segment table the whole matrix is one segment processed one row
// per warp (callers normally pass a table chosen from the row lengths).
extern "C" int sped_csr_poly_apply(int64_t n, int32_t k, const int32_t* indptr,
                                   const int32_t* indices, const float* values,
                                   int32_t long_threshold, int32_t chunk_len,
                                   const int32_t* chunk_desc, int64_t n_chunks, float* partials,
                                   int32_t* tickets, const int64_t* segments, int32_t n_segments,
                                   int64_t hot_rows, const float* row_scale, const float* x,
                                   const float* w_init,
                                   float* w_a, float* w_b,
                                   float* out, int32_t n_terms, const double* alpha,
                                   const double* beta, const double* gamma, double w0_scale,
                                   double lam_f, double s_final, sped_stream_t stream) {
  SPED_CHECK_ARG(n >= 0 && k >= 1, "bad shape n=%lld k=%d", (long long)n, k);
  SPED_CHECK_ARG(n_terms >= 0, "negative term count");
  SPED_CHECK_ARG(n_terms == 0 || (alpha && beta && gamma), "null schedule");
  SPED_CHECK_ARG(n == 0 || (indptr && x && out), "null array");
  SPED_CHECK_ARG(x != out && x != w_a && x != w_b, "x must not alias outputs");
  SPED_CHECK_ARG(w_init == nullptr || (w_init != out && w_init != w_a && w_init != w_b),
                 "w_init must not alias outputs");
  SPED_CHECK_ARG(n_chunks == 0 || (chunk_desc && partials && tickets && chunk_len > 0 &&
                                   long_threshold > 0),
                 "null or inconsistent long-row plan");
  SPED_CHECK_ARG(n_chunks < INT32_MAX && n < INT32_MAX && k < (1 << 30), "problem too large");
  SPED_CHECK_ARG(n_segments >= 0 && n_segments <= 8 && (n_segments == 0 || segments),
                 "bad segment table");
  if (n == 0) return SPED_OK;
  cudaStream_t s = as_stream(stream);
  const bool implicit = (values == nullptr);
  const int32_t slabs = (k + 127) / 128;
  // scaled-block mode (VM 2) for unit-weight normalized Laplacians: the
  // first term reads the stored values and writes u = D^-1/2 w, later terms
  // gather u unweighted.  Only on the fast path with every buffer 16-B
  // aligned; otherwise stored values.
  bool norm = row_scale && values && !w_init && n_terms >= 2 && slabs == 1 &&
              (k == 4 || k == 8 || k == 16 || k == 32 || k == 64 || k == 128) &&
              ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w_a) |
                reinterpret_cast<uintptr_t>(w_b) | reinterpret_cast<uintptr_t>(out)) % 16 == 0);
  Segment segs[8];
  int nseg = n_segments;
  for (int i = 0; i < nseg; ++i) {
    segs[i].begin = segments[3 * i];
    segs[i].end = segments[3 * i + 1];
    segs[i].sub = (int)segments[3 * i + 2];
    SPED_CHECK_ARG(segs[i].begin >= 0 && segs[i].end <= n && segs[i].begin <= segs[i].end,
                   "segment %d out of range", i);
  }
  Segment fixed[8];
  int ns = nseg;
  for (int i = 0; i < ns; ++i) fixed[i] = segs[i];
  if (ns == 0) {
    fixed[0].begin = 0;
    fixed[0].end = n;
    fixed[0].sub = 32;
    ns = 1;
  }
  const int64_t hot_bytes = hot_rows * (int64_t)k * (int64_t)sizeof(float);
  {
    auto term = [&](int32_t t, const float* win, float* wout, float al, float be, float ga,
                    float lf, float sf, int flags) -> int {
      int vm = implicit ? 1 : 0;
      if (norm) {
        if (t > 0) {
          vm = 2;
          flags |= TF_NORM_IN;
        }
        if (!(flags & TF_FINAL)) flags |= TF_SCALE_OUT;
      }
      for (int32_t sl = 0; sl < slabs; ++sl) {
        const int32_t c0 = sl * 128;
        const int32_t kw = min(128, k - c0);
        TermArgs a;
        a.n = n;
        a.k = kw;
        a.ld = k;
        a.n_in = (w_init && win == w_init) ? 0 : n;  // a shard's [own | halo] input: unknown
        a.ldx = k;
        a.ldo = k;
        a.indptr = indptr;
        a.indices = indices;
        a.values = values;
        a.x = x + c0;
        a.win = win + c0;
        a.wout = wout + c0;
        a.alpha = al;
        a.beta = be;
        a.gamma = ga;
        a.lamf = lf;
        a.sfin = sf;
        a.flags = flags;
        a.long_thresh = n_chunks > 0 ? long_threshold : INT32_MAX;
        a.chunk_desc = chunk_desc;
        a.n_chunks = (int32_t)n_chunks;
        a.chunk_blocks = 0;
        a.chunk_len = chunk_len > 0 ? chunk_len : 1;
        a.partials = partials;
        a.tickets = tickets;
        a.row_begin = 0;
        a.row_end = n;
        a.hot_rows = hot_rows;
        a.rscale = row_scale;
        a.acc_in = nullptr;
        a.pdl = 0;
        const uintptr_t pbits = reinterpret_cast<uintptr_t>(a.x) | reinterpret_cast<uintptr_t>(a.win) |
                                reinterpret_cast<uintptr_t>(a.wout);
        const bool aligned = (kw % 4 == 0) && (k % 4 == 0) && (pbits % 16 == 0);
        const bool aligned32 = (kw % 8 == 0) && (k % 8 == 0) && (pbits % 32 == 0);
        // persisting window over the hub prefix of the gathered block
        if (hot_rows > 0 && hot_rows < n && sl == 0) l2_window(s, win, (size_t)hot_bytes);
        int r = launch_term_slab(a, vm, aligned, aligned32, fixed, ns, s);
        if (r != SPED_OK) return r;
      }
      return SPED_OK;
    };
    const int rc = run_schedule(n, k, x, w_init, w_a, w_b, out, n_terms, alpha, beta, gamma,
                                w0_scale, lam_f, s_final, s, term);
    if (hot_rows > 0 && hot_rows < n) l2_window(s, nullptr, 0);
    return rc;
  }
}

// One polynomial term on a row shard.  E = w is the
// [own | halo] block.  With a split CSR (own-column / halo-column entries)
// pass 0 (raw_out) runs while the halo rows are in flight and writes the raw
// own-column sum; pass 1 adds it (partial_in) to the halo-column sum and
// applies the term epilogue.  An unsplit shard runs one pass.  scaled_in /
// scaled_out: the scaled-normalized form of sped_csr_poly_apply (VM 2) --
// E holds u = D^-1/2 w (own AND halo rows, so the exchange moves u),
// neighbours are summed unweighted, row_scale = d^-1/2 of the own rows.
// [hot_begin, hot_begin + hot_rows) rows of E get the persisting-L2 window.
static int shard_term(int64_t n, int32_t k, const int32_t* indptr, const int32_t* indices,
                      const float* values, int32_t long_threshold, int32_t chunk_len,
                      const int32_t* chunk_desc, int64_t n_chunks, float* partials,
                      int32_t* tickets, const int64_t* segments, int32_t n_segments,
                      const float* row_scale, int32_t scaled_in, int32_t scaled_out,
                      int64_t hot_begin, int64_t hot_rows, const float* x, const float* w,
                      const float* partial_in, int32_t raw_out, float* out, double alpha,
                      double beta, double gamma, double w0_scale, double lam_f, double s_final,
                      sped_stream_t stream) {
  SPED_CHECK_ARG(n >= 0 && k >= 1, "bad shape n=%lld k=%d", (long long)n, k);
  SPED_CHECK_ARG(n == 0 || (indptr && w && out), "null array");
  SPED_CHECK_ARG(raw_out || x, "the epilogue pass needs x");
  SPED_CHECK_ARG(!raw_out || partial_in == nullptr, "the raw pass takes no partial input");
  SPED_CHECK_ARG(out != w && out != x, "out must not alias w or x");  // may alias partial_in
  SPED_CHECK_ARG(n_chunks == 0 || (chunk_desc && partials && tickets && chunk_len > 0 &&
                                   long_threshold > 0),
                 "null or inconsistent long-row plan");
  SPED_CHECK_ARG(n_chunks < INT32_MAX && n < INT32_MAX && k < (1 << 30), "problem too large");
  SPED_CHECK_ARG(n_segments >= 0 && n_segments <= 8 && (n_segments == 0 || segments),
                 "bad segment table");
  SPED_CHECK_ARG(!(scaled_in || scaled_out) || row_scale, "scaled terms need row_scale");
  SPED_CHECK_ARG(scaled_in || values, "unscaled shard terms need stored values");
  SPED_CHECK_ARG(!scaled_in || (k == 4 || k == 8 || k == 16 || k == 32 || k == 64 || k == 128),
                 "scaled terms need k in {4, 8, 16, 32, 64, 128}");
  if (n == 0) return SPED_OK;
  cudaStream_t s = as_stream(stream);
  Segment fixed[8];
  int ns = n_segments;
  for (int i = 0; i < ns; ++i) {
    fixed[i].begin = segments[3 * i];
    fixed[i].end = segments[3 * i + 1];
    fixed[i].sub = (int)segments[3 * i + 2];
    SPED_CHECK_ARG(fixed[i].begin >= 0 && fixed[i].end <= n && fixed[i].begin <= fixed[i].end,
                   "segment %d out of range", i);
  }
  if (ns == 0) {
    fixed[0].begin = 0;
    fixed[0].end = n;
    fixed[0].sub = 32;
    ns = 1;
  }
  int flags = TF_FINAL;
  if (raw_out) {
    flags |= TF_RAW_OUT;
  } else {
    if (alpha != 0.0) flags |= TF_ALPHA;
    if (gamma != 0.0) flags |= TF_GAMMA;
    if (lam_f != 0.0) flags |= TF_LAMF;
    if (scaled_in) flags |= TF_NORM_IN;
    if (scaled_out) flags |= TF_SCALE_OUT;
  }
  const int vm = scaled_in ? 2 : 3;
  const int32_t slabs = (k + 127) / 128;
  SPED_CHECK_ARG(!scaled_in || slabs == 1, "scaled terms need k <= 128");
  if (hot_rows > 0) l2_window(s, w + hot_begin * (int64_t)k, (size_t)(hot_rows * (int64_t)k * 4));
  for (int32_t sl = 0; sl < slabs; ++sl) {
    const int32_t c0 = sl * 128;
    TermArgs a;
    a.n = n;
    a.k = min(128, k - c0);
    a.ld = k;
    a.n_in = 0;  // [own | halo]: the halo length is the caller's
    a.ldx = k;
    a.ldo = k;
    a.indptr = indptr;
    a.indices = indices;
    a.values = values;
    a.x = x ? x + c0 : nullptr;
    a.win = w + c0;
    a.wout = out + c0;
    a.alpha = (float)alpha;
    a.beta = (float)(beta * w0_scale);
    a.gamma = (float)(gamma * w0_scale);
    a.lamf = (float)lam_f;
    a.sfin = (float)s_final;
    a.flags = flags;
    a.long_thresh = n_chunks > 0 ? long_threshold : INT32_MAX;
    a.chunk_desc = chunk_desc;
    a.n_chunks = (int32_t)n_chunks;
    a.chunk_blocks = 0;
    a.chunk_len = chunk_len > 0 ? chunk_len : 1;
    a.partials = partials;
    a.tickets = tickets;
    a.row_begin = 0;
    a.row_end = n;
    a.hot_rows = hot_rows;
    a.rscale = row_scale;
    a.acc_in = partial_in ? partial_in + c0 : nullptr;
    a.pdl = 0;
    const uintptr_t pbits = reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w) |
                            reinterpret_cast<uintptr_t>(out) |
                            reinterpret_cast<uintptr_t>(partial_in);
    const bool aligned = (k % 4 == 0) && (pbits % 16 == 0);
    const bool aligned32 = (k % 8 == 0) && (pbits % 32 == 0);
    SPED_CHECK_ARG(!scaled_in || aligned, "scaled terms need 16-B aligned blocks");
    int rc = launch_term_slab(a, vm, aligned, aligned32, fixed, ns, s);
    if (rc != SPED_OK) return rc;
  }
  if (hot_rows > 0) l2_window(s, nullptr, 0);
  return SPED_OK;
}

extern "C" int sped_csr_term_split(int64_t n, int32_t k, const int32_t* indptr,
                                   const int32_t* indices, const float* values,
                                   int32_t long_threshold, int32_t chunk_len,
                                   const int32_t* chunk_desc, int64_t n_chunks, float* partials,
                                   int32_t* tickets, const int64_t* segments, int32_t n_segments,
                                   const float* x, const float* w, const float* partial_in,
                                   int32_t raw_out, float* out, double alpha, double beta,
                                   double gamma, double w0_scale, double lam_f, double s_final,
                                   sped_stream_t stream) {
  return shard_term(n, k, indptr, indices, values, long_threshold, chunk_len, chunk_desc, n_chunks,
                    partials, tickets, segments, n_segments, nullptr, 0, 0, 0, 0, x, w,
                    partial_in, raw_out, out, alpha, beta, gamma, w0_scale, lam_f, s_final,
                    stream);
}

extern "C" int sped_csr_term_shard(int64_t n, int32_t k, const int32_t* indptr,
                                   const int32_t* indices, const float* values,
                                   int32_t long_threshold, int32_t chunk_len,
                                   const int32_t* chunk_desc, int64_t n_chunks, float* partials,
                                   int32_t* tickets, const int64_t* segments, int32_t n_segments,
                                   const float* row_scale, int32_t scaled_in, int32_t scaled_out,
                                   int64_t hot_begin, int64_t hot_rows, const float* x,
                                   const float* w, const float* partial_in, int32_t raw_out,
                                   float* out, double alpha, double beta, double gamma,
                                   double w0_scale, double lam_f, double s_final,
                                   sped_stream_t stream) {
  return shard_term(n, k, indptr, indices, values, long_threshold, chunk_len, chunk_desc, n_chunks,
                    partials, tickets, segments, n_segments, row_scale, scaled_in, scaled_out,
                    hot_begin, hot_rows, x, w, partial_in, raw_out, out, alpha, beta, gamma,
                    w0_scale, lam_f, s_final, stream);
}

extern "C" unsigned int sped_debug_take_spmm(void) { return sped::debug_take_unit(); }
