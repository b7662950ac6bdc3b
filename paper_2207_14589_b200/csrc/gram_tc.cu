// K5 on the 5th-gen tensor cores: Gram of Z = [V | M] with tcgen05.mma
// kind::tf32 in 3xTF32 (hi*hi + hi*lo + lo*hi, fp32 accumulation in TMEM),
// for K2 = 2k in {64, 128, 256} (k = 32 / 64 / 128).
//
//   G = Z^T Z  (K2 x K2), contraction over the n rows.
//
// Operands come from ONE shared-memory tile per stage: the MMA's A = Z^T
// (M = K2 columns of Z) and B (N = K2 columns of Z) are both K-major (the
// n-row contraction is contiguous) and read the same canonical no-swizzle
// layout.  Per 8-row K step: 128-byte core matrices (8 columns x 4 rows),
// the two 4-row halves of a column group 144 B apart (LBO) and column groups
// 288 B apart (SBO), K steps padded by 32 B: the padding makes the
// transposing stores from registers bank-conflict free (32 consecutive rows
// of one column land in 32 different banks).  (MN-major tf32 operands read
// back as zeros on sm_100a in our probes, tools/probe/tc_probe.cu.)  Each thread loads
// float4s of V / M rows, splits them into tf32 hi/lo parts (cvt.rna.tf32)
// and stores both tiles; one elected thread issues the MMAs and commits them
// to the stage's mbarrier, which the loaders wait on before refilling it
// (double buffering).
//
// Precision: the tensor core accumulates in fp32 with a directed (toward
// zero) rounding per MMA, so the error grows with the number of MMAs folded
// into one accumulator (measured: ~8.5e-5 relative after 8192 rows).  K steps
// are therefore spread round-robin over NACC TMEM accumulators and every
// SPLIT rows the accumulators are drained (tcgen05.ld), summed and added in
// fp64 into the CTA's private fp64 partial Gram; the partials are summed in
// CTA order by the reduce kernel (deterministic).  Each fp32 accumulator then
// folds at most 3*SPLIT/(8*NACC) MMAs (96 at k=32).
//
// K2 = 256 is computed as two M=128 tiles over the upper triangle:
// rows 0..127 x cols 0..255 (TMEM cols 0..255) and rows 128..255 x cols
// 128..255 (TMEM cols 256..383).

#include "async_copy.cuh"
#include "sped_common.cuh"
#include "tcgen05.cuh"

namespace sped {
namespace tc {

using namespace ::sped::async;

constexpr int SBO_B = 272;   // column-group (8 MN) stride, bytes
constexpr int LBO_B = 128;   // second 4-row K half, bytes

template <int TC>  // TC = columns of the K-major tile
__device__ __forceinline__ int kmaj_offset2(int r, int c) {
  return (r >> 3) * ((TC / 8) * (SBO_B / 4)) + ((r >> 2) & 1) * (LBO_B / 4) + (c >> 3) * (SBO_B / 4) +
         (c & 7) * 4 + (r & 3);
}


// ---------------------------------------------------------------------------
// v2 (K2 = 64, 128): warp-specialised pipeline, nothing CTA-synchronous in
// the steady state.
//
//   warp 13     producer: lane 0 runs the cp.async.bulk ring (NR raw stages
//               of KC rows of V and of M), refilling a stage once raw_free
//   warps 0-7   convert: raw fp32 rows -> hi/lo tf32 K-major tiles (NTB
//               buffers); arrive raw_free / tile_full (mbarriers, count 256)
//   warp 8      MMA issuer: lane 0 waits tile_full, issues the tile's MMAs
//               into the current accumulator BANK, commits tile_free per
//               tile and bank_full per slice
//   warps 9-12  drain: wait bank_full, tcgen05.ld the bank's NACC
//               accumulators, fold them in fp64 into shared-memory row sums,
//               arrive bank_free.  Two banks: the MMAs of slice s+1 run while
//               slice s drains.
//
// Measured (n = 1e7, k = 32, B200): 0.70 ms = 3.7 TB/s of the 2.56 GB read
// (v1, one CTA-synchronous loop with three M=64 MMAs per K step: 1.95 ms).
// The copy ring alone streams at 6.1 TB/s; what remains is shared-memory
// bandwidth: per 64-row chunk the bulk copy (16 KB), the converters' reads
// (16 KB) and tile writes (32 KB) and the SS-mode MMA operand reads (8 x 8 KB)
// share the SM's 128 B/clk.
//
// Only the blocks the solvers read are kept: rows 0..k-1 of G (S and C) and
// the Q = M^T M block (rows and columns k..2k-1).  The CTA writes its fp64
// partial once at the end (rows 0..k-1, then Q).
#ifndef GRAM_BIG_SPLIT
#define GRAM_BIG_SPLIT 512
#endif
#ifndef GRAM_BIG_KC
#define GRAM_BIG_KC 16
#endif
#ifndef GRAM_BIG_NR
#define GRAM_BIG_NR 8   // with the coalesced drain: 8 raw stages x 2 tile buffers (mu-EG 0.914 -> 0.878 ms)
#endif
#ifndef GRAM_BIG_NTB
#define GRAM_BIG_NTB 2
#endif
template <int K2, bool DQ = false>
struct Cfg2 {
  // Y mode (K2 = 64): the tile is Y = [hi | lo] (128 columns) and ONE
  // M=128 x N=128 MMA per 8-row K step forms Y^T Y = [[HH, HL], [LH, LL]]:
  // all four 3xTF32 products (plus lo*lo) at the M=128 rate, where three
  // M=64 MMAs run at well under half of it (SS-mode M=64).  Otherwise (K2 =
  // 128) separate hi / lo tiles and three M=128 x N=128 MMAs.
  // BIG mode (K2 = 256): two MMA groups per K step -- rows 0..127 x cols
  // 0..255 (M=128, N=256: S and C) and rows 128..255 x cols 128..255 (N=128:
  // Q) -- 384 TMEM columns, so one accumulator bank, and the fp64 row sums
  // (128 x 384) live in the CTA's global partial (read-modify-write by the
  // owning drain thread) instead of shared memory.
  // DQ (diag-Q mode, mu-EG): only diag(Q) is needed, so the Q MMA group is
  // dropped and the converters sum the squares of the M values they convert
  // (fp64, fixed per-thread columns); 256 TMEM columns per bank then leave
  // room for two banks, so the drain of slice s overlaps the MMAs of s+1.
  static constexpr bool YM = (K2 == 64);
  static constexpr bool BIG = (K2 == 256);
  static constexpr bool BIGQ = BIG && !DQ;            // BIG with the Q MMA group
  static constexpr int NACC = BIG ? 1 : 2;            // accumulators per bank
  static constexpr int NBANK = BIGQ ? 1 : 2;
  static constexpr int ACC_COLS = YM ? 2 * K2 : (BIG ? (DQ ? 256 : 384) : K2);  // TMEM columns per accumulator
  static constexpr int SPLIT = (K2 == 64) ? 1024 : (BIG ? GRAM_BIG_SPLIT : 512);  // rows per slice (drain)
  static constexpr int KC = (K2 == 64) ? 64 : (BIG ? GRAM_BIG_KC : 32);  // rows per chunk
  static constexpr int NR = (K2 == 64) ? 4 : (BIG ? GRAM_BIG_NR : 3);     // raw (bulk copy) stages
  static constexpr int NTB = (K2 == 64) ? 3 : (BIG ? GRAM_BIG_NTB : 2);    // converted tile buffers
  static constexpr int RAW_FLOATS = KC * K2;
  static constexpr int TCOLS = YM ? 2 * K2 : K2;      // columns of one K-major tile
  static constexpr int KSTEP_FLOATS = (TCOLS / 8) * (SBO_B / 4);
  static constexpr int TILE_FLOATS = (KC / 8) * KSTEP_FLOATS;
  static constexpr int TBUF_FLOATS = YM ? TILE_FLOATS : 2 * TILE_FLOATS;  // per buffer
  static constexpr int CPS = SPLIT / KC;
  static constexpr int HALF = K2 / 2;                 // = k
  static constexpr int SUM_LD = K2 + 1;               // padded fp64 row stride (rows < k)
  static constexpr int QLD = HALF + 1;                // padded stride of the Q block
  static constexpr int SUM_BLOCK = HALF * SUM_LD + HALF * QLD;
  static constexpr int SUM_DOUBLES = BIG ? 0 : (YM ? 2 : 1) * SUM_BLOCK;  // Y: H rows + L rows
  static constexpr int SMEM = NR * RAW_FLOATS * 4 + NTB * TBUF_FLOATS * 4 + SUM_DOUBLES * 8 + 1024;
  static constexpr int NTHREADS = 14 * 32;
};


template <int K2, bool DQ>
__global__ void __launch_bounds__(Cfg2<K2, DQ>::NTHREADS, 1)
    gram_tc2_kernel(int64_t n, int32_t k, const float* __restrict__ V, const float* __restrict__ M,
                    double* __restrict__ partial, int64_t nslices) {
  using C = Cfg2<K2, DQ>;
  static_assert(!DQ || K2 == 256, "diag-Q mode is the k = 128 kernel");
  extern __shared__ __align__(1024) uint8_t smem[];
  float* raw = reinterpret_cast<float*>(smem);
  float* tiles = raw + C::NR * C::RAW_FLOATS;
  double* sums = reinterpret_cast<double*>(tiles + C::NTB * C::TBUF_FLOATS);
  __shared__ uint64_t full_bar[C::NR], raw_free[C::NR];
  __shared__ uint64_t tile_full[C::NTB], tile_free[C::NTB];
  __shared__ uint64_t bank_full[2], bank_free[2];
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_sh)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < C::NR; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&raw_free[i], 256);
    }
    for (int i = 0; i < C::NTB; ++i) {
      mbar_init(&tile_full[i], 256);
      mbar_init(&tile_free[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bank_full[i], 1);
      mbar_init(&bank_free[i], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int e = tid; e < C::SUM_DOUBLES; e += C::NTHREADS) sums[e] = 0.0;
  // fp64 partial of this CTA: rows 0..k-1 (K2 columns), then Q (k x k)
  double* out = partial + (int64_t)blockIdx.x * (C::HALF * K2 + C::HALF * C::HALF);
  if constexpr (C::BIG)
    for (int e = tid; e < C::HALF * K2 + C::HALF * C::HALF; e += C::NTHREADS) out[e] = 0.0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_sh;

  // this CTA's slices: blockIdx.x + j*gridDim.x; only the globally last slice
  // can be partial, and it is the last slice of its CTA
  const int64_t my_slices = (nslices - blockIdx.x + gridDim.x - 1) / gridDim.x;
  int64_t nq = 0;
  int last_chunks = C::CPS;
  if (my_slices > 0) {
    const int64_t last_sl = blockIdx.x + (my_slices - 1) * gridDim.x;
    const int64_t rows_last = min((int64_t)C::SPLIT, n - last_sl * C::SPLIT);
    last_chunks = (int)((rows_last + C::KC - 1) / C::KC);
    nq = (my_slices - 1) * C::CPS + last_chunks;
  }
  auto chunk_rows = [&](int64_t q, int64_t& r0) -> int {
    const int64_t sl = blockIdx.x + (q / C::CPS) * gridDim.x;
    r0 = sl * C::SPLIT + (q % C::CPS) * C::KC;
    const int64_t v = n - r0;
    return (int)(v > C::KC ? C::KC : v);
  };

  // DQ: sum of squares of this thread's M columns (fixed per thread: one
  // 4-row x 4-column block per chunk, (KC/4)*(K2/4) == 256 converter threads)
  double dq[4] = {0.0, 0.0, 0.0, 0.0};
  __shared__ double dq_s[DQ ? 4 * 128 : 1];
  if (warp < 8) {
    // ---------------- converters ----------------
    for (int64_t q = 0; q < nq; ++q) {
      const int rs = (int)(q % C::NR), ts = (int)(q % C::NTB);
      int64_t r0;
      const int valid = chunk_rows(q, r0);
      mbar_wait(&full_bar[rs], (uint32_t)((q / C::NR) & 1));
      if (q >= C::NTB) mbar_wait(&tile_free[ts], (uint32_t)(((q / C::NTB) - 1) & 1));
      float* hi = tiles + ts * C::TBUF_FLOATS;
      // Y mode: lo columns follow the hi columns in the same tile
      float* lo = C::YM ? hi + (K2 / 8) * (SBO_B / 4) : hi + C::TILE_FLOATS;
      const float* src = raw + rs * C::RAW_FLOATS;
      // one 4-row x 4-column block per thread: 4 LDS.128 of raw rows, a
      // register transpose, 4 STS.128 each of hi and lo (4 consecutive rows
      // of one column are contiguous in the K-major core matrix; 8 lanes of a
      // phase hit 8 distinct 16-B bank groups)
      for (int f = tid; f < (C::KC / 4) * (K2 / 4); f += 256) {
        const int rq = f / (K2 / 4), cq = f % (K2 / 4);
        const int c = cq * 4;
        const float* base = (c < C::HALF) ? (src + c) : (src + C::KC * C::HALF + (c - C::HALF));
        float4 z[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = rq * 4 + i;
          z[i] = (r < valid) ? *reinterpret_cast<const float4*>(base + r * C::HALF)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        const int off = kmaj_offset2<C::TCOLS>(rq * 4, c);
        if constexpr (DQ) {
          static_assert(!DQ || (C::KC / 4) * (K2 / 4) == 256, "one block per converter thread");
          if (c >= C::HALF) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              dq[0] += (double)z[i].x * (double)z[i].x;
              dq[1] += (double)z[i].y * (double)z[i].y;
              dq[2] += (double)z[i].z * (double)z[i].z;
              dq[3] += (double)z[i].w * (double)z[i].w;
            }
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float x0 = (&z[0].x)[j], x1 = (&z[1].x)[j], x2 = (&z[2].x)[j], x3 = (&z[3].x)[j];
          const float h0 = __uint_as_float(to_tf32(x0)), h1 = __uint_as_float(to_tf32(x1));
          const float h2 = __uint_as_float(to_tf32(x2)), h3 = __uint_as_float(to_tf32(x3));
          *reinterpret_cast<float4*>(hi + off + 4 * j) = make_float4(h0, h1, h2, h3);
          *reinterpret_cast<float4*>(lo + off + 4 * j) =
              make_float4(__uint_as_float(to_tf32(x0 - h0)), __uint_as_float(to_tf32(x1 - h1)),
                          __uint_as_float(to_tf32(x2 - h2)), __uint_as_float(to_tf32(x3 - h3)));
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&raw_free[rs]);
      mbar_arrive(&tile_full[ts]);
    }
  } else if (warp == 13) {
    // ---------------- producer: the cp.async.bulk ring ----------------
    if (lane == 0) {
      for (int64_t q = 0; q < nq; ++q) {
        const int rs = (int)(q % C::NR);
        if (q >= C::NR) mbar_wait(&raw_free[rs], (uint32_t)(((q / C::NR) - 1) & 1));
        int64_t r0;
        const int valid = chunk_rows(q, r0);
        float* dst = raw + rs * C::RAW_FLOATS;
        const uint32_t bytes = (uint32_t)valid * (uint32_t)C::HALF * 4u;
        mbar_expect_tx(&full_bar[rs], 2 * bytes);
        // BIG: read-once stream evict_first, so the fp64 partial rows the
        // drain read-modify-writes stay in L2 (they went to DRAM: +1.5 GB)
        if constexpr (C::BIG) {
          bulk_g2s_stream(dst, V + r0 * C::HALF, bytes, &full_bar[rs]);
          bulk_g2s_stream(dst + C::KC * C::HALF, M + r0 * C::HALF, bytes, &full_bar[rs]);
        } else {
          bulk_g2s(dst, V + r0 * C::HALF, bytes, &full_bar[rs]);
          bulk_g2s(dst + C::KC * C::HALF, M + r0 * C::HALF, bytes, &full_bar[rs]);
        }
      }
    }
    __syncwarp();
  } else if (warp == 8) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      constexpr uint32_t KSTEP_B = C::KSTEP_FLOATS * 4;
      constexpr uint32_t idesc = C::BIG ? instr_desc_tf32(128, 256)
                                        : instr_desc_tf32(C::YM ? 128 : K2, C::ACC_COLS);
      constexpr uint32_t idesc_q = instr_desc_tf32(128, 128);  // BIG: the Q block
      for (int64_t q = 0; q < nq; ++q) {
        const int ts = (int)(q % C::NTB);
        const int64_t s = q / C::CPS;
        const int ch = (int)(q % C::CPS);
        const int bank = (int)(s % C::NBANK);
        const bool slice_end = (ch == C::CPS - 1) || (q == nq - 1);
        if (ch == 0 && s >= C::NBANK)
          mbar_wait_sleep(&bank_free[bank], (uint32_t)(((s / C::NBANK) - 1) & 1));
        mbar_wait(&tile_full[ts], (uint32_t)((q / C::NTB) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const float* hi = tiles + ts * C::TBUF_FLOATS;
        const uint32_t hi_a = smem_u32(hi), lo_a = smem_u32(hi + C::TILE_FLOATS);
#pragma unroll
        for (int kb = 0; kb < C::KC / 8; ++kb) {
          const int gk = ch * (C::KC / 8) + kb;  // K step within the slice
          const uint32_t acc0 = (gk >= C::NACC) ? 1u : 0u;
          const uint32_t tacc = tmem + (uint32_t)((bank * C::NACC + gk % C::NACC) * C::ACC_COLS);
          const uint64_t dh = smem_desc(hi_a + kb * KSTEP_B, SBO_B, LBO_B);
          if constexpr (C::YM) {
            mma_tf32(tacc, dh, dh, idesc, acc0);  // [H|L]^T [H|L]
          } else if constexpr (C::BIG) {
            // rows 0..127 x cols 0..255, then rows/cols 128..255 (16 column groups on)
            const uint64_t dl = smem_desc(lo_a + kb * KSTEP_B, SBO_B, LBO_B);
            mma_tf32(tacc, dh, dh, idesc, acc0);
            mma_tf32(tacc, dh, dl, idesc, 1u);
            mma_tf32(tacc, dl, dh, idesc, 1u);
            if constexpr (DQ) continue;  // diag(Q) comes from the converters
            const uint32_t goff = 16u * SBO_B;
            const uint64_t qh = smem_desc(hi_a + goff + kb * KSTEP_B, SBO_B, LBO_B);
            const uint64_t ql = smem_desc(lo_a + goff + kb * KSTEP_B, SBO_B, LBO_B);
            mma_tf32(tacc + 256, qh, qh, idesc_q, acc0);
            mma_tf32(tacc + 256, qh, ql, idesc_q, 1u);
            mma_tf32(tacc + 256, ql, qh, idesc_q, 1u);
          } else {
            const uint64_t dl = smem_desc(lo_a + kb * KSTEP_B, SBO_B, LBO_B);
            mma_tf32(tacc, dh, dh, idesc, acc0);
            mma_tf32(tacc, dh, dl, idesc, 1u);
            mma_tf32(tacc, dl, dh, idesc, 1u);
          }
        }
        mma_commit(&tile_free[ts]);
        if (slice_end) mma_commit(&bank_full[bank]);
      }
    }
    __syncwarp();
  } else {
    // ---------------- drain (warps 9-12: TMEM lane quarter warp % 4) ----------
    const int quarter = warp & 3;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    // TMEM lane = accumulator row.  Y mode (M = 128): lanes 0-63 hold the H
    // rows (HH | HL), lanes 64-127 the L rows (LH | LL) of column m = lane % 64;
    // row m of G is the sum of both halves of both.  K2 = 128: lane m = row m.
    const int row = C::YM ? (quarter * 32 + lane) & (K2 - 1) : quarter * 32 + lane;
    double* sblk = sums + ((C::YM && quarter >= 2) ? C::SUM_BLOCK : 0);
    for (int64_t s = 0; s < my_slices; ++s) {
      const int bank = (int)(s % C::NBANK);
      mbar_wait_sleep(&bank_full[bank], (uint32_t)((s / C::NBANK) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int chunks = (s == my_slices - 1) ? last_chunks : C::CPS;
      const int nk = min(C::NACC, chunks * (C::KC / 8));
      if constexpr (C::BIG) {
        // TMEM lane m: row m of [S | C] (cols 0..255) and row m of Q (cols
        // 256..383; not in DQ mode); fp64 sums accumulate in the global
        // partial, stored COLUMN-major (element (m, c) at c*128 + m) so the
        // 32 lanes of a drain warp read-modify-write 256 contiguous bytes per
        // instruction instead of 32 separate lines
#pragma unroll 1
        for (int c0 = 0; c0 < C::ACC_COLS; c0 += 16) {
          float v[16];
          tmem_ld16(tmem + (uint32_t)(bank * C::ACC_COLS + c0) + lane_base, v);
          double* dst = (c0 < 256) ? out + (int64_t)c0 * C::HALF + row
                                   : out + C::HALF * K2 + (int64_t)(c0 - 256) * C::HALF + row;
          double cur[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) cur[i] = dst[i * C::HALF];
#pragma unroll
          for (int i = 0; i < 16; ++i) dst[i * C::HALF] = cur[i] + (double)v[i];
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        mbar_arrive(&bank_free[bank]);
        continue;
      }
#pragma unroll 1
      for (int c0 = 0; c0 < K2; c0 += 16) {
        double acc[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = 0.0;
        for (int a2 = 0; a2 < nk; ++a2) {
          const uint32_t tb = tmem + (uint32_t)((bank * C::NACC + a2) * C::ACC_COLS + c0) + lane_base;
          float v[16];
          tmem_ld16(tb, v);
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[i] += (double)v[i];
          if constexpr (C::YM) {
            tmem_ld16(tb + K2, v);  // the lo columns of the same row
#pragma unroll
            for (int i = 0; i < 16; ++i) acc[i] += (double)v[i];
          }
        }
        if (row < C::HALF) {
#pragma unroll
          for (int i = 0; i < 16; ++i) sblk[row * C::SUM_LD + c0 + i] += acc[i];
        } else if (c0 >= C::HALF) {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            sblk[C::HALF * C::SUM_LD + (row - C::HALF) * C::QLD + (c0 - C::HALF) + i] += acc[i];
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&bank_free[bank]);
    }
  }
  if constexpr (DQ) {
    if (tid < 256 && (tid % (K2 / 4)) * 4 >= C::HALF) {
      const int rq = tid / (K2 / 4), c = (tid % (K2 / 4)) * 4 - C::HALF;
#pragma unroll
      for (int j = 0; j < 4; ++j) dq_s[rq * 128 + c + j] = dq[j];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if constexpr (DQ) {  // diag(Q) of this CTA's rows, fixed summation order
    for (int e = tid; e < C::HALF; e += C::NTHREADS)
      out[C::HALF * K2 + e * C::HALF + e] =
          ((dq_s[e] + dq_s[128 + e]) + dq_s[256 + e]) + dq_s[384 + e];
  }
  if constexpr (!C::BIG)
  for (int e = tid; e < C::HALF * K2; e += C::NTHREADS) {
    const int i = (e / K2) * C::SUM_LD + (e % K2);
    out[e] = C::YM ? sums[i] + sums[C::SUM_BLOCK + i] : sums[i];
  }
  if constexpr (!C::BIG)
  for (int e = tid; e < C::HALF * C::HALF; e += C::NTHREADS) {
    const int i = C::HALF * C::SUM_LD + (e / C::HALF) * C::QLD + (e % C::HALF);
    out[C::HALF * K2 + e] = C::YM ? sums[i] + sums[C::SUM_BLOCK + i] : sums[i];
  }
  if (warp == 8) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// Sum the per-CTA partials (CTA order) into S / C / Q.  colmajor: the
// partial stores element (row i, col j) at j*k + i (the k = 128 drain).
__global__ void gram_tc2_reduce(int32_t k, int32_t nparts, const double* __restrict__ partial,
                                double* __restrict__ G, int colmajor) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int K2 = 2 * k, per = k * K2 + k * k;
  if (e >= per) return;
  double s = 0.0;
  for (int p = 0; p < nparts; ++p) s += partial[(int64_t)p * per + e];
  if (e < k * K2) {
    const int i = colmajor ? e % k : e / K2, j = colmajor ? e / k : e % K2;
    if (j < k)
      G[i * k + j] = s;  // S (full rows; symmetric by construction of the MMAs)
    else
      G[k * k + i * k + (j - k)] = s;  // C
  } else {
    const int q = e - k * K2;
    G[2 * k * k + (colmajor ? (q % k) * k + q / k : q)] = s;  // Q
  }
}

template <int K2, bool DQ = false>
int launch2(int64_t n, int32_t k, const float* V, const float* M, double* G, double* partial,
            cudaStream_t s) {
  using C = Cfg2<K2, DQ>;
  static PerDeviceOnce attr;
  const int rc = attr([]() -> int {
    SPED_CUDA(cudaFuncSetAttribute(gram_tc2_kernel<K2, DQ>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    return SPED_OK;
  });
  if (rc != SPED_OK) return rc;
  const int64_t nslices = (n + C::SPLIT - 1) / C::SPLIT;
  const unsigned grid = (unsigned)std::min<int64_t>(nslices, (int64_t)num_sms());
  gram_tc2_kernel<K2, DQ><<<grid, C::NTHREADS, C::SMEM, s>>>(n, k, V, M, partial, nslices);
  SPED_LAUNCH_CHECK();
  const int per = k * K2 + k * k;
  gram_tc2_reduce<<<(per + 255) / 256, 256, 0, s>>>(k, (int)grid, partial, G, C::BIG ? 1 : 0);
  SPED_LAUNCH_CHECK();
  return SPED_OK;
}

}  // namespace tc

bool gram_tc_supported(int32_t k, bool with_m) { return with_m && (k == 32 || k == 64 || k == 128); }

size_t gram_tc_workspace(int64_t n, int32_t k) {
  (void)n;
  const int K2 = 2 * k;
  return sizeof(double) * (size_t)num_sms() * 2 * K2 * K2 + 256;
}

int gram_tc(int64_t n, int32_t k, const float* V, const float* M, double* G, void* ws,
            cudaStream_t s, bool diag_q) {
  double* partial = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
  switch (k) {
    case 32: return tc::launch2<64>(n, k, V, M, G, partial, s);
    case 64: return tc::launch2<128>(n, k, V, M, G, partial, s);
    case 128:
      return diag_q ? tc::launch2<256, true>(n, k, V, M, G, partial, s)
                    : tc::launch2<256>(n, k, V, M, G, partial, s);
    default: set_error("gram_tc: unsupported k=%d", k); return SPED_ERR_UNSUPPORTED;
  }
}

}  // namespace sped
