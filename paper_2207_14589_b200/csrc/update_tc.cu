// K6 for k = 128 on the 5th-gen tensor cores: the mu-EG block update
//
//     V' = (P A + eta M) diag(s)          (mu_eg_step, solvers.py:121-144, in
//                                          the Gram form of SURVEY 8a)
//
// as a tall-skinny GEMM, P (n x 128) times the k x k coefficient matrix A,
// with tcgen05.mma kind::tf32 in 3xTF32 (Phi Ahi + Phi Alo + Plo Ahi, fp32
// accumulation in TMEM) and the normalisation fused into the epilogue.
//
// One persistent CTA per SM walks 128-row tiles:
//  * A is split into hi/lo tf32 once per CTA and kept in shared memory as the
//    K-major B operand (N = 128 output columns, K = 128): 136 KB;
//  * 8 converter warps read P rows straight from HBM (one row per lane, so the
//    16-B stores into the K-major core matrices are bank-conflict free; 8
//    lanes per 128-B row piece instead was slower, 1.04 vs 0.87 ms, on the
//    8-way store conflicts), split them into hi/lo tf32 and fill a 2-slot
//    ring of 32-column chunks (4 K steps, 34 KB per slot), with three chunks
//    of loads in flight;
//  * one thread issues 3 MMAs (M = 128, N = 128, K = 8) per K step into one
//    of two TMEM accumulators (128 columns each) and commits each chunk to
//    its slot's "free" barrier and each tile to the accumulator's "full"
//    barrier;
//  * 8 epilogue warps (TMEM lane quarter warp % 4, column half by warp / 4)
//    drain the accumulator of tile j while tile j+1 is multiplied:
//    out = (acc + eta M) * s.  TMEM hands each lane one row, so M tiles are
//    loaded coalesced (issued BEFORE the accumulator wait, overlapping the
//    MMAs) and transposed through a 2.5 KB per-warp staging buffer, and the
//    results go back through it to full-sector coalesced stores (row-per-lane
//    16-B stores ran at 2.6 TB/s: 1.16 ms vs 0.44 ms without stores).
// Bytes 12nk (read P, M; write V').  n = 2e6: 0.87 ms (3.5 TB/s; the SIMT
// kernel it replaces, block_update_k128, was FMA-issue bound at 1.44 ms).
// What limits it now is latency through the coupled stages: the 136 KB B
// operand leaves room for only a 2-chunk ring, so the converters stall on
// MMA completion, which waits on the epilogue (ncu: tensor pipe 20 %, DRAM
// 41 %, stalls on the ring / accumulator barriers).  Precision: 48 MMAs
// fold into one fp32 accumulator per tile (the Gram's drain analysis gives
// ~3e-8 relative per MMA), well inside the 1e-5 step tolerance.

#include <algorithm>

#include "async_copy.cuh"
#include "sped_common.cuh"
#include "tcgen05.cuh"

namespace sped {
namespace {

using namespace ::sped::async;
using namespace ::sped::tc;

#ifndef UPD_COAL
#define UPD_COAL 1  // coalesced converter loads: 0.881 -> 0.836 ms at n = 2e6 (r02_ab_update_tc128_transposed.log)
#endif
constexpr int UK = 128;                    // k
constexpr int UTM = 128;                   // rows per tile (MMA M)
constexpr int UKC = 32;                    // columns per chunk
constexpr int UNCH = UK / UKC;             // chunks per tile
constexpr int UNSLOT = 2;                  // chunk ring depth
constexpr int USBO = 272;                  // 8-row group stride, bytes (16-B pad: no bank conflicts)
constexpr int ULBO = 128;                  // second 4-column half of a K step, bytes
constexpr int UKSTEP_F = (UTM / 8) * (USBO / 4);   // floats per K step (128 rows x 8 columns)
constexpr int UCHUNK_F = (UKC / 8) * UKSTEP_F;     // floats per chunk (hi or lo)
constexpr int UB_F = (UK / 8) * UKSTEP_F;          // floats of the B operand (hi or lo)
constexpr int UTHREADS = 17 * 32;          // 8 converters, 8 epilogue, 1 MMA warp
constexpr int UMMA_WARP = 16;
constexpr int USTG_LD = 20;                // epilogue staging row stride (floats): conflict-free
constexpr int USTG_F = 32 * USTG_LD;       // per epilogue warp: 32 rows x 16 columns (+pad)
constexpr int USMEM = (2 * UB_F + UNSLOT * 2 * UCHUNK_F + 8 * USTG_F) * 4 + UK * 4;

// float offset of (row m, column kk) of a K-major tile (kk within the tile)
__device__ __forceinline__ int ukmaj(int m, int kk) {
  return (kk >> 3) * UKSTEP_F + ((kk >> 2) & 1) * (ULBO / 4) + (m >> 3) * (USBO / 4) + (m & 7) * 4;
}

__device__ __forceinline__ void split_store(float* hi, float* lo, int off, float4 x) {
  const float h0 = __uint_as_float(to_tf32(x.x)), h1 = __uint_as_float(to_tf32(x.y));
  const float h2 = __uint_as_float(to_tf32(x.z)), h3 = __uint_as_float(to_tf32(x.w));
  *reinterpret_cast<float4*>(hi + off) = make_float4(h0, h1, h2, h3);
  *reinterpret_cast<float4*>(lo + off) =
      make_float4(__uint_as_float(to_tf32(x.x - h0)), __uint_as_float(to_tf32(x.y - h1)),
                  __uint_as_float(to_tf32(x.z - h2)), __uint_as_float(to_tf32(x.w - h3)));
}

template <bool HAS_M>
__global__ void __launch_bounds__(UTHREADS, 1)
    update_tc128_kernel(int64_t n, const float* __restrict__ P, const float* __restrict__ A,
                        const float* __restrict__ M, float eta, const float* __restrict__ scale,
                        float* __restrict__ out) {
  // no-swizzle UMMA operands need 16-B alignment only; keeping the pointer a
  // plain offset of the __shared__ array lets every access compile to STS/LDS
  extern __shared__ __align__(128) float sm[];
  float* Bhi = sm;
  float* Blo = Bhi + UB_F;
  float* ring = Blo + UB_F;  // slot s: hi at ring + 2*s*UCHUNK_F, lo right after
  float* stg_all = ring + UNSLOT * 2 * UCHUNK_F;  // epilogue transposition buffers
  float* ssc = stg_all + 8 * USTG_F;
  __shared__ uint64_t slot_full[UNSLOT], slot_free[UNSLOT], acc_full[2], acc_free[2];
  __shared__ uint32_t tmem_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t ntiles = (n + UTM - 1) / UTM;
  const int64_t my_tiles = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;

  if (warp == UMMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_sh)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < UNSLOT; ++i) {
      mbar_init(&slot_full[i], 256);
      mbar_init(&slot_free[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_free[i], 256);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // B operand: element (output column c, K index q) = A[q][c], K-major
  for (int e = tid; e < UK * (UK / 4); e += UTHREADS) {
    const int c = e % UK, q4 = e / UK;  // lanes take consecutive c: conflict-free stores
    float4 x;
    x.x = __ldg(A + (4 * q4 + 0) * UK + c);
    x.y = __ldg(A + (4 * q4 + 1) * UK + c);
    x.z = __ldg(A + (4 * q4 + 2) * UK + c);
    x.w = __ldg(A + (4 * q4 + 3) * UK + c);
    split_store(Bhi, Blo, ukmaj(c, 4 * q4), x);
  }
  for (int e = tid; e < UK; e += UTHREADS) ssc[e] = scale ? __ldg(scale + e) : 1.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_sh;

  if (warp < 8) {
    // ---------------- converters: P rows -> hi/lo K-major chunks ----------
    const int64_t nq = my_tiles * UNCH;
    float4 cur[4], nxt[4];
    auto load = [&](int64_t q, float4 (&v)[4]) {
      const int64_t r0 = (blockIdx.x + (q / UNCH) * gridDim.x) * (int64_t)UTM;
      const int c0 = (int)(q % UNCH) * UKC;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int idx = tid + 256 * i;  // 128 rows x 8 float4 per chunk
#if UPD_COAL
        // 8 rows x 4 consecutive float4 per instruction (64 B of each row)
        const int m = ((idx >> 5) & 15) * 8 + (idx & 7), kq = ((idx >> 9) & 1) * 4 + ((idx >> 3) & 3);
#else
        const int m = idx & (UTM - 1), kq = idx >> 7;  // one row per lane: conflict-free stores
#endif
        const int64_t r = r0 + m;
        v[i] = (r < n) ? __ldg(reinterpret_cast<const float4*>(P + r * UK + c0) + kq)
                       : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    float4 nx2[4], nx3[4];  // three chunks of loads in flight ahead of the stores
    if (nq > 0) load(0, cur);
    if (nq > 1) load(1, nxt);
    if (nq > 2) load(2, nx2);
    for (int64_t q = 0; q < nq; ++q) {
      if (q + 3 < nq) load(q + 3, nx3);
      const int slot = (int)(q % UNSLOT);
      if (q >= UNSLOT) mbar_wait(&slot_free[slot], (uint32_t)(((q / UNSLOT) - 1) & 1));
      float* hi = ring + slot * 2 * UCHUNK_F;
      float* lo = hi + UCHUNK_F;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int idx = tid + 256 * i;
#if UPD_COAL
        split_store(hi, lo, ukmaj(((idx >> 5) & 15) * 8 + (idx & 7),
                                  4 * (((idx >> 9) & 1) * 4 + ((idx >> 3) & 3))), cur[i]);
#else
        split_store(hi, lo, ukmaj(idx & (UTM - 1), 4 * (idx >> 7)), cur[i]);
#endif
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&slot_full[slot]);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        cur[i] = nxt[i];
        nxt[i] = nx2[i];
        nx2[i] = nx3[i];
      }
    }
  } else if (warp == UMMA_WARP) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      constexpr uint32_t idesc = instr_desc_tf32(UTM, UK);
      constexpr uint32_t KSTEP_B = UKSTEP_F * 4;
      const uint32_t bhi = smem_u32(Bhi), blo = smem_u32(Blo);
      for (int64_t j = 0; j < my_tiles; ++j) {
        const int ab = (int)(j & 1);
        if (j >= 2) mbar_wait(&acc_free[ab], (uint32_t)(((j / 2) - 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t tacc = tmem + (uint32_t)(ab * UK);
        for (int c = 0; c < UNCH; ++c) {
          const int64_t q = j * UNCH + c;
          const int slot = (int)(q % UNSLOT);
          mbar_wait(&slot_full[slot], (uint32_t)((q / UNSLOT) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t ahi = smem_u32(ring + slot * 2 * UCHUNK_F);
          const uint32_t alo = ahi + UCHUNK_F * 4;
#pragma unroll
          for (int s = 0; s < UKC / 8; ++s) {
            const int ks = c * (UKC / 8) + s;
            const uint64_t dah = smem_desc(ahi + s * KSTEP_B, USBO, ULBO);
            const uint64_t dal = smem_desc(alo + s * KSTEP_B, USBO, ULBO);
            const uint64_t dbh = smem_desc(bhi + ks * KSTEP_B, USBO, ULBO);
            const uint64_t dbl = smem_desc(blo + ks * KSTEP_B, USBO, ULBO);
            mma_tf32(tacc, dah, dbh, idesc, (c | s) ? 1u : 0u);
            mma_tf32(tacc, dah, dbl, idesc, 1u);
            mma_tf32(tacc, dal, dbh, idesc, 1u);
          }
          mma_commit(&slot_free[slot]);
        }
        mma_commit(&acc_full[ab]);
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue (warps 8-15) -------------------------------
    const int quarter = warp & 3;                    // TMEM lanes 32*quarter ..
    const int cbase = ((warp - 8) >> 2) * (UK / 2);  // column half
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    float* stg = stg_all + (warp - 8) * USTG_F;
    const int crow = lane >> 2, c4 = (lane & 3) * 4;  // coalesced order: 8 rows x 4 float4
    for (int64_t j = 0; j < my_tiles; ++j) {
      const int ab = (int)(j & 1);
      const int64_t rq = (blockIdx.x + j * gridDim.x) * (int64_t)UTM + quarter * 32;  // row of lane 0
      // M of this warp's 32 rows x 64 columns, coalesced, in flight during the MMAs
      float4 mv[16];
#pragma unroll
      for (int g = 0; g < 4; ++g)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t r = rq + 8 * i + crow;
          mv[4 * g + i] = (HAS_M && r < n)
                              ? __ldg(reinterpret_cast<const float4*>(M + r * UK + cbase + 16 * g + c4))
                              : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      mbar_wait_sleep(&acc_full[ab], (uint32_t)((j / 2) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int g = 0; g < 4; ++g) {  // 16 columns per round
        const int cg = cbase + 16 * g;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          *reinterpret_cast<float4*>(stg + (8 * i + crow) * USTG_LD + c4) = mv[4 * g + i];
        __syncwarp();
        float v[16];
        tmem_ld16(tmem + (uint32_t)(ab * UK + cg) + lane_base, v);
        float* my = stg + lane * USTG_LD;  // this lane's row
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const float4 m4 = *reinterpret_cast<const float4*>(my + 4 * h);
          const float* sc = ssc + cg + 4 * h;
          float4 o = make_float4(v[4 * h], v[4 * h + 1], v[4 * h + 2], v[4 * h + 3]);
          if (HAS_M)
            o = make_float4(fmaf(eta, m4.x, o.x), fmaf(eta, m4.y, o.y), fmaf(eta, m4.z, o.z),
                            fmaf(eta, m4.w, o.w));
          *reinterpret_cast<float4*>(my + 4 * h) =
              make_float4(o.x * sc[0], o.y * sc[1], o.z * sc[2], o.w * sc[3]);
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t r = rq + 8 * i + crow;
          if (r < n)
            *reinterpret_cast<float4*>(out + r * UK + cg + c4) =
                *reinterpret_cast<const float4*>(stg + (8 * i + crow) * USTG_LD + c4);
        }
        __syncwarp();
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&acc_free[ab]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == UMMA_WARP) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
  }
}

}  // namespace

// P A (+ eta M), columns scaled by `scale` (NULL = 1); k = 128, 16-B aligned.
int launch_update_tc128(int64_t n, const float* P, const float* A, const float* M, float eta,
                        const float* scale, float* out, cudaStream_t s) {
  static PerDeviceOnce attr;  // per device: function attributes are per context
  {
    const int rc_ = attr([&]() -> int {
      SPED_CUDA(cudaFuncSetAttribute(update_tc128_kernel<true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, USMEM));
      SPED_CUDA(cudaFuncSetAttribute(update_tc128_kernel<false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, USMEM));
      return SPED_OK;
    });
    if (rc_ != SPED_OK) return rc_;
  }
  const int64_t ntiles = (n + UTM - 1) / UTM;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)num_sms()));
  if (M)
    update_tc128_kernel<true><<<grid, UTHREADS, USMEM, s>>>(n, P, A, M, eta, scale, out);
  else
    update_tc128_kernel<false><<<grid, UTHREADS, USMEM, s>>>(n, P, A, M, eta, scale, out);
  SPED_LAUNCH_CHECK();
  return SPED_OK;
}

}  // namespace sped
