// K5 on the 5th-gen tensor cores: Gram of Z = [V | M] with tcgen05.mma
// kind::tf32 in 3xTF32 (hi*hi + hi*lo + lo*hi, fp32 accumulation in TMEM),
// for K2 = 2k in {64, 128, 256} (k = 32 / 64 / 128).
//
//   G = Z^T Z  (K2 x K2), contraction over the n rows.
//
// Operands come from ONE shared-memory tile per stage: the MMA's A = Z^T
// (M = K2 columns of Z, MN-major) and B = Z (N = K2 columns, MN-major) read
// the same canonical "interleaved" (no-swizzle) layout: element (row r, col
// c) at float offset ((c/4)*KC + r)*4 + c%4, i.e. 16-byte column groups of KC
// rows (SBO = 16*KC bytes, one K=8 block = 128 bytes).  Each thread loads
// float4s of V / M rows, splits them into tf32 hi/lo parts (cvt.rna.tf32)
// and stores both tiles; one elected thread issues the MMAs and commits them
// to the stage's mbarrier, which the loaders wait on before refilling it
// (double buffering).  Rows are processed in SPLIT-row slices; each slice's
// TMEM accumulator is drained with tcgen05.ld into an fp32 partial Gram, and
// the partials are summed in fp64 in slice order by sped_gram's reduce
// kernel (deterministic, and no fp32 sum spans more than SPLIT rows).
//
// K2 = 256 is computed as two M=128 tiles over the upper triangle:
// rows 0..127 x cols 0..255 (TMEM cols 0..255) and rows 128..255 x cols
// 128..255 (TMEM cols 256..383).

#include "sped_common.cuh"

namespace sped {
namespace tc {

constexpr int THREADS = 128;
constexpr int SPLIT = 8192;  // rows per accumulator slice

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t sbo_bytes, uint32_t lbo_bytes) {
  // SM100 UMMA shared-memory descriptor, SWIZZLE_NONE, version 1.
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (Blackwell)
  // base_offset = 0, lbo_mode = 0, layout_type (bits 61..63) = 0 (no swizzle)
  return d;
}

__host__ __device__ constexpr uint32_t instr_desc_tf32(int M, int N) {
  // c_format F32 (1) @4, a/b format TF32 (2) @7/@10, a/b major MN (1) @15/@16,
  // n_dim = N>>3 @17, m_dim = M>>4 @24
  return (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// tcgen05.ld 32 lanes x 32 bit, 16 consecutive columns per thread
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

template <int K2>
struct Cfg {
  static constexpr int KC = (K2 == 256) ? 32 : 64;             // rows per stage
  static constexpr int TILE_FLOATS = K2 * KC;                   // one of hi / lo
  static constexpr int STAGE_BYTES = 2 * TILE_FLOATS * 4;       // hi + lo
  static constexpr int TMEM_COLS = (K2 == 64) ? 64 : (K2 == 128) ? 128 : 512;
  static constexpr int SMEM = 2 * STAGE_BYTES + 1024;
};

// Gram partials: one fp32 K2 x K2 block (upper triangle meaningful) per
// SPLIT-row slice.
template <int K2>
__global__ void __launch_bounds__(THREADS, 1) gram_tc_kernel(int64_t n, int32_t k,
                                                             const float* __restrict__ V,
                                                             const float* __restrict__ M,
                                                             float* __restrict__ partial,
                                                             int64_t nslices) {
  using C = Cfg<K2>;
  extern __shared__ __align__(1024) uint8_t smem[];
  float* stage_f = reinterpret_cast<float*>(smem);
  __shared__ uint64_t bars[2];
  __shared__ uint64_t done_bar;
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_sh)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&done_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_sh;

  uint32_t stage_uses[2] = {0, 0};
  uint32_t done_uses = 0;
  const uint32_t sbo = 16u * C::KC;
  for (int64_t slice = blockIdx.x; slice < nslices; slice += gridDim.x) {
    const int64_t r_begin = slice * SPLIT;
    const int64_t r_end = min(n, r_begin + SPLIT);
    const int nchunks = (int)((r_end - r_begin + C::KC - 1) / C::KC);
    for (int ch = 0; ch < nchunks; ++ch) {
      const int s = ch & 1;
      if (stage_uses[s] > 0) mbar_wait(&bars[s], (stage_uses[s] - 1) & 1);
      float* hi = stage_f + s * (2 * C::TILE_FLOATS);
      float* lo = hi + C::TILE_FLOATS;
      const int64_t r0 = r_begin + (int64_t)ch * C::KC;
      // fill: KC rows x K2 columns as float4 groups
#pragma unroll 4
      for (int e = tid; e < C::KC * (K2 / 4); e += THREADS) {
        const int g = e / C::KC;      // column group (4 columns)
        const int r = e % C::KC;      // row within chunk
        const int64_t row = r0 + r;
        const int c = g * 4;
        float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
        if (row < r_end) {
          const float* src = (c < k) ? (V + row * k + c) : (M + row * k + (c - k));
          z = *reinterpret_cast<const float4*>(src);
        }
        uint4 h, l;
        h.x = to_tf32(z.x);
        h.y = to_tf32(z.y);
        h.z = to_tf32(z.z);
        h.w = to_tf32(z.w);
        l.x = to_tf32(z.x - __uint_as_float(h.x));
        l.y = to_tf32(z.y - __uint_as_float(h.y));
        l.z = to_tf32(z.z - __uint_as_float(h.z));
        l.w = to_tf32(z.w - __uint_as_float(h.w));
        const int off = (g * C::KC + r) * 4;
        *reinterpret_cast<uint4*>(hi + off) = h;
        *reinterpret_cast<uint4*>(lo + off) = l;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t hi_a = smem_u32(hi), lo_a = smem_u32(lo);
#pragma unroll
        for (int kb = 0; kb < C::KC / 8; ++kb) {
          const uint32_t acc0 = (ch > 0 || kb > 0) ? 1u : 0u;
          if (K2 <= 128) {
            constexpr int MM = K2;
            constexpr uint32_t idesc = instr_desc_tf32(MM, K2);
            const uint64_t dh = smem_desc(hi_a + kb * 128, sbo, 128);
            const uint64_t dl = smem_desc(lo_a + kb * 128, sbo, 128);
            mma_tf32(tmem, dh, dh, idesc, acc0);
            mma_tf32(tmem, dh, dl, idesc, 1u);
            mma_tf32(tmem, dl, dh, idesc, 1u);
          } else {
            // tile 0: rows 0..127 x cols 0..255
            constexpr uint32_t id0 = instr_desc_tf32(128, 256);
            const uint64_t ah0 = smem_desc(hi_a + kb * 128, sbo, 128);
            const uint64_t al0 = smem_desc(lo_a + kb * 128, sbo, 128);
            mma_tf32(tmem, ah0, ah0, id0, acc0);
            mma_tf32(tmem, ah0, al0, id0, 1u);
            mma_tf32(tmem, al0, ah0, id0, 1u);
            // tile 1: rows 128..255 x cols 128..255 (column groups 32..63)
            constexpr uint32_t id1 = instr_desc_tf32(128, 128);
            const uint32_t goff = 32u * sbo;
            const uint64_t ah1 = smem_desc(hi_a + goff + kb * 128, sbo, 128);
            const uint64_t al1 = smem_desc(lo_a + goff + kb * 128, sbo, 128);
            mma_tf32(tmem + 256, ah1, ah1, id1, acc0);
            mma_tf32(tmem + 256, ah1, al1, id1, 1u);
            mma_tf32(tmem + 256, al1, ah1, id1, 1u);
          }
        }
        mma_commit(&bars[s]);
      }
      stage_uses[s] += 1;
    }
    // drain the slice accumulator
    if (tid == 0) mma_commit(&done_bar);
    mbar_wait(&done_bar, done_uses & 1);
    done_uses += 1;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    float* out = partial + slice * (int64_t)K2 * K2;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    if (K2 == 64) {
      // M = 64: row m lives in lane (m % 16) + 32 * (m / 16)
      const int m = warp * 16 + lane;
      for (int c0 = 0; c0 < K2; c0 += 16) {
        float v[16];
        tmem_ld16(tmem + lane_base + c0, v);
        if (lane < 16) {
#pragma unroll
          for (int i = 0; i < 16; ++i) out[m * K2 + c0 + i] = v[i];
        }
      }
    } else if (K2 == 128) {
      const int m = warp * 32 + lane;
      for (int c0 = 0; c0 < K2; c0 += 16) {
        float v[16];
        tmem_ld16(tmem + lane_base + c0, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) out[m * K2 + c0 + i] = v[i];
      }
    } else {
      const int m = warp * 32 + lane;
      for (int c0 = 0; c0 < 256; c0 += 16) {
        float v[16];
        tmem_ld16(tmem + lane_base + c0, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) out[m * K2 + c0 + i] = v[i];
      }
      for (int c0 = 0; c0 < 128; c0 += 16) {
        float v[16];
        tmem_ld16(tmem + 256 + lane_base + c0, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) out[(128 + m) * K2 + 128 + c0 + i] = v[i];
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(C::TMEM_COLS));
  }
}

// Sum slice partials in fp64 (slice order) and scatter into S / C / Q.
__global__ void gram_tc_reduce(int32_t k, int32_t K2, int64_t nslices,
                               const float* __restrict__ partial, double* __restrict__ G) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= K2 * K2) return;
  const int i = e / K2, j = e % K2;
  if (j < i) return;
  double s = 0.0;
  for (int64_t sl = 0; sl < nslices; ++sl) s += (double)partial[sl * K2 * K2 + e];
  auto put = [&](int a, int b) {
    if (a < k && b < k) G[a * k + b] = s;
    else if (a < k) G[k * k + a * k + (b - k)] = s;
    else if (b >= k) G[2 * k * k + (a - k) * k + (b - k)] = s;
  };
  put(i, j);
  if (i != j) put(j, i);
}

template <int K2>
int launch(int64_t n, int32_t k, const float* V, const float* M, double* G, float* partial,
           cudaStream_t s) {
  using C = Cfg<K2>;
  static bool attr = false;
  if (!attr) {
    SPED_CUDA(cudaFuncSetAttribute(gram_tc_kernel<K2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   C::SMEM));
    attr = true;
  }
  const int64_t nslices = (n + SPLIT - 1) / SPLIT;
  const int per_sm = (K2 == 256) ? 1 : (K2 == 128 ? 2 : 3);
  const unsigned grid = (unsigned)std::min<int64_t>(nslices, (int64_t)num_sms() * per_sm);
  gram_tc_kernel<K2><<<grid, THREADS, C::SMEM, s>>>(n, k, V, M, partial, nslices);
  SPED_LAUNCH_CHECK();
  gram_tc_reduce<<<(K2 * K2 + 255) / 256, 256, 0, s>>>(k, K2, nslices, partial, G);
  SPED_LAUNCH_CHECK();
  return SPED_OK;
}

}  // namespace tc

bool gram_tc_supported(int32_t k, bool with_m) { return with_m && (k == 32 || k == 64 || k == 128); }

size_t gram_tc_workspace(int64_t n, int32_t k) {
  const int K2 = 2 * k;
  const int64_t nslices = (n + tc::SPLIT - 1) / tc::SPLIT;
  return sizeof(float) * (size_t)nslices * K2 * K2 + 256;
}

int gram_tc(int64_t n, int32_t k, const float* V, const float* M, double* G, void* ws,
            cudaStream_t s) {
  float* partial = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
  switch (k) {
    case 32: return tc::launch<64>(n, k, V, M, G, partial, s);
    case 64: return tc::launch<128>(n, k, V, M, G, partial, s);
    case 128: return tc::launch<256>(n, k, V, M, G, partial, s);
    default: set_error("gram_tc: unsupported k=%d", k); return SPED_ERR_UNSUPPORTED;
  }
}

}  // namespace sped
