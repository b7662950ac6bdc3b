// K4: bit-exact numpy `Generator(PCG64).integers(0, m, size)` on the device
// (the minibatch draw of the stochastic oracle, solvers.py:171).
//
// numpy path for 1 < m <= 2^32-1 (int64 output, rng = m-1 < 0xFFFFFFFF):
//   random_bounded_uint64_fill -> buffered_bounded_lemire_uint32 ->
//   pcg64_next32: the 64-bit PCG XSL-RR output of the *stepped* state is split
//   low half first, the high half is buffered (has_uint32/uinteger) and the
//   buffer survives across calls.  Lemire: p = d * m (64-bit); accept iff
//   (p mod 2^32) >= (2^32 - m) mod m; value = p >> 32.
// Because the buffer carries over, ell successive integers(0, m, B) calls equal
// one call of ell*B draws, so a whole polynomial's batches come from one
// launch sequence.
//
// Parallelisation: thread t owns 64-bit outputs [t*G, (t+1)*G) and jumps its
// LCG state ahead with the O(log n) affine-power method (128-bit arithmetic).
// Pass 1 counts accepted candidates per block, a scan gives block offsets,
// pass 2 regenerates and compacts (rank < count) into `out` and records the
// index of the last consumed 32-bit draw.

#include <cub/cub.cuh>

#include "sped_common.cuh"

namespace sped {
namespace {

typedef unsigned __int128 u128;

constexpr int PG = 8;          // 64-bit outputs per thread
constexpr int PT = 256;        // threads per block

__host__ __device__ __forceinline__ u128 mk128(uint64_t hi, uint64_t lo) {
  return ((u128)hi << 64) | (u128)lo;
}
__device__ __forceinline__ u128 pcg_mult() {
  return mk128(2549297995355413924ULL, 4865540595714422341ULL);
}

// state after `delta` steps of s <- s*a + c
__device__ __forceinline__ u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
  u128 cur_mult = pcg_mult(), cur_plus = inc;
  u128 acc_mult = 1, acc_plus = 0;
  while (delta > 0) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

__device__ __forceinline__ uint64_t pcg_output(u128 s) {
  const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  const unsigned rot = (unsigned)(hi >> 58);
  const uint64_t x = hi ^ lo;
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

struct Params {
  u128 state, inc;
  int32_t has;          // buffered candidate at index 0
  uint32_t uinteger;
  uint32_t m;
  uint32_t thresh;
  int64_t n_out64;      // 64-bit outputs generated in total
};

__device__ __forceinline__ bool accept(uint32_t d, uint32_t m, uint32_t thresh, uint32_t* val) {
  const uint64_t p = (uint64_t)d * (uint64_t)m;
  *val = (uint32_t)(p >> 32);
  return (uint32_t)p >= thresh;
}

// count accepted candidates of this thread (buffered candidate belongs to
// thread 0 of block 0, ahead of its outputs)
__device__ __forceinline__ int thread_count(const Params& P, int64_t j0) {
  int c = 0;
  uint32_t v;
  if (j0 == 0 && P.has) c += accept(P.uinteger, P.m, P.thresh, &v);
  if (j0 >= P.n_out64) return c;
  u128 s = pcg_advance(P.state, P.inc, (uint64_t)j0);
  const int64_t jn = min((int64_t)PG, P.n_out64 - j0);
  for (int64_t q = 0; q < jn; ++q) {
    s = s * pcg_mult() + P.inc;
    const uint64_t o = pcg_output(s);
    c += accept((uint32_t)o, P.m, P.thresh, &v);
    c += accept((uint32_t)(o >> 32), P.m, P.thresh, &v);
  }
  return c;
}

__global__ void __launch_bounds__(PT) pcg_count_kernel(Params P, int32_t* block_counts) {
  typedef cub::BlockReduce<int, PT> BR;
  __shared__ typename BR::TempStorage tmp;
  const int64_t t = (int64_t)blockIdx.x * PT + threadIdx.x;
  const int c = thread_count(P, t * PG);
  const int tot = BR(tmp).Sum(c);
  if (threadIdx.x == 0) block_counts[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(PT) pcg_emit_kernel(Params P, const int32_t* block_offsets,
                                                      int64_t count, int32_t* out,
                                                      int64_t* last_draw) {
  typedef cub::BlockScan<int, PT> BS;
  __shared__ typename BS::TempStorage tmp;
  const int64_t t = (int64_t)blockIdx.x * PT + threadIdx.x;
  const int64_t j0 = t * PG;
  const int c = thread_count(P, j0);
  int excl = 0;
  BS(tmp).ExclusiveSum(c, excl);
  int64_t rank = (int64_t)block_offsets[blockIdx.x] + excl;
  if (rank >= count || c == 0) return;
  uint32_t v;
  if (j0 == 0 && P.has) {
    if (accept(P.uinteger, P.m, P.thresh, &v)) {
      if (rank < count) out[rank] = (int32_t)v;
      if (rank == count - 1) *last_draw = 0;
      ++rank;
    }
  }
  if (j0 >= P.n_out64) return;
  u128 s = pcg_advance(P.state, P.inc, (uint64_t)j0);
  const int64_t jn = min((int64_t)PG, P.n_out64 - j0);
  for (int64_t q = 0; q < jn && rank < count; ++q) {
    s = s * pcg_mult() + P.inc;
    const uint64_t o = pcg_output(s);
    const int64_t base = (int64_t)P.has + 2 * (j0 + q);  // draw index of the low half
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t d = h ? (uint32_t)(o >> 32) : (uint32_t)o;
      if (accept(d, P.m, P.thresh, &v) && rank < count) {
        out[rank] = (int32_t)v;
        if (rank == count - 1) *last_draw = base + h;
        ++rank;
      }
    }
  }
}

}  // namespace
}  // namespace sped

using namespace sped;

extern "C" size_t sped_pcg64_workspace_bytes(int64_t count) {
  // generous: candidates for count*(1+2^-3) + 4096 draws
  const int64_t outs = (count + count / 8 + 4096) / 2 + 1;
  const int64_t blocks = (outs + (int64_t)PT * PG - 1) / ((int64_t)PT * PG);
  size_t scan_tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_tmp, (int32_t*)nullptr, (int32_t*)nullptr,
                                (int)(blocks + 1));
  return 512 + sizeof(int32_t) * 2 * (blocks + 1) + sizeof(int64_t) + scan_tmp;
}

extern "C" int sped_pcg64_integers(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                                   uint64_t inc_lo, int32_t has_uint32, uint32_t uinteger,
                                   uint64_t m, int64_t count, int32_t* out, int64_t* draws32_out,
                                   void* workspace, size_t workspace_bytes, sped_stream_t stream) {
  SPED_CHECK_ARG(count >= 0 && draws32_out, "bad pcg64 arguments");
  SPED_CHECK_ARG(m >= 1 && m <= (uint64_t)INT32_MAX, "m must be in [1, 2^31-1]");
  cudaStream_t s = as_stream(stream);
  *draws32_out = 0;
  if (count == 0) return SPED_OK;
  SPED_CHECK_ARG(out != nullptr, "null output");
  if (m == 1) {  // numpy: rng == 0 fills `off` without drawing
    SPED_CUDA(cudaMemsetAsync(out, 0, sizeof(int32_t) * count, s));
    return SPED_OK;
  }
  SPED_CHECK_ARG(workspace && workspace_bytes >= sped_pcg64_workspace_bytes(count),
                 "pcg64 workspace too small");
  Params P;
  P.state = mk128(state_hi, state_lo);
  P.inc = mk128(inc_hi, inc_lo);
  P.has = has_uint32 ? 1 : 0;
  P.uinteger = uinteger;
  P.m = (uint32_t)m;
  P.thresh = (uint32_t)((0x100000000ULL - m) % m);
  // candidates: the rejection rate is thresh/2^32 < m/2^32
  const double prej = (double)P.thresh / 4294967296.0;
  int64_t need = count + (int64_t)(count * prej * 2.0) + 4096;
  if (need > count + count / 8 + 4096) need = count + count / 8 + 4096;
  P.n_out64 = need / 2 + 1;
  const int64_t blocks = (P.n_out64 + (int64_t)PT * PG - 1) / ((int64_t)PT * PG);
  SPED_CHECK_ARG(blocks < INT32_MAX, "count too large");
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  int32_t* counts = reinterpret_cast<int32_t*>(ws);
  int32_t* offsets = counts + (blocks + 1);
  int64_t* last = reinterpret_cast<int64_t*>(
      (reinterpret_cast<uintptr_t>(offsets + blocks + 1) + 15) & ~uintptr_t(15));
  void* scan_tmp = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(last + 1) + 255) &
                                           ~uintptr_t(255));
  size_t scan_bytes = workspace_bytes - (reinterpret_cast<uint8_t*>(scan_tmp) - ws);
  SPED_CUDA(cudaMemsetAsync(counts + blocks, 0, sizeof(int32_t), s));
  SPED_CUDA(cudaMemsetAsync(last, 0xff, sizeof(int64_t), s));
  pcg_count_kernel<<<(unsigned)blocks, PT, 0, s>>>(P, counts);
  SPED_LAUNCH_CHECK();
  SPED_CUDA(cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, counts, offsets, (int)(blocks + 1), s));
  pcg_emit_kernel<<<(unsigned)blocks, PT, 0, s>>>(P, offsets, count, out, last);
  SPED_LAUNCH_CHECK();
  int64_t last_h = -1;
  SPED_CUDA(cudaMemcpyAsync(&last_h, last, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SPED_CUDA(cudaStreamSynchronize(s));
  if (last_h < 0) {
    set_error("pcg64: candidate pool exhausted (count=%lld)", (long long)count);
    return SPED_ERR_UNSUPPORTED;
  }
  *draws32_out = last_h + 1;
  return SPED_OK;
}
