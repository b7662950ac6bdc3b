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
// The generator state can live on the device (sped_pcg64_integers_device:
// words state_hi, state_lo, inc_hi, inc_lo, has_uint32, uinteger): the
// kernels read it there and a one-thread finalize kernel advances it by the
// number of 32-bit draws consumed, so a draw never waits on the host and a
// whole stochastic solver step can be captured in a CUDA graph.
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

// the generator words of the device-resident state
__device__ __forceinline__ Params with_state(Params P, const uint64_t* __restrict__ sw) {
  P.state = mk128(sw[0], sw[1]);
  P.inc = mk128(sw[2], sw[3]);
  P.has = sw[4] ? 1 : 0;
  P.uinteger = (uint32_t)sw[5];
  return P;
}

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

__global__ void __launch_bounds__(PT) pcg_count_kernel(Params P0, const uint64_t* sw,
                                                       int32_t* block_counts) {
  const Params P = with_state(P0, sw);
  typedef cub::BlockReduce<int, PT> BR;
  __shared__ typename BR::TempStorage tmp;
  const int64_t t = (int64_t)blockIdx.x * PT + threadIdx.x;
  const int c = thread_count(P, t * PG);
  const int tot = BR(tmp).Sum(c);
  if (threadIdx.x == 0) block_counts[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(PT) pcg_emit_kernel(Params P0, const uint64_t* sw,
                                                      const int32_t* block_offsets,
                                                      int64_t count, int32_t* out,
                                                      int64_t* last_draw) {
  const Params P = with_state(P0, sw);
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

// numpy's state after `last_draw + 1` 32-bit draws (sampling.py's
// pcg64_advance_state on the device); an exhausted candidate pool leaves the
// state unchanged and sets status bit 0.
__global__ void pcg_finalize_kernel(uint64_t* sw, const int64_t* last_draw, int32_t* status) {
  const int64_t l = *last_draw;
  if (l < 0) {
    if (status) atomicOr(status, 1);
    return;
  }
  const int64_t r = (l + 1) - (sw[4] ? 1 : 0);
  if (r <= 0) {
    sw[4] = 0;
    return;
  }
  const u128 st = pcg_advance(mk128(sw[0], sw[1]), mk128(sw[2], sw[3]), (uint64_t)((r + 1) / 2));
  sw[0] = (uint64_t)(st >> 64);
  sw[1] = (uint64_t)st;
  sw[4] = (uint64_t)(r % 2);
  sw[5] = pcg_output(st) >> 32;
}

struct PcgWs {
  int32_t *counts, *offsets;
  int64_t* last;
  uint64_t* words;  // host-state entry point: the state staged here
  void* scan_tmp;
  size_t scan_bytes;
};

PcgWs pcg_ws(void* workspace, size_t workspace_bytes, int64_t blocks) {
  PcgWs w;
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  w.counts = reinterpret_cast<int32_t*>(ws);
  w.offsets = w.counts + (blocks + 1);
  w.last = reinterpret_cast<int64_t*>(
      (reinterpret_cast<uintptr_t>(w.offsets + blocks + 1) + 15) & ~uintptr_t(15));
  w.words = reinterpret_cast<uint64_t*>(w.last + 1);
  w.scan_tmp = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(w.words + 6) + 255) &
                                       ~uintptr_t(255));
  w.scan_bytes = workspace_bytes - (reinterpret_cast<uint8_t*>(w.scan_tmp) - ws);
  return w;
}

// draws `count` integers with the state in device memory `sw`, all on stream
// `s` (no host synchronisation); advances `sw`.
int pcg_draw_device(uint64_t* sw, uint64_t m, int64_t count, int32_t* out, int32_t* status,
                    void* workspace, size_t workspace_bytes, cudaStream_t s, int64_t** last_out) {
  Params P{};
  P.m = (uint32_t)m;
  P.thresh = (uint32_t)((0x100000000ULL - m) % m);
  // candidates: the rejection rate is thresh/2^32 < m/2^32
  const double prej = (double)P.thresh / 4294967296.0;
  int64_t need = count + (int64_t)(count * prej * 2.0) + 4096;
  if (need > count + count / 8 + 4096) need = count + count / 8 + 4096;
  P.n_out64 = need / 2 + 1;
  const int64_t blocks = (P.n_out64 + (int64_t)PT * PG - 1) / ((int64_t)PT * PG);
  SPED_CHECK_ARG(blocks < INT32_MAX, "count too large");
  PcgWs w = pcg_ws(workspace, workspace_bytes, blocks);
  SPED_CUDA(cudaMemsetAsync(w.counts + blocks, 0, sizeof(int32_t), s));
  SPED_CUDA(cudaMemsetAsync(w.last, 0xff, sizeof(int64_t), s));
  pcg_count_kernel<<<(unsigned)blocks, PT, 0, s>>>(P, sw, w.counts);
  SPED_LAUNCH_CHECK();
  SPED_CUDA(cub::DeviceScan::ExclusiveSum(w.scan_tmp, w.scan_bytes, w.counts, w.offsets,
                                          (int)(blocks + 1), s));
  pcg_emit_kernel<<<(unsigned)blocks, PT, 0, s>>>(P, sw, w.offsets, count, out, w.last);
  SPED_LAUNCH_CHECK();
  pcg_finalize_kernel<<<1, 1, 0, s>>>(sw, w.last, status);
  SPED_LAUNCH_CHECK();
  if (last_out) *last_out = w.last;
  return SPED_OK;
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
  return 512 + sizeof(int32_t) * 2 * (blocks + 1) + sizeof(int64_t) * 7 + scan_tmp;
}

extern "C" int sped_pcg64_integers_device(uint64_t* state_words, uint64_t m, int64_t count,
                                          int32_t* out, int32_t* status, void* workspace,
                                          size_t workspace_bytes, sped_stream_t stream) {
  SPED_CHECK_ARG(count >= 0 && state_words, "bad pcg64 arguments");
  SPED_CHECK_ARG(m >= 1 && m <= (uint64_t)INT32_MAX, "m must be in [1, 2^31-1]");
  if (count == 0) return SPED_OK;
  SPED_CHECK_ARG(out != nullptr, "null output");
  cudaStream_t s = as_stream(stream);
  if (m == 1) {  // numpy: rng == 0 fills `off` without drawing
    SPED_CUDA(cudaMemsetAsync(out, 0, sizeof(int32_t) * count, s));
    return SPED_OK;
  }
  SPED_CHECK_ARG(workspace && workspace_bytes >= sped_pcg64_workspace_bytes(count),
                 "pcg64 workspace too small");
  return pcg_draw_device(state_words, m, count, out, status, workspace, workspace_bytes, s,
                         nullptr);
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
  // stage the host state in the workspace, draw, read back the last draw
  uint64_t words[6] = {state_hi, state_lo, inc_hi, inc_lo, (uint64_t)(has_uint32 ? 1 : 0),
                       (uint64_t)uinteger};
  // the staging words follow the block table: the same layout pcg_draw_device uses
  Params P{};
  P.m = (uint32_t)m;
  P.thresh = (uint32_t)((0x100000000ULL - m) % m);
  const double prej = (double)P.thresh / 4294967296.0;
  int64_t need = count + (int64_t)(count * prej * 2.0) + 4096;
  if (need > count + count / 8 + 4096) need = count + count / 8 + 4096;
  const int64_t blocks = (need / 2 + 1 + (int64_t)PT * PG - 1) / ((int64_t)PT * PG);
  PcgWs w = pcg_ws(workspace, workspace_bytes, blocks);
  SPED_CUDA(cudaMemcpyAsync(w.words, words, sizeof(words), cudaMemcpyHostToDevice, s));
  int64_t* last = nullptr;
  const int rc = pcg_draw_device(w.words, m, count, out, nullptr, workspace, workspace_bytes, s,
                                 &last);
  if (rc != SPED_OK) return rc;
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
