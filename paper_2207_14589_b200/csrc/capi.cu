// C-ABI plumbing: error text, ABI version, and row gather for halo staging.

#include "sped_common.cuh"

namespace sped {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

namespace {
// Halo staging: dst[r] = src[rows[r]] for rows of `cols` elements of T
// (float4 when k % 4 == 0 and both blocks are 16-B aligned, else float).
// threadIdx.x walks a row's columns, threadIdx.y picks the row: no per-element
// index division, and each row id is read once per row.
template <class T>
__global__ void gather_rows_kernel(int64_t count, int32_t cols, const int32_t* __restrict__ rows,
                                   const T* __restrict__ src, T* __restrict__ dst) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.y + threadIdx.y; r < count;
       r += (int64_t)gridDim.x * blockDim.y) {
    const T* s = src + (int64_t)__ldg(rows + r) * cols;
    T* d = dst + r * cols;
    for (int c = threadIdx.x; c < cols; c += blockDim.x) d[c] = __ldg(s + c);
  }
}

template <class T>
void launch_gather(int64_t count, int32_t cols, const int32_t* rows, const T* src, T* dst,
                   cudaStream_t s) {
  const int bx = cols >= 32 ? 32 : (cols >= 16 ? 16 : (cols >= 8 ? 8 : (cols >= 4 ? 4 : (cols >= 2 ? 2 : 1))));
  const dim3 block(bx, 256 / bx);
  gather_rows_kernel<T><<<grid_for(count, (int)block.y, num_sms() * 8), block, 0, s>>>(count, cols, rows,
                                                                                     src, dst);
}
}  // namespace

}  // namespace sped

using namespace sped;

extern "C" const char* sped_last_error(void) { return g_err; }

extern "C" int sped_abi_version(void) { return 1; }

extern "C" int sped_gather_rows(int64_t count, int32_t k, const int32_t* rows, const float* src,
                                float* dst, sped_stream_t stream) {
  SPED_CHECK_ARG(count >= 0 && k >= 1, "bad gather arguments");
  if (count == 0) return SPED_OK;
  SPED_CHECK_ARG(rows && src && dst, "null gather array");
  cudaStream_t s = as_stream(stream);
  const bool vec = (k % 4 == 0) &&
                   ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) % 16 == 0);
  if (vec)
    launch_gather<float4>(count, k / 4, rows, reinterpret_cast<const float4*>(src),
                          reinterpret_cast<float4*>(dst), s);
  else
    launch_gather<float>(count, k, rows, src, dst, s);
  SPED_LAUNCH_CHECK();
  return SPED_OK;
}

// debug-check builds (sped_common.cuh): OR of every unit's check bits, cleared
extern "C" unsigned int sped_debug_take_spmm(void);
extern "C" unsigned int sped_debug_take_csr(void);
extern "C" unsigned int sped_debug_take_edge_batch(void);
extern "C" int sped_debug_checks(void) { return SPED_DEBUG_CHECKS; }
extern "C" unsigned int sped_debug_take(void) {
  return sped_debug_take_spmm() | sped_debug_take_csr() | sped_debug_take_edge_batch();
}
