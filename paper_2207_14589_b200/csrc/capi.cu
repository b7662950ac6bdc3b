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
__global__ void gather_rows_kernel(int64_t count, int32_t k, const int32_t* __restrict__ rows,
                                   const float* __restrict__ src, float* __restrict__ dst) {
  const int64_t total = count * (int64_t)k;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / k;
    const int c = (int)(i % k);
    dst[i] = src[(int64_t)rows[r] * k + c];
  }
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
  gather_rows_kernel<<<grid_for(count * k, 256, num_sms() * 16), 256, 0, as_stream(stream)>>>(
      count, k, rows, src, dst);
  SPED_LAUNCH_CHECK();
  return SPED_OK;
}
