// Standalone tcgen05 probe: one 8-row K step of D = Z^T Z with MN-major
// no-swizzle descriptors (the sped gram_tc layout), M=N in {64,128}.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t sbo, uint32_t lbo, int version) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)version << 46;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int M, int N, int amaj, int bmaj) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)amaj << 15) | ((uint32_t)bmaj << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int K2>
__global__ void probe(const float* Z /* 8 x K2 row-major */, float* D /* K2 x K2 */, int version, int lbo, int mode) {
  __shared__ __align__(1024) float tile[K2 * 8];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tbase)), "r"(K2 <= 64 ? 64 : 128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (mode == 1) {
    // MN-major: element (r, c) at ((c/4)*8 + r)*4 + c%4   (KC = 8)
    for (int e = tid; e < 8 * K2; e += blockDim.x) {
      int r = e / K2, c = e % K2;
      tile[((c / 4) * 8 + r) * 4 + c % 4] = Z[r * K2 + c];
    }
  } else {
    // K-major: element (m=c, k=r): (k/4)*LBO + (m/8)*128B + (m%8)*16B + (k%4)*4B, LBO = K2*16B
    for (int e = tid; e < 8 * K2; e += blockDim.x) {
      int r = e / K2, c = e % K2;
      tile[(r / 4) * (K2 * 4) + (c / 8) * 32 + (c % 8) * 4 + (r % 4)] = Z[r * K2 + c];
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t tmem = tbase;
  if (tid == 0) {
    uint32_t a = smem_u32(tile);
    uint64_t da = (mode == 1) ? smem_desc(a, 8 * 16, lbo, version) : smem_desc(a, 128, K2 * 16, version);
    uint32_t id = idesc(K2, K2, mode, mode);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                 :: "r"(tmem), "l"(da), "l"(da), "r"(id), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}\n" :: "r"(smem_u32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int c0 = 0; c0 < K2; c0 += 16) {
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15])
      : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    int lanerow = warp * 32 + lane;  // raw TMEM lane
    for (int i = 0; i < 16; ++i) D[lanerow * K2 + c0 + i] = __uint_as_float(r[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(K2 <= 64 ? 64 : 128));
}

template <int K2>
void run(int version, int lbo, int mode) {
  std::vector<float> Z(8 * K2);
  for (int r = 0; r < 8; ++r) for (int c = 0; c < K2; ++c) Z[r * K2 + c] = (float)((r * 7 + c * 3) % 5 - 2);
  std::vector<double> ref(K2 * K2, 0.0);
  for (int i = 0; i < K2; ++i) for (int j = 0; j < K2; ++j) for (int r = 0; r < 8; ++r) ref[i * K2 + j] += Z[r * K2 + i] * Z[r * K2 + j];
  float *dZ, *dD;
  cudaMalloc(&dZ, sizeof(float) * Z.size());
  cudaMalloc(&dD, sizeof(float) * 128 * K2);
  cudaMemset(dD, 0, sizeof(float) * 128 * K2);
  cudaMemcpy(dZ, Z.data(), sizeof(float) * Z.size(), cudaMemcpyHostToDevice);
  probe<K2><<<1, 128>>>(dZ, dD, version, lbo, mode);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> D(128 * K2);
  cudaMemcpy(D.data(), dD, sizeof(float) * D.size(), cudaMemcpyDeviceToHost);
  // map rows: M=128 -> lane m; M=64 -> lane (m%16)+32*(m/16)
  double err = 0, mag = 0; int nz = 0;
  for (int m = 0; m < K2; ++m) {
    int lanerow = (K2 == 128) ? m : (m % 16) + 32 * (m / 16);
    for (int j = 0; j < K2; ++j) { double d = D[lanerow * K2 + j]; err = fmax(err, fabs(d - ref[m * K2 + j])); mag = fmax(mag, fabs(ref[m*K2+j])); nz += d != 0; }
  }
  // alt mapping M=64 -> lanes 0..63
  double err2 = 0;
  for (int m = 0; m < K2; ++m) for (int j = 0; j < K2; ++j) err2 = fmax(err2, fabs(D[m * K2 + j] - ref[m * K2 + j]));
  printf("K2=%d version=%d lbo=%d mode=%d cuda=%s  maxerr=%g (alt %g) |ref|max=%g nonzero=%d  D[0][0..3]=%g %g %g %g ref %g %g %g %g\n",
         K2, version, lbo, mode, cudaGetErrorString(e), err, err2, mag, nz, D[0], D[1], D[2], D[3], ref[0], ref[1], ref[2], ref[3]);
  cudaFree(dZ); cudaFree(dD);
}

int main() {
  run<128>(1, 128, 0);
  run<64>(1, 128, 0);
  run<128>(1, 128, 1);
  return 0;
}
