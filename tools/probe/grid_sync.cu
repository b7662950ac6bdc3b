// Probe: cost of a grid-wide barrier on B200 (cooperative-groups grid.sync
// vs a hand-rolled sense-reversing barrier), 1024-thread CTAs, 1 per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o grid_sync grid_sync.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void __launch_bounds__(1024, 1) cg_sync(int iters) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) g.sync();
}

__device__ __forceinline__ void my_barrier(unsigned* count, unsigned* gen, unsigned nb, unsigned& local_gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned target = local_gen + 1;
    __threadfence();
    if (atomicAdd(count, 1) == nb - 1) {
      atomicExch(count, 0);
      __threadfence();
      atomicExch(gen, target);
    } else {
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(gen));
      } while (v != target);
    }
  }
  local_gen += 1;
  __syncthreads();
}

__global__ void __launch_bounds__(1024, 1) my_sync(int iters, unsigned* count, unsigned* gen) {
  unsigned lg = 0;
  for (int i = 0; i < iters; ++i) my_barrier(count, gen, gridDim.x, lg);
}

// red.release + ld.acquire version with per-arrival counter (no reset):
// generation = arrivals / nb
__device__ __forceinline__ void mono_barrier(unsigned* count, unsigned nb, unsigned& epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    epoch += 1;
    const unsigned target = epoch * nb;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(count) : "memory");
    } while ((int)(v - target) < 0);
  }
  __syncthreads();
}

__global__ void __launch_bounds__(1024, 1) mono_sync(int iters, unsigned* count) {
  unsigned ep = 0;
  for (int i = 0; i < iters; ++i) mono_barrier(count, gridDim.x, ep);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* buf;
  cudaMalloc(&buf, 256);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 20000;
  for (int grid : {8, 32, 74, sms}) {
    void* args1[] = {(void*)&iters};
    cudaLaunchCooperativeKernel((void*)cg_sync, grid, 1024, args1, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)cg_sync, grid, 1024, args1, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms1;
    cudaEventElapsedTime(&ms1, a, b);
    cudaMemset(buf, 0, 256);
    unsigned* cnt = buf;
    unsigned* gen = buf + 32;
    void* args2[] = {(void*)&iters, (void*)&cnt, (void*)&gen};
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)my_sync, grid, 1024, args2, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms2;
    cudaEventElapsedTime(&ms2, a, b);
    cudaMemset(buf, 0, 256);
    void* args3[] = {(void*)&iters, (void*)&cnt};
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)mono_sync, grid, 1024, args3, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms3;
    cudaEventElapsedTime(&ms3, a, b);
    printf("grid %3d: cg grid.sync %.3f us, sense barrier %.3f us, monotonic barrier %.3f us\n",
           grid, ms1 * 1e3 / iters, ms2 * 1e3 / iters, ms3 * 1e3 / iters);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
