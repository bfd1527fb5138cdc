// Probe: blocks per SM the occupancy API reports for 256-thread kernels with
// and without a tcgen05.alloc, at 2 CTAs/SM launch bounds.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256, 2) k_plain(float* o) {
  float a[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) a[i] = o[threadIdx.x + i * 256];
  float s = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) s += a[i] * a[(i + 7) & 31];
  o[threadIdx.x] = s;
}
__global__ void __launch_bounds__(256, 2) k_tm(float* o) {
  __shared__ unsigned tb;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        (unsigned)__cvta_generic_to_shared(&tb)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  o[threadIdx.x] = (float)tb;
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tb));
}
int main() {
  int nb = -1;
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k_plain);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_plain, 256, 0);
  printf("plain: regs %d -> %d blocks/SM\n", fa.numRegs, nb);
  cudaFuncGetAttributes(&fa, k_tm);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_tm, 256, 0);
  printf("tmem alloc: regs %d -> %d blocks/SM\n", fa.numRegs, nb);
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxRegistersPerMultiprocessor, 0);
  printf("regs/SM %d\n", v);
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxBlocksPerMultiprocessor, 0);
  printf("blocks/SM %d\n", v);
  return 0;
}
