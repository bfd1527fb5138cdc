// Probe: do two TMEM-allocating CTAs share an SM when launched normally
// (no cooperative launch)?  Each CTA records SM id and start/end time.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256, 2) k_tm(unsigned long long* rec) {
  __shared__ unsigned tb;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        (unsigned)__cvta_generic_to_shared(&tb)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  unsigned long long t1 = t0;
  while (t1 - t0 < 200000) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));  // 200 us
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tb));
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    rec[blockIdx.x * 3] = smid;
    rec[blockIdx.x * 3 + 1] = t0;
    rec[blockIdx.x * 3 + 2] = t1;
  }
}
int main() {
  const int n = 296;
  unsigned long long* d;
  cudaMalloc(&d, n * 3 * 8);
  k_tm<<<n, 256>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<unsigned long long> h(n * 3);
  cudaMemcpy(h.data(), d, n * 24, cudaMemcpyDeviceToHost);
  unsigned long long tmin = ~0ull, tmax = 0;
  for (int i = 0; i < n; ++i) { tmin = std::min(tmin, h[i * 3 + 1]); tmax = std::max(tmax, h[i * 3 + 2]); }
  int overlap = 0;
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j)
      if (h[i * 3] == h[j * 3] && h[i * 3 + 1] < h[j * 3 + 2] && h[j * 3 + 1] < h[i * 3 + 2]) ++overlap;
  printf("%s: span %.1f us for %d CTAs of 200 us; co-resident pairs on one SM: %d\n", cudaGetErrorString(e),
         (tmax - tmin) / 1e3, n, overlap);
  return 0;
}
