// Probe: how many clusters of size 8/16 with 512 threads x 128 regs and ~200 KB
// smem can be co-resident, and does a 512-column TMEM alloc + st/ld round trip work.
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__global__ void __launch_bounds__(512, 1) kprobe(unsigned* out) {
  extern __shared__ unsigned char sm[];
  __shared__ unsigned taddr_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (unsigned)__cvta_generic_to_shared(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const unsigned base = taddr_s;
  const unsigned ta = base + ((unsigned)(32 * (warp & 3)) << 16) + (unsigned)((warp >> 2) * 128);
  unsigned v0 = threadIdx.x * 7 + 1, v1 = threadIdx.x * 11 + 3, v2 = 5, v3 = 9;
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(ta), "r"(v0), "r"(v1), "r"(v2), "r"(v3));
  asm volatile("tcgen05.wait::st.sync.aligned;");
  unsigned w0, w1, w2, w3;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3) : "r"(ta));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  const bool ok = (w0 == v0) && (w1 == v1) && (w2 == v2) && (w3 == v3);
  sm[threadIdx.x] = ok;
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  if (!ok) atomicAdd(out, 1u);
  if (threadIdx.x == 0) atomicAdd(out + 1, 1u);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = 200 * 1024;
  cudaFuncSetAttribute(kprobe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(kprobe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {2, 4, 8, 9, 10, 11, 12, 13, 14, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 8);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr; cfg.numAttrs = 1;
    int ncl = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, kprobe, &cfg);
    printf("cluster %2d: max active clusters %d (%s) -> %d SMs of %d\n", cs, ncl, cudaGetErrorString(e), ncl * cs, sms);
    if (e == cudaSuccess && ncl > 0) {
      unsigned* d; cudaMalloc(&d, 8); cudaMemset(d, 0, 8);
      cfg.gridDim = dim3(cs * ncl);
      e = cudaLaunchKernelEx(&cfg, kprobe, d);
      cudaError_t e2 = cudaDeviceSynchronize();
      unsigned h[2]; cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
      printf("   launch %s / %s: CTAs %u, TMEM mismatches %u\n", cudaGetErrorString(e), cudaGetErrorString(e2), h[1], h[0]);
      cudaFree(d);
    }
  }
  return 0;
}
