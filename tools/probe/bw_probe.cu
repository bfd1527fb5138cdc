// Probe: on-chip and per-SM HBM bandwidths that bound the frame kernel.
//   (1) TMEM read throughput per SM (tcgen05.ld.32x32b.xN, B loads per wait)
//   (2) shared-memory read throughput per SM (16-byte loads)
//   (3) global-load bandwidth with `ctas` SMs active, T threads, L float4 per thread in flight
//   (4) the same with 1-D bulk copies (cp.async.bulk, TMA engine) into a shared ring
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/probe/bw_probe tools/probe/bw_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int N, int B>
__global__ void __launch_bounds__(512, 1) k_tmem_rd(int iters, unsigned long long* cyc, float* sink) {
  __shared__ unsigned tb;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tb)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const unsigned ta = tb + ((unsigned)(32 * (warp & 3)) << 16) + (unsigned)((warp >> 2) * 128);
  float acc = 0.f;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c0 = 0; c0 < 128; c0 += N * B) {
      float v[B][N];
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const unsigned a = ta + c0 + b * N;
        if constexpr (N == 16)
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                       : "=f"(v[b][0]), "=f"(v[b][1]), "=f"(v[b][2]), "=f"(v[b][3]), "=f"(v[b][4]), "=f"(v[b][5]), "=f"(v[b][6]), "=f"(v[b][7]),
                         "=f"(v[b][8]), "=f"(v[b][9]), "=f"(v[b][10]), "=f"(v[b][11]), "=f"(v[b][12]), "=f"(v[b][13]), "=f"(v[b][14]), "=f"(v[b][15])
                       : "r"(a));
        else
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                       : "=f"(v[b][0]), "=f"(v[b][1]), "=f"(v[b][2]), "=f"(v[b][3]) : "r"(a));
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int b = 0; b < B; ++b)
#pragma unroll
        for (int j = 0; j < N; ++j) acc += v[b][j];
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 1.2345f) sink[threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

__global__ void __launch_bounds__(512, 1) k_smem_rd(int iters, unsigned long long* cyc, float* sink) {
  extern __shared__ float4 sm4[];
  const int n4 = 200 * 1024 / 16;
  for (int i = threadIdx.x; i < n4; i += blockDim.x) sm4[i] = make_float4(i, 1, 2, 3);
  __syncthreads();
  float acc = 0.f;
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
    for (int i = threadIdx.x; i < n4; i += blockDim.x) {
      const float4 v = sm4[i];
      acc += v.x + v.y + v.z + v.w;
    }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 1.2345f) sink[threadIdx.x] = acc;
}

// each thread: L independent float4 streaming loads per step, grid-strided over `bytes`
template <int L>
__global__ void k_gld(const float4* __restrict__ src, size_t n4, int reps, float* sink) {
  float acc = 0.f;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i + (L - 1) * stride < n4; i += L * stride) {
      float4 v[L];
#pragma unroll
      for (int l = 0; l < L; ++l) v[l] = __ldcs(src + i + l * stride);
#pragma unroll
      for (int l = 0; l < L; ++l) acc += v[l].x + v[l].y + v[l].z + v[l].w;
    }
  if (acc == 1.2345f) sink[threadIdx.x] = acc;
}

// one thread per CTA drives a ring of `stages` x `chunk` byte bulk copies
__global__ void __launch_bounds__(128, 1) k_bulk(const char* __restrict__ src, size_t bytes, int chunk, int stages, float* sink) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) unsigned long long bar[16];
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t per = bytes / gridDim.x / chunk * chunk;
  const char* base = src + (size_t)blockIdx.x * per;
  const int nch = (int)(per / chunk);
  float acc = 0.f;
  if (threadIdx.x == 0) {
    unsigned phase[16] = {0};
    for (int c = 0; c < nch + stages; ++c) {
      const int s = c % stages;
      if (c >= stages) {  // wait for chunk c - stages
        unsigned done = 0;
        while (!done)
          asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                       : "=r"(done) : "r"(smem_u32(&bar[s])), "r"(phase[s]) : "memory");
        phase[s] ^= 1u;
        acc += ((float*)(ring + (size_t)s * chunk))[0];
      }
      if (c < nch) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(chunk) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(smem_u32(ring + (size_t)s * chunk)), "l"(base + (size_t)c * chunk), "r"(chunk), "r"(smem_u32(&bar[s])) : "memory");
      }
    }
  }
  if (acc == 1.2345f) sink[threadIdx.x] = acc;
}

int main() {
  unsigned long long* cyc;
  float* sink;
  CK(cudaMalloc(&cyc, 1024 * 8));
  CK(cudaMalloc(&sink, 4096));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  unsigned long long h[1024];
  auto rep = [&](const char* what, double bytes_per_cta, int ctas) {
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h, cyc, ctas * 8, cudaMemcpyDeviceToHost));
    double mx = 0, sum = 0;
    for (int i = 0; i < ctas; ++i) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
    printf("%-34s %7.1f B/clk/SM (mean cta), %7.1f (slowest)\n", what, bytes_per_cta / (sum / ctas), bytes_per_cta / mx);
  };
  const int it = 200;
  k_tmem_rd<16, 1><<<sms, 512>>>(it, cyc, sink); rep("tmem ld x16, wait each", 512.0 * 128 * 4 * it, sms);
  k_tmem_rd<16, 2><<<sms, 512>>>(it, cyc, sink); rep("tmem ld x16, 2 per wait", 512.0 * 128 * 4 * it, sms);
  k_tmem_rd<16, 4><<<sms, 512>>>(it, cyc, sink); rep("tmem ld x16, 4 per wait", 512.0 * 128 * 4 * it, sms);
  k_tmem_rd<4, 4><<<sms, 512>>>(it, cyc, sink); rep("tmem ld x4, 4 per wait", 512.0 * 128 * 4 * it, sms);
  k_tmem_rd<16, 4><<<1, 512>>>(it, cyc, sink); rep("tmem ld x16, 4 per wait (1 SM)", 512.0 * 128 * 4 * it, 1);
  CK(cudaFuncSetAttribute(k_smem_rd, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  k_smem_rd<<<sms, 512, 200 * 1024>>>(50, cyc, sink); rep("smem ld.128", 200.0 * 1024 * 50, sms);

  const size_t bytes = (size_t)4 << 30;
  float4* src;
  CK(cudaMalloc(&src, bytes));
  CK(cudaMemset(src, 0, bytes));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  int clk;
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  for (int ctas : {sms, sms / 2, sms / 4, 16}) {
    for (int thr : {256, 512}) {
      auto run = [&](auto kern, const char* nm) {
        kern<<<ctas, thr>>>(src, bytes / 16, 1, sink);
        CK(cudaEventRecord(e0));
        kern<<<ctas, thr>>>(src, bytes / 16, 2, sink);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        const double gbs = 2.0 * bytes / (ms * 1e-3) / 1e9;
        printf("gld %-8s ctas %3d thr %3d: %7.0f GB/s total, %6.1f GB/s per SM\n", nm, ctas, thr, gbs, gbs / ctas);
      };
      run(k_gld<4>, "L=4");
      run(k_gld<15>, "L=15");
    }
    for (int chunk : {8192, 16384}) {
      for (int stages : {4, 8, 12}) {
        const int smem = chunk * stages;
        if (smem > 220 * 1024) continue;
        CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        k_bulk<<<ctas, 128, smem>>>((const char*)src, bytes, chunk, stages, sink);
        CK(cudaEventRecord(e0));
        k_bulk<<<ctas, 128, smem>>>((const char*)src, bytes, chunk, stages, sink);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        const double gbs = (double)bytes / (ms * 1e-3) / 1e9;
        printf("bulk ctas %3d chunk %5d x %2d stages (%3d KB in flight): %7.0f GB/s total, %6.1f GB/s per SM\n",
               ctas, chunk, stages, smem / 1024, gbs, gbs / ctas);
      }
    }
  }
  CK(cudaGetLastError());
  return 0;
}
