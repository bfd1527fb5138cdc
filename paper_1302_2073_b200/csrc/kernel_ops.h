// kernel_ops.h — launch interfaces of the resident frame kernels, each
// instantiated in its own translation unit (resident_k.cu, tmem_k.cu) so the
// library builds in parallel.
#pragma once

#include <cuda_runtime.h>

#include "prost_kernels.cuh"

namespace prost {
struct RArgs;
}

namespace prost_ops {
using prost::Args;
using prost::RArgs;

// Register-resident frame kernel (prost_resident.cuh), fp32, one channel.
struct ResOps {
  cudaError_t (*launch)(const Args&, const RArgs&, int nt, size_t smem, cudaStream_t st);
  cudaError_t (*prepare)(size_t smem);
  int (*occupancy)(int nt, size_t smem);
  size_t (*smem)(int qpc, int nwarp);
  int ntmax;
};
ResOps pick_resident(int K, bool half);

// TMEM-resident frame kernel (prost_tmem.cuh), fp32, 1 or 3 channels, k <= 20,
// with NG slot groups per CTA.
struct TmOps {
  cudaError_t (*launch)(const Args&, const RArgs&, size_t smem, cudaStream_t st);
  cudaError_t (*prepare)(size_t smem);
  int (*occupancy)(size_t smem);
  size_t (*smem)(int qpc);
  int qt;  // row groups per thread held in TMEM
  int ng;  // slot groups per CTA
  void (*describe)();
  int (*clusters)(size_t smem, int cluster);  // cluster instances: clusters that fit the chip at once
};
// blk: the frame-blocking instance; cl: one thread-block cluster per team
TmOps pick_tmem(int K, bool half, int ng, bool blk = false, bool cl = false);

}  // namespace prost_ops
