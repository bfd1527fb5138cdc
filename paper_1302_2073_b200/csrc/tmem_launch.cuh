// tmem_launch.cuh — launchers of the k_tmem instances (kernel_ops.h TmOps),
// shared by the translation units that instantiate them (tmem_k.cu: one
// frame per launch; tmem_blk_k.cu: frame blocking; tmem_cl_k.cu: a team per
// thread-block cluster).
#pragma once

#include <cstdio>
#include <cstdlib>

#include "kernel_ops.h"
#include "prost_tmem.cuh"

namespace prost_ops {

using namespace prost;

inline bool tm_pdl() {
  static const bool on = [] {
    const char* e = getenv("PROST_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <int K, int PM, int NG, bool BLK, bool CL>
struct Tm {
  static constexpr auto kernel = k_tmem<K, PM, NG, BLK, CL>;
  // the instance with the timing counters (RArgs.prof set: the bench's counters pass)
  static constexpr auto kernel_prof = k_tmem<K, PM, NG, BLK, CL, true>;
  static cudaError_t launch(const Args& a, const RArgs& ra, size_t smem, cudaStream_t st) {
    Args aa = a;
    RArgs rr = ra;
    void* args[] = {&aa, &rr};
    const void* kf = ra.prof ? (const void*)kernel_prof : (const void*)kernel;
    if constexpr (CL) {
      // one cluster per team: its CTAs are co-scheduled by construction and
      // teams never wait for each other, so no cooperative launch is needed
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(ra.T * ra.G);
      cfg.blockDim = dim3(TM_NT);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      // programmatic dependent launch: the next frame's clusters are placed
      // on free SMs while this one drains and wait in pdl_enter
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = ra.G;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[1].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = (ra.prof || !tm_pdl()) ? 1 : 2;
      return cudaLaunchKernelExC(&cfg, kf, args);
    }
    if (TM_CPS == 1)
      return cudaLaunchCooperativeKernel(kf, dim3(ra.T * ra.G), dim3(TM_NT), args, smem, st);
    // The occupancy calculator reports one CTA per SM for any kernel that
    // allocates tensor memory, so a cooperative launch of TM_CPS CTAs per SM is
    // refused; the hardware co-schedules them (tools/probe/coresid_probe.cu),
    // and the grid is sized to the chip, so every CTA is resident at once.
    return cudaLaunchKernel(kf, dim3(ra.T * ra.G), dim3(TM_NT), args, smem, st);
  }
  static cudaError_t prepare(size_t smem) {
    cudaError_t e = cudaSuccess;
    for (const auto kk : {kernel, kernel_prof}) {
      if (e == cudaSuccess) e = cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (CL && e == cudaSuccess) e = cudaFuncSetAttribute(kk, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    }
    return e;
  }
  // CTAs per SM; cluster instances: clusters of `cluster` CTAs that fit the chip at once
  static int occupancy(size_t smem) {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, TM_NT, smem) != cudaSuccess) return 0;
    return nb;
  }
  static int clusters(size_t smem, int cluster) {
    if (!CL) return 0;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cluster);
    cfg.blockDim = dim3(TM_NT);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, (const void*)kernel, &cfg) != cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    return n;
  }
  static size_t smem(int qpc) { return tmem_smem<K, NG>(qpc); }
  static void describe() {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, kernel);
    int nb0 = -1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb0, kernel, TM_NT, 0);
    fprintf(stderr,
            "prost: k_tmem<%d, NG=%d, BLK=%d, CL=%d> regs %d local %zu static smem %zu max threads %d; "
            "occupancy(smem 0) %d\n",
            K, NG, (int)BLK, (int)CL, fa.numRegs, fa.localSizeBytes, fa.sharedSizeBytes, fa.maxThreadsPerBlock,
            nb0);
  }
  static TmOps ops() {
    return TmOps{&launch, &prepare, &occupancy, &smem, TmemGeom<K>::QT, NG, &describe, &clusters};
  }
};

template <bool BLK, bool CL>
TmOps pick_instance(int K, bool half) {
  switch (K) {
    case 4: return half ? Tm<4, PM_HALF, 1, BLK, CL>::ops() : Tm<4, PM_ANY, 1, BLK, CL>::ops();
    case 8: return half ? Tm<8, PM_HALF, 1, BLK, CL>::ops() : Tm<8, PM_ANY, 1, BLK, CL>::ops();
    case 15: return half ? Tm<15, PM_HALF, 1, BLK, CL>::ops() : Tm<15, PM_ANY, 1, BLK, CL>::ops();
    case 16: return half ? Tm<16, PM_HALF, 1, BLK, CL>::ops() : Tm<16, PM_ANY, 1, BLK, CL>::ops();
    case 20: return half ? Tm<20, PM_HALF, 1, BLK, CL>::ops() : Tm<20, PM_ANY, 1, BLK, CL>::ops();
    default: return TmOps{};
  }
}

}  // namespace prost_ops
