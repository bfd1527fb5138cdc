// resident_k.cu — instances of the register-resident frame kernel k_resident
// (prost_resident.cuh) and their launchers (kernel_ops.h).
#include "kernel_ops.h"
#include "prost_resident.cuh"

using namespace prost;

namespace prost_ops {



template <int K, int NTMAX, int PM>
struct Res {
  static cudaError_t launch(const Args& a, const RArgs& ra, int nt, size_t smem, cudaStream_t st) {
    Args aa = a;
    RArgs rr = ra;
    void* args[] = {&aa, &rr};
    return cudaLaunchCooperativeKernel((const void*)k_resident<K, NTMAX, PM>, dim3(ra.T * ra.G),
                                       dim3(nt), args, smem, st);
  }
  static cudaError_t prepare(size_t smem) {
    return cudaFuncSetAttribute(k_resident<K, NTMAX, PM>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  static int occupancy(int nt, size_t smem) {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_resident<K, NTMAX, PM>, nt, smem) !=
        cudaSuccess)
      return 0;
    return nb;
  }
  static size_t smem(int qpc, int nwarp) { return resident_smem<K>(qpc, nwarp); }
  static ResOps ops() { return ResOps{&launch, &prepare, &occupancy, &smem, NTMAX}; }
};

// p = 0.5 (every BASELINE config) gets its own instance with the two-RSQ
// penalty; other exponents use the runtime-dispatched instance.
// 512 threads x 128 registers for k <= 16: the 60 basis registers of a 4-row
// group plus the CG working set (ptxas budgets registers per 128-thread granule).
ResOps pick_resident(int K, bool half) {
  switch (K) {
    case 4: return half ? Res<4, 768, PM_HALF>::ops() : Res<4, 768, PM_ANY>::ops();
    case 8: return half ? Res<8, 768, PM_HALF>::ops() : Res<8, 768, PM_ANY>::ops();
    case 15: return half ? Res<15, 512, PM_HALF>::ops() : Res<15, 512, PM_ANY>::ops();
    case 16: return half ? Res<16, 512, PM_HALF>::ops() : Res<16, 512, PM_ANY>::ops();
    default: return ResOps{nullptr, nullptr, nullptr, nullptr, 0};
  }
}

}  // namespace prost_ops
