// tmem_blk_k.cu — the frame-blocking instances of k_tmem (prost_push_many),
// in their own translation unit so the library builds in parallel.
#include <cstdio>

#include "kernel_ops.h"
#include "prost_tmem.cuh"

using namespace prost;

namespace prost_ops {



template <int K, int PM, int NG, bool BLK>
struct Tm {
  static cudaError_t launch(const Args& a, const RArgs& ra, size_t smem, cudaStream_t st) {
    Args aa = a;
    RArgs rr = ra;
    void* args[] = {&aa, &rr};
    if (TM_CPS == 1)
      return cudaLaunchCooperativeKernel((const void*)k_tmem<K, PM, NG, BLK>, dim3(ra.T * ra.G), dim3(TM_NT),
                                         args, smem, st);
    // The occupancy calculator reports one CTA per SM for any kernel that
    // allocates tensor memory, so a cooperative launch of TM_CPS CTAs per SM is
    // refused; the hardware co-schedules them (tools/probe/coresid_probe.cu),
    // and the grid is sized to the chip, so every CTA is resident at once.
    return cudaLaunchKernel((const void*)k_tmem<K, PM, NG, BLK>, dim3(ra.T * ra.G), dim3(TM_NT), args, smem, st);
  }
  static cudaError_t prepare(size_t smem) {
    return cudaFuncSetAttribute(k_tmem<K, PM, NG, BLK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  static int occupancy(size_t smem) {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_tmem<K, PM, NG, BLK>, TM_NT, smem) != cudaSuccess)
      return 0;
    return nb;
  }
  static size_t smem(int qpc) { return tmem_smem<K, NG>(qpc); }
  static void describe() {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, k_tmem<K, PM, NG, BLK>);
    int nb0 = -1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb0, k_tmem<K, PM, NG, BLK>, TM_NT, 0);
    fprintf(stderr, "prost: k_tmem<%d, NG=%d> regs %d local %zu static smem %zu max threads %d; occupancy(smem 0) %d\n",
            K, NG, fa.numRegs, fa.localSizeBytes, fa.sharedSizeBytes, fa.maxThreadsPerBlock, nb0);
  }
  static TmOps ops() { return TmOps{&launch, &prepare, &occupancy, &smem, TmemGeom<K>::QT, NG, &describe}; }
};

template <bool BLK>
TmOps pick_blk(int K, bool half) {
  switch (K) {
    case 4: return half ? Tm<4, PM_HALF, 1, BLK>::ops() : Tm<4, PM_ANY, 1, BLK>::ops();
    case 8: return half ? Tm<8, PM_HALF, 1, BLK>::ops() : Tm<8, PM_ANY, 1, BLK>::ops();
    case 15: return half ? Tm<15, PM_HALF, 1, BLK>::ops() : Tm<15, PM_ANY, 1, BLK>::ops();
    case 16: return half ? Tm<16, PM_HALF, 1, BLK>::ops() : Tm<16, PM_ANY, 1, BLK>::ops();
    case 20: return half ? Tm<20, PM_HALF, 1, BLK>::ops() : Tm<20, PM_ANY, 1, BLK>::ops();
    default: return TmOps{nullptr, nullptr, nullptr, nullptr, 0, 1, nullptr};
  }
}

TmOps pick_tmem_blocking(int K, bool half) { return pick_blk<true>(K, half); }

}  // namespace prost_ops
