// tmem_k.cu — the single-frame instances of the TMEM-resident frame kernel
// k_tmem (prost_tmem.cuh) and the TmOps selector (kernel_ops.h).
#include "tmem_launch.cuh"

namespace prost_ops {

TmOps pick_tmem_blocking(int K, bool half);  // tmem_blk_k.cu
TmOps pick_tmem_cluster(int K, bool half);   // tmem_cl_k.cu

TmOps pick_tmem(int K, bool half, int ng, bool blk, bool cl) {
  // NG = 2 (two streams per CTA in parallel warp groups) measured slower on
  // C3: the launcher keeps the template, only NG = 1 is built
  if (ng != 1) return TmOps{};
  if (cl) return blk ? TmOps{} : pick_tmem_cluster(K, half);
  return blk ? pick_tmem_blocking(K, half) : pick_instance<false, false>(K, half);
}

}  // namespace prost_ops
