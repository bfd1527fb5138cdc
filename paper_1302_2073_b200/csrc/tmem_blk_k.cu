// tmem_blk_k.cu — the frame-blocking instances of k_tmem (prost_push_many),
// in their own translation unit so the library builds in parallel.
#include "tmem_launch.cuh"

namespace prost_ops {

TmOps pick_tmem_blocking(int K, bool half) { return pick_instance<true, false>(K, half); }

}  // namespace prost_ops
