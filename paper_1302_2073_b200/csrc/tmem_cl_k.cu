// tmem_cl_k.cu — the cluster instances of k_tmem: one thread-block cluster
// per team, team sums over DSMEM and the hardware cluster barrier (used when
// every team fits one cluster and the clusters fit the chip: the one-stream
// latency layout).
#include "tmem_launch.cuh"

namespace prost_ops {

TmOps pick_tmem_cluster(int K, bool half) { return pick_instance<false, true>(K, half); }

}  // namespace prost_ops
