// Instantiations of the cluster-split Potts kernel (pf_cluster.cuh): even K = 10..16, D fp32 / bf16.
#include "pf_cluster.cuh"

namespace pf {

#define PF_CLUSTER_INST(NLV, DBFV)                                                                      \
    template __global__ void pf_iter_cluster<NLV, 8, DBFV>(const __grid_constant__ StagedArgs a);       \
    static_assert(ClusterLayout<NLV, 8, DBFV>::bytes(1) + 256 <= 227 * 1024, "cluster kernel smem");
PF_CLUSTER_INST(10, 0)
PF_CLUSTER_INST(10, 1)
PF_CLUSTER_INST(12, 0)
PF_CLUSTER_INST(12, 1)
PF_CLUSTER_INST(14, 0)
PF_CLUSTER_INST(14, 1)
PF_CLUSTER_INST(16, 0)
PF_CLUSTER_INST(16, 1)

bool cluster_kernel_lookup(int NL, int DBF, StagedKernelInfo *info) {
#define PF_CLUSTER_CASE(NLV, DBFV)                                                                      \
    if (NL == NLV && DBF == DBFV) {                                                                     \
        info->func = (const void *)&pf_iter_cluster<NLV, 8, DBFV>;                                      \
        info->threads = 32 * (8 + 2);                                                                   \
        info->smem_bytes = ClusterLayout<NLV, 8, DBFV>::bytes(0);                                       \
        info->tile_y = 8;                                                                               \
        info->ostage = 1;                                                                               \
        info->groups = 1;                                                                               \
        return true;                                                                                    \
    }
    PF_CLUSTER_CASE(10, 0)
    PF_CLUSTER_CASE(10, 1)
    PF_CLUSTER_CASE(12, 0)
    PF_CLUSTER_CASE(12, 1)
    PF_CLUSTER_CASE(14, 0)
    PF_CLUSTER_CASE(14, 1)
    PF_CLUSTER_CASE(16, 0)
    PF_CLUSTER_CASE(16, 1)
    return false;
}

}  // namespace pf
