// Instantiations of the cluster-split Potts kernel (pf_cluster.cuh): even K = 10..16, D fp32 / bf16,
// lambda = log2 u stored as fp32 or (D fp32 only) binary16.
#include "pf_cluster.cuh"

namespace pf {

#define PF_CLUSTER_INST(NLV, DBFV, UHV)                                                                 \
    template __global__ void pf_iter_cluster<NLV, 8, DBFV, UHV>(const __grid_constant__ StagedArgs a);  \
    static_assert(ClusterLayout<NLV, 8, DBFV>::bytes(1) + 256 <= 227 * 1024, "cluster kernel smem");
#define PF_CLUSTER_INST3(NLV) PF_CLUSTER_INST(NLV, 0, 0) PF_CLUSTER_INST(NLV, 1, 0) PF_CLUSTER_INST(NLV, 0, 1)
PF_CLUSTER_INST3(10)
PF_CLUSTER_INST3(12)
PF_CLUSTER_INST3(14)
PF_CLUSTER_INST3(16)

bool cluster_kernel_lookup(int NL, int DBF, int UH, StagedKernelInfo *info) {
#define PF_CLUSTER_CASE(NLV, DBFV, UHV)                                                                 \
    if (NL == NLV && DBF == DBFV && UH == UHV) {                                                        \
        info->func = (const void *)&pf_iter_cluster<NLV, 8, DBFV, UHV>;                                 \
        info->threads = 32 * (8 + 2);                                                                   \
        info->smem_bytes = ClusterLayout<NLV, 8, DBFV>::bytes(0);                                       \
        info->tile_y = 8;                                                                               \
        info->ostage = 1;                                                                               \
        info->groups = 1;                                                                               \
        info->s_slots = 4;                                                                              \
        return true;                                                                                    \
    }
#define PF_CLUSTER_CASE3(NLV) PF_CLUSTER_CASE(NLV, 0, 0) PF_CLUSTER_CASE(NLV, 1, 0) PF_CLUSTER_CASE(NLV, 0, 1)
    PF_CLUSTER_CASE3(10)
    PF_CLUSTER_CASE3(12)
    PF_CLUSTER_CASE3(14)
    PF_CLUSTER_CASE3(16)
    return false;
}

}  // namespace pf
