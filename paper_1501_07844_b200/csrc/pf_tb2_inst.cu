// Instantiations of the two-iterations-per-pass kernel (pf_tb2.cuh): Potts K = 2..4, l2 / l-inf capacities.
#include "pf_tb2.cuh"

namespace pf {

#define PF_TB2_INST(KV, CAPV)                                                                           \
    template __global__ void pf_iter_tb2<KV, 8, CAPV>(const __grid_constant__ StagedArgs a);            \
    static_assert(TB2Layout<KV, 8>::bytes() + 256 <= 227 * 1024, "tb2 kernel smem");
PF_TB2_INST(2, 0)
PF_TB2_INST(2, 1)
PF_TB2_INST(3, 0)
PF_TB2_INST(3, 1)
PF_TB2_INST(4, 0)
PF_TB2_INST(4, 1)

bool tb2_kernel_lookup(int K, int CAP, StagedKernelInfo *info) {
#define PF_TB2_CASE(KV, CAPV)                                                                           \
    if (K == KV && CAP == CAPV) {                                                                       \
        info->func = (const void *)&pf_iter_tb2<KV, 8, CAPV>;                                           \
        info->threads = TB2Layout<KV, 8>::kThreads;                                                     \
        info->smem_bytes = TB2Layout<KV, 8>::bytes();                                                   \
        info->tile_y = 8;                                                                               \
        info->ostage = 1;                                                                               \
        info->groups = 1;                                                                               \
        info->s_slots = 0;                                                                              \
        return true;                                                                                    \
    }
    PF_TB2_CASE(2, 0)
    PF_TB2_CASE(2, 1)
    PF_TB2_CASE(3, 0)
    PF_TB2_CASE(3, 1)
    PF_TB2_CASE(4, 0)
    PF_TB2_CASE(4, 1)
    return false;
}

}  // namespace pf
