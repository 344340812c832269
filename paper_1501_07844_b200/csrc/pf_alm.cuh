// pf_alm.cuh -- explicit-flow augmented-Lagrangian Potts solver (comparison arm); see pf_alm.cu.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pf {

struct AlmArgs {
    const float *q_in;   // flows read by pass 1 (plane 0 of the ping-pong buffer)
    float *q_out;        // flows written by pass 1, read by pass 2
    float *u, *p, *pS;   // multipliers, sink flows, source flow (updated in place by pass 2)
    const void *D;       // data terms (fp32, or bf16 when d_bf16)
    const float *S;      // capacity field (shared or per label); null for scalars
    int d_bf16, s_per_node, cap, check;
    int nx, ny, nz, pitch, NL, zchunk;
    float c, inv_c, tau;
    float s[16];         // per-label capacity scalar / shared-field factor
    unsigned int *resid_bits;
};

cudaError_t launch_alm_init(const AlmArgs &a, cudaStream_t st);
cudaError_t launch_alm_iteration(const AlmArgs &a, cudaStream_t st);

}  // namespace pf
