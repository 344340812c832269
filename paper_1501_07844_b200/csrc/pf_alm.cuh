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
    int zchunk2;         // z-chunk of pass 2 (short: one thread per voxel column segment)
    float c, inv_c, tau;
    float s[16];         // per-label capacity scalar / shared-field factor
    unsigned int *resid_bits;
    // DAG / HMF (Eq. 10-11): positions 0..NI-1 internal (topological), NI..NV-1 end labels; u of the
    // internal nodes in u_int [z][NI][y][pitch]; p of every position [z][NV][y][pitch], p_S in pS;
    // W[0][j] = weight of S -> position j, W[1 + i][j] = weight of position i -> position j (0: no edge)
    int dag, NI, NV;
    float *u_int;
    float W[17][16];
};

cudaError_t launch_alm_init(const AlmArgs &a, cudaStream_t st);
cudaError_t launch_alm_iteration(const AlmArgs &a, cudaStream_t st);

}  // namespace pf
