// pf_aux.cuh -- auxiliary kernels (init, labeling, energies, validation).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "pf_kernels.cuh"

namespace pf {

struct EnergyArgs {
    const float *u;   // current u, plane 0 (the plane above the slab must be current for the primal)
    int ulog;         // 1: u holds log2 u (pseudo-flow state), 0: u itself (explicit-flow ALM)
    const float *q;   // current q, plane 0 (the plane below must be current for the dual)
    const void *D;    // fp32, or bf16 when d_bf16
    const float *S;
    int d_bf16;
    int nx, ny, pitch, nzl, zg0, nzg, ndim;
    int NI, NL, NV;
    int NF;      // flow-carrying nodes (positions 0..NF-1)
    int model;   // 0: DAG (dense weights), 1: Ishikawa chain
    int s_kind, cap;
    GraphConst g;
};

constexpr int kEnergyBlocks = 592;

struct NodeWeights {
    float W[16];   // W_(v, B) per end label B (0: B not below v)
};

cudaError_t launch_fill(float *p, int64_t n, float v, cudaStream_t st);
cudaError_t launch_node_labeling(const float *u, float *out, const NodeWeights &w, int NL, int nx, int ny, int pitch,
                                 int64_t nz, int ulog, cudaStream_t st);
cudaError_t launch_argmax(const float *u, uint8_t *out, int NL, int nx, int ny, int pitch, int64_t nz, int ulog,
                          cudaStream_t st);
cudaError_t launch_export_u(const float *u, float *out, int NL, int nx, int ny, int pitch, int64_t nz, int ulog,
                            cudaStream_t st);
cudaError_t launch_log2_inplace(float *p, int64_t n, cudaStream_t st);
cudaError_t launch_f32_to_bf16(const float *src, uint16_t *dst, int64_t n, cudaStream_t st);
cudaError_t launch_check_nonneg(const float *p, int64_t n, unsigned int *flag, cudaStream_t st);
cudaError_t launch_energy(const EnergyArgs &a, double *partial, int nblocks, double *out, cudaStream_t st);

}  // namespace pf
