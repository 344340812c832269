// pf_aux.cuh -- auxiliary kernels (init, labeling, energies, validation).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "pf_kernels.cuh"

namespace pf {

struct EnergyArgs {
    const void *u;    // current label state, plane 0 (the plane above the slab must be current for the primal)
    int ufmt;         // 0: u itself fp32 (explicit-flow ALM), 1: log2 u fp32, 2: log2 u binary16 (u_half)
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
    const GraphWide *gw;   // non-null: the graph is beyond the compiled set (GraphConst unused), device memory
};

constexpr int kEnergyBlocks = 592;

struct NodeWeights {
    float W[16];   // W_(v, B) per end label B (0: B not below v)
};

cudaError_t launch_fill(float *p, int64_t n, float v, cudaStream_t st);
cudaError_t launch_node_labeling(const void *u, float *out, const NodeWeights &w, int NL, int nx, int ny, int pitch,
                                 int64_t nz, int ufmt, cudaStream_t st);
cudaError_t launch_argmax(const void *u, uint8_t *out, int NL, int nx, int ny, int pitch, int64_t nz, int ufmt,
                          cudaStream_t st);
cudaError_t launch_export_u(const void *u, float *out, int NL, int nx, int ny, int pitch, int64_t nz, int ufmt, int raw,
                            cudaStream_t st);
cudaError_t launch_import_u(const float *in, void *u, int NL, int nx, int ny, int pitch, int64_t nz, int ufmt,
                            int linear, cudaStream_t st);
cudaError_t launch_fill_half(void *p, int64_t n, float v, cudaStream_t st);
cudaError_t launch_f32_to_bf16(const float *src, uint16_t *dst, int64_t n, cudaStream_t st);
cudaError_t launch_check_nonneg(const float *p, int64_t n, unsigned int *flag, cudaStream_t st);
cudaError_t launch_energy(const EnergyArgs &a, double *partial, int nblocks, double *out, cudaStream_t st);

}  // namespace pf
