// pf_kernels.cuh -- sm_100a kernels of the pseudo-flow iteration (arXiv 1501.07844).
//
// One launch of pf_iter_kernel performs one pass of the while-loop body of
// Algorithm 1 or Algorithm 2 over the whole
// (slab of the) volume, fused into a single HBM pass:
//
//   a1  div q_v(x)          backward differences of the OLD flows
//   a2  d_v = div q_v (+D_L), top-down pushes in O
//   a3  u~_L = u_L exp(-(d_L - m)/c), a = sum u~, u' = u~/a          (R1)
//       on the stored log2 state lambda = log2 u (label_update, pf_math.cuh; reading R18)
//   a4  M_L = u~_L, bottom-up pushes in O^-1
//   a5  q^ = q_v - c tau nabla M_v                                  (Eq. 8, Eq. 16)
//   a6  q' = Proj_{|q| <= S_v}(q^)                                   (R5, R14)
//   a7  u', q' written to the other half of the ping-pong pair
//   a8  optional residual max|u' - u| (fused, one atomic per warp)
//
// Work decomposition ("2.5-D z-march"): a CTA owns a 32 x TY tile of (x, y)
// columns and walks a chunk of z planes.  For every plane p it computes the
// unnormalised masses M(p) of its tile plus a +1 halo in x and y (two extra
// warps) into a 3-deep shared-memory ring, writes u'(p), then finishes the flow
// step of plane p-1, which needs M(p-1) at x, x+e_x, x+e_y and M(p) at x.  Each
// voxel's state is read from HBM once per iteration; the +1 halo columns/rows are
// re-read from L2.  Node positions: 0..NI-1 internal nodes in topological order,
// NI..NV-1 end labels in node-id order (a topological order, since end labels
// have no children).
//
// Layouts (internal, per z-plane contiguous so a plane of every label is one
// chunk for the halo exchange):  u (stored as log2 u), D: [z][l][y][x];  q: [z][k][v][y][x];
// S field: [z][y][x] (shared) or [z][v][y][x] (per node).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pf {

constexpr int kMaxNodes = 16;     // non-source nodes handled by the compiled kernels
constexpr int kMaxInternal = 4;   // internal (non-end) nodes
constexpr int kTX = 32;

}  // namespace pf
#include "pf_math.cuh"
namespace pf {

struct GraphConst {
    float w[kMaxInternal][kMaxNodes];  // w[i][j]: weight of edge (position i -> position j); 0 = no edge; S excluded
    float s[kMaxNodes];                // capacity scalar per position (PF_S_SCALAR_PER_NODE)
};

struct IterArgs {
    const float *u_in;
    float *u_out;
    const float *q_in;
    float *q_out;
    const void *D;    // fp32, or bf16 when d_bf16
    int d_bf16;
    const float *S;   // null when capacities are scalars
    int nx, ny, nzl;  // local extents
    int pitch;        // row pitch in elements (>= nx, multiple of 4 for TMA)
    int zg0, nzg;     // global z of local plane 0, global nz
    int zchunk;
    int s_kind;       // 0 scalar per node, 1 shared field, 2 field per node
    int cap;          // 0 l2, 1 box
    int shift;        // 0 min, 1 none
    int check;        // compute the residual this launch
    float inv_c;
    float ctau;
    unsigned int *resid_bits;          // max |u' - u| as float bits (non-negative)
    unsigned long long *err_voxel;     // min global linear voxel index with a(x) <= 0 / non-finite
    GraphConst g;
};

__device__ __forceinline__ float ldg(const float *p) { return __ldg(p); }

template <int NI, int NL, int TY, int MODEL>
struct IterSmem {
    static constexpr int NV = Model<MODEL, NI, NL>::NF;
    static constexpr int kPlane = NV * (TY + 1) * (kTX + 1);
    static constexpr int kBytes = 3 * kPlane * (int)sizeof(float);
};

template <int NV /* flow nodes */, int TY, int CAP>
__device__ __forceinline__ void flow_out_global(const IterArgs &a, const float *Mz, const float *Mp, bool has_z,
                                                int sme, int x, int y, int zg, int64_t P, const float *qb, float *qo,
                                                const float *Sb) {
    constexpr int RS = kTX + 1, PS = (TY + 1) * RS;
    const bool gxv = x < a.nx - 1, gyv = y < a.ny - 1, gzv = has_z && (zg < a.nzg - 1);
    const int Pi = (int)P;  // channel stride fits 32 bits (an x-y plane has < 2^31 / 48 voxels)
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        const float mc = Mz[v * PS + sme];
        const float gx = gxv ? Mz[v * PS + sme + 1] - mc : 0.f;
        const float gy = gyv ? Mz[v * PS + sme + RS] - mc : 0.f;
        const float gz = gzv ? Mp[v * PS + sme] - mc : 0.f;
        float hx = ldg(qb + v * P), hy = ldg(qb + (NV + v) * P), hz = ldg(qb + (2 * NV + v) * P);
        const float sv = a.s_kind == 0 ? a.g.s[v] : (a.s_kind == 1 ? ldg(Sb) * a.g.s[v] : ldg(Sb + v * P));
        flow_step<CAP>(a.ctau, gx, gy, gz, sv, hx, hy, hz);
        st_stream(qo + v * Pi, hx);
        st_stream(qo + (NV + v) * Pi, hy);
        st_stream(qo + (2 * NV + v) * Pi, hz);
    }
}

template <int NI, int NL, int TY, int MODEL>
__global__ void __launch_bounds__(32 * TY + 64) pf_iter_kernel(const IterArgs a) {
    constexpr int NV = Model<MODEL, NI, NL>::NF;  // node loops run over the flow-carrying nodes
    constexpr int RS = kTX + 1;              // smem row stride
    constexpr int PS = (TY + 1) * RS;        // smem per-node plane stride
    constexpr int RING = NV * PS;            // smem per ring slot
    extern __shared__ float Ms[];            // [3][NV][TY+1][33]

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool is_main = warp < TY;
    int lx, ly;
    if (is_main) {
        lx = lane; ly = warp;
    } else {
        const int h = (warp - TY) * 32 + lane;
        if (h < kTX) { lx = h; ly = TY; }
        else if (h < kTX + TY) { lx = kTX; ly = h - kTX; }
        else { lx = -1; ly = 0; }
    }
    const int x = blockIdx.x * kTX + lx, y = blockIdx.y * TY + ly;
    const bool active = (lx >= 0) && (x < a.nx) && (y < a.ny);
    const int64_t P = (int64_t)a.pitch * a.ny;
    const int pix = active ? y * a.pitch + x : 0;
    const int zc0 = blockIdx.z * a.zchunk;
    const int zc1 = min(zc0 + a.zchunk, a.nzl);
    const bool has_above = (a.zg0 + zc1) < a.nzg;
    const int64_t ups = (int64_t)NL * P;
    const int64_t qps = (int64_t)3 * NV * P;
    const int sme = ly * RS + (lx < 0 ? 0 : lx);
    const float k2 = kLog2e * a.inv_c;

    float qzp[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) qzp[v] = 0.f;
    if (active && (a.zg0 + zc0) > 0) {
        const float *qb = a.q_in + (int64_t)(zc0 - 1) * qps + 2 * NV * P + pix;
#pragma unroll
        for (int v = 0; v < NV; ++v) qzp[v] = ldg(qb + v * P);
    }

    float resid = 0.f;
    for (int p = zc0; p <= zc1; ++p) {
        if (p == zc1 && !has_above) break;  // block-uniform
        float *Mp = Ms + (p % 3) * RING;
        // ---------------- stage A: masses of plane p (tile + halo)
        if (active) {
            const float *qb = a.q_in + (int64_t)p * qps + pix;
            float dq[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const float qx = ldg(qb + v * P);
                const float qxm = (x > 0) ? ldg(qb + v * P - 1) : 0.f;
                const float qy = ldg(qb + (NV + v) * P);
                const float qym = (y > 0) ? ldg(qb + (NV + v) * P - a.pitch) : 0.f;
                const float qz = ldg(qb + (2 * NV + v) * P);
                dq[v] = ((qx - qxm) + (qy - qym)) + (qz - qzp[v]);
                qzp[v] = qz;
            }
            const int64_t Db = (int64_t)p * ups + pix;
            float Dv[NL], d[NI + NL];
#pragma unroll
            for (int l = 0; l < NL; ++l) Dv[l] = load_D(a.D, Db + l * P, a.d_bf16);
            label_excess<MODEL, NI, NL>(dq, Dv, d, a.g.w);
            const float *ub = a.u_in + (int64_t)p * ups + pix;
            float uold[NL], ut[NL], un[NL];   // log2 states (old / new), masses u~
#pragma unroll
            for (int l = 0; l < NL; ++l) uold[l] = ldg(ub + l * P);
            const float sum = label_update<NI, NL>(d, uold, ut, un, a.shift, k2);
            if (is_main && p < zc1) {
                if (label_sum_bad(sum)) {
                    const unsigned long long vox = ((unsigned long long)(a.zg0 + p) * a.ny + y) * a.nx + x;
                    atomicMin(a.err_voxel, vox);
                }
                float *uo = a.u_out + (int64_t)p * ups + pix;
#pragma unroll
                for (int l = 0; l < NL; ++l) st_stream(uo + l * (int)P, un[l]);
                if (a.check) resid = resid_log2<NL>(un, uold, resid);
            }
            float M[NV];
            node_masses<MODEL, NI, NL>(ut, M, a.g.w);
#pragma unroll
            for (int v = 0; v < NV; ++v) Mp[v * PS + sme] = M[v];
        }
        __syncthreads();
        // ---------------- stage B: flow step + projection of plane p-1
        if (is_main && active && p > zc0) {
            const int z = p - 1;
            const float *Mz = Ms + (z % 3) * RING;
            const float *qb = a.q_in + (int64_t)z * qps + pix;
            float *qo = a.q_out + (int64_t)z * qps + pix;
            const float *Sb = a.S ? a.S + (int64_t)z * (a.s_kind == 1 ? 1 : NV) * P + pix : nullptr;
            if (a.cap == 0) flow_out_global<NV, TY, 0>(a, Mz, Mp, true, sme, x, y, a.zg0 + z, P, qb, qo, Sb);
            else flow_out_global<NV, TY, 1>(a, Mz, Mp, true, sme, x, y, a.zg0 + z, P, qb, qo, Sb);
        }
    }
    // last plane of the volume: no plane above, nabla_z = 0
    if (!has_above && is_main && active) {
        const int z = zc1 - 1;
        const float *Mz = Ms + (z % 3) * RING;
        const float *qb = a.q_in + (int64_t)z * qps + pix;
        float *qo = a.q_out + (int64_t)z * qps + pix;
        const float *Sb = a.S ? a.S + (int64_t)z * (a.s_kind == 1 ? 1 : NV) * P + pix : nullptr;
        if (a.cap == 0) flow_out_global<NV, TY, 0>(a, Mz, Mz, false, sme, x, y, a.zg0 + z, P, qb, qo, Sb);
        else flow_out_global<NV, TY, 1>(a, Mz, Mz, false, sme, x, y, a.zg0 + z, P, qb, qo, Sb);
    }
    if (a.check) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) resid = fmaxf(resid, __shfl_xor_sync(0xffffffffu, resid, o));
        if (lane == 0 && resid > 0.f) atomicMax(a.resid_bits, __float_as_uint(resid));
    }
}

// Launch table entry (pf_iter_table.cu); returns false if (NI, NL) is not compiled in.
// Generic path (pf_generic.cu): any DAG up to kWideNodes non-source nodes (<= 16 end labels) -- the graphs beyond
// the compiled kernel set (> kMaxInternal internal or > kMaxNodes nodes).  Dense weights over all positions.
constexpr int kWideNodes = 31;
struct GraphWide {
    float w[kWideNodes][32];   // w[i][j]: weight of edge (position i -> position j), i internal; 0 = no edge
    float s[32];               // capacity scalar per position
};

struct IterKernelInfo {
    const void *func;
    int threads;
    int smem_bytes;
    int tile_y;
};

bool iter_kernel_lookup(int NI, int NL, int MODEL, IterKernelInfo *info);

}  // namespace pf
