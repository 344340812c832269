// pf_alm.cu -- explicit-flow (full-flow) augmented-Lagrangian max-flow for the Potts model on sm_100a:
// the comparison arm of SURVEY 8(f2) (pf_config.method = PF_METHOD_EXPLICIT_ALM).
//
// The paper's point (P:5) is that the pseudo-flow iteration (Alg. 1) keeps the source
// and sink flows p_S, p_L implicit.  This is the classic alternative that stores them: block-coordinate
// ascent on the augmented Lagrangian of Eq. 3 with u as the multipliers,
//   L_c = p_S + sum_L u_L r_L - c/2 sum_L r_L^2,   r_L = div q_L - p_S + p_L,   p_L <= D_L, |q_L| <= S_L,
// one sweep per iteration in block-coordinate order (q, then p, then p_S, then u) (the labels are independent given p_S):
//   q_L  <- Proj_{|q| <= S_L}( q_L + tau grad(div q_L - p_S + p_L - u_L / c) )     [alm_flow_all_kernel (K <= 8),
//                                                                                     alm_flow_kernel]
//   p_L  <- min(D_L, p_S - div q_L + u_L / c)              (new q)                  [alm_potential_kernel]
//   p_S  <- (sum_L (p_L + div q_L - u_L / c)) / K + 1 / (K c)
//   u_L  <- u_L - c (div q_L - p_S + p_L)
// The p / p_S / u update needs the divergence of the NEW flows at every voxel, so one iteration is two
// dependent HBM passes (the pseudo-flow iteration is one): that, and the extra p_L, p_S buffers, are what
// the comparison measures.  Discretisation as everywhere (reading R4): forward grad with 0 at the last
// index, div = -grad^T with q^k(-1) = 0.
//
// Layouts (pf_api.cu): q ping-pong [z][k][L][y][pitch] with planes -1..nz (as the pseudo-flow solver),
// u, p [z][L][y][pitch] updated in place, p_S [z][y][pitch] in place, D, S as the pseudo-flow solver.
#include <cfloat>
#include <cstdint>
#include <cuda_runtime.h>

#include "pf_alm.cuh"
#include "pf_kernels.cuh"   // constants + pf_math.cuh (flow_step3, load_D)

namespace pf {

namespace {

constexpr int kAlmTY = 8;   // flow kernel tile height (32 x 8 voxels, +1 halo row / column for the gradient)

__device__ __forceinline__ float ld(const float *p) { return __ldg(p); }

// capacity S_L(z, pixel): scalar per label, shared field x per-label factor, or a field per label
__device__ __forceinline__ float cap_at(const AlmArgs &a, int L, int z, int pix, int64_t P) {
    if (!a.S) return a.s[L];
    if (a.s_per_node) return ld(a.S + ((int64_t)z * (a.dag ? a.NV : a.NL) + L) * P + pix);
    return ld(a.S + (int64_t)z * P + pix) * a.s[L];
}

// Proj_{|q| <= S} (l2: the pseudo-flow solver's exactly-rescaled projection; box: clamp)
__device__ __forceinline__ void project(int cap, float sv, float &hx, float &hy, float &hz) {
    if (cap == 0) flow_step3<0>(0.f, 0.f, 0.f, 0.f, 0.f, 0.f, sv, hx, hy, hz);
    else flow_step3<1>(0.f, 0.f, 0.f, 0.f, 0.f, 0.f, sv, hx, hy, hz);
}

// Pass 1, one label per CTA z-slice of the grid: f = div q - p_S + p_L - u_L / c on the tile and its +x/+y
// halo, then q' = Proj(q + tau grad f) on the tile.  z-march with a 3-slot shared ring of f planes.
__global__ void __launch_bounds__(32 * kAlmTY + 64) alm_flow_kernel(const AlmArgs a) {
    constexpr int TY = kAlmTY, RS = 33, PS = (TY + 1) * RS;
    __shared__ float F[3 * PS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool is_main = warp < TY;
    int lx, ly;
    if (is_main) {
        lx = lane; ly = warp;
    } else {
        const int h = (warp - TY) * 32 + lane;
        if (h < 32) { lx = h; ly = TY; }
        else if (h < 32 + TY) { lx = 32; ly = h - 32; }
        else { lx = -1; ly = 0; }
    }
    const int nch = (a.nz + a.zchunk - 1) / a.zchunk;
    const int L = blockIdx.z / nch, chunk = blockIdx.z - L * nch;
    const int x = blockIdx.x * 32 + lx, y = blockIdx.y * TY + ly;
    const bool active = lx >= 0 && x < a.nx && y < a.ny;
    const int64_t P = (int64_t)a.pitch * a.ny;
    const int64_t qps = (int64_t)3 * a.NL * P, ups = (int64_t)a.NL * P;
    const int pix = active ? y * a.pitch + x : 0;
    const int sme = ly * RS + (lx < 0 ? 0 : lx);
    const int zc0 = chunk * a.zchunk, zc1 = min(zc0 + a.zchunk, a.nz);
    const bool has_above = zc1 < a.nz;
    const float cx = x < a.nx - 1 ? a.tau : 0.f, cy = y < a.ny - 1 ? a.tau : 0.f;

    // q of the plane below the chunk (z-component enters div of the first plane)
    float qzp = 0.f;
    if (active && zc0 > 0) qzp = ld(a.q_in + (int64_t)(zc0 - 1) * qps + (2 * a.NL + L) * P + pix);
    float qcx = 0.f, qcy = 0.f, qcz = 0.f;   // q(p-1) at the voxel, for its flow step one plane later
    for (int p = zc0; p <= zc1; ++p) {
        if (p == zc1 && !has_above) break;   // block-uniform
        float *Fp = F + (p % 3) * PS;
        float f = 0.f, qx = 0.f, qy = 0.f, qz = 0.f;
        if (active) {
            const float *qb = a.q_in + (int64_t)p * qps + pix;
            qx = ld(qb + L * P);
            qy = ld(qb + (a.NL + L) * P);
            qz = ld(qb + (2 * a.NL + L) * P);
            const float qxm = x > 0 ? ld(qb + L * P - 1) : 0.f;
            const float qym = y > 0 ? ld(qb + (a.NL + L) * P - a.pitch) : 0.f;
            const float dq = ((qx - qxm) + (qy - qym)) + (qz - qzp);
            const int64_t o = (int64_t)p * ups + L * P + pix;
            f = ((dq - ld(a.pS + (int64_t)p * P + pix)) + ld(a.p + o)) - ld(a.u + o) * a.inv_c;
            qzp = qz;
        }
        if (lx >= 0) Fp[sme] = f;   // (idle halo lanes have lx < 0 and no slot)
        __syncthreads();
        if (is_main && active && p > zc0) {
            const int z = p - 1;
            const float *Fz = F + (z % 3) * PS;
            const float fc = Fz[sme];
            const float gx = Fz[sme + 1] - fc, gy = Fz[sme + RS] - fc;
            const float gz = f - fc;   // f(z+1) at the voxel; z + 1 <= nz - 1 here
            const float sv = cap_at(a, L, z, pix, P);
            float hx = fmaf(cx, gx, qcx), hy = fmaf(cy, gy, qcy), hz = fmaf(a.tau, gz, qcz);   // ascent step
            project(a.cap, sv, hx, hy, hz);
            float *qo = a.q_out + (int64_t)z * qps + pix;
            qo[L * P] = hx;
            qo[(a.NL + L) * P] = hy;
            qo[(2 * a.NL + L) * P] = hz;
        }
        qcx = qx; qcy = qy; qcz = qz;
    }
    if (!has_above && is_main && active) {   // last plane of the volume: grad_z f = 0
        const int z = zc1 - 1;
        const float *Fz = F + (z % 3) * PS;
        const float fc = Fz[sme];
        const float gx = Fz[sme + 1] - fc, gy = Fz[sme + RS] - fc;
        const float sv = cap_at(a, L, z, pix, P);
        float hx = fmaf(cx, gx, qcx), hy = fmaf(cy, gy, qcy), hz = qcz;
        project(a.cap, sv, hx, hy, hz);
        float *qo = a.q_out + (int64_t)z * qps + pix;
        qo[L * P] = hx;
        qo[(a.NL + L) * P] = hy;
        qo[(2 * a.NL + L) * P] = hz;
    }
}

// Pass 1, all labels of a point per thread (Potts): the same arithmetic as alm_flow_kernel, with the
// per-point work (addressing, p_S, S, the ring barrier) shared by the K labels of the point.
constexpr int kAlmAllTY = 8;   // pass-1 all-labels tile height (TY = 4: 2.06 vs 1.84 ms per C2 ALM iteration)
template <int NL>
__global__ void __launch_bounds__(32 * kAlmAllTY + 64) alm_flow_all_kernel(const AlmArgs a) {
    constexpr int TY = kAlmAllTY, RS = 33, PS = (TY + 1) * RS;
    __shared__ float F[3 * NL * PS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool is_main = warp < TY;
    int lx, ly;
    if (is_main) {
        lx = lane; ly = warp;
    } else {
        const int h = (warp - TY) * 32 + lane;
        if (h < 32) { lx = h; ly = TY; }
        else if (h < 32 + TY) { lx = 32; ly = h - 32; }
        else { lx = -1; ly = 0; }
    }
    const int chunk = blockIdx.z;
    const int x = blockIdx.x * 32 + lx, y = blockIdx.y * TY + ly;
    const bool active = lx >= 0 && x < a.nx && y < a.ny;
    const int64_t P = (int64_t)a.pitch * a.ny;
    const int64_t qps = (int64_t)3 * NL * P, ups = (int64_t)NL * P;
    const int pix = active ? y * a.pitch + x : 0;
    const int sme = ly * RS + (lx < 0 ? 0 : lx);
    const int zc0 = chunk * a.zchunk, zc1 = min(zc0 + a.zchunk, a.nz);
    const bool has_above = zc1 < a.nz;
    const float cx = x < a.nx - 1 ? a.tau : 0.f, cy = y < a.ny - 1 ? a.tau : 0.f;

    float qzp[NL], qc[3][NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) {
        qzp[l] = (active && zc0 > 0) ? ld(a.q_in + (int64_t)(zc0 - 1) * qps + (2 * NL + l) * P + pix) : 0.f;
        qc[0][l] = qc[1][l] = qc[2][l] = 0.f;
    }
    auto flow_out = [&](int z, const float (&fn)[NL], bool has_z) {
        const float *Fz = F + (z % 3) * NL * PS;
        float *qo = a.q_out + (int64_t)z * qps + pix;
#pragma unroll
        for (int l = 0; l < NL; ++l) {
            const float fc = Fz[l * PS + sme];
            const float gx = Fz[l * PS + sme + 1] - fc, gy = Fz[l * PS + sme + RS] - fc;
            const float sv = cap_at(a, l, z, pix, P);
            float hx = fmaf(cx, gx, qc[0][l]), hy = fmaf(cy, gy, qc[1][l]);
            float hz = has_z ? fmaf(a.tau, fn[l] - fc, qc[2][l]) : qc[2][l];
            project(a.cap, sv, hx, hy, hz);
            qo[l * P] = hx;
            qo[(NL + l) * P] = hy;
            qo[(2 * NL + l) * P] = hz;
        }
    };
    for (int p = zc0; p <= zc1; ++p) {
        if (p == zc1 && !has_above) break;   // block-uniform
        float *Fp = F + (p % 3) * NL * PS;
        float f[NL], qn[3][NL];
        if (active) {
            const float *qb = a.q_in + (int64_t)p * qps + pix;
            const int64_t o = (int64_t)p * ups + pix;
            const float ps = ld(a.pS + (int64_t)p * P + pix);
#pragma unroll
            for (int l = 0; l < NL; ++l) {
                const float qx = ld(qb + l * P), qy = ld(qb + (NL + l) * P), qz = ld(qb + (2 * NL + l) * P);
                const float qxm = x > 0 ? ld(qb + l * P - 1) : 0.f;
                const float qym = y > 0 ? ld(qb + (NL + l) * P - a.pitch) : 0.f;
                const float dq = ((qx - qxm) + (qy - qym)) + (qz - qzp[l]);
                f[l] = ((dq - ps) + ld(a.p + o + l * P)) - ld(a.u + o + l * P) * a.inv_c;
                qzp[l] = qz;
                qn[0][l] = qx; qn[1][l] = qy; qn[2][l] = qz;
            }
        } else {
#pragma unroll
            for (int l = 0; l < NL; ++l) { f[l] = 0.f; qn[0][l] = qn[1][l] = qn[2][l] = 0.f; }
        }
        if (lx >= 0) {
#pragma unroll
            for (int l = 0; l < NL; ++l) Fp[l * PS + sme] = f[l];
        }
        __syncthreads();
        if (is_main && active && p > zc0) flow_out(p - 1, f, true);
#pragma unroll
        for (int l = 0; l < NL; ++l) { qc[0][l] = qn[0][l]; qc[1][l] = qn[1][l]; qc[2][l] = qn[2][l]; }
        // the ring slot written next (p + 1) % 3 was last read by flow_out(p - 2) before this barrier
    }
    if (!has_above && is_main && active) {   // last plane of the volume: grad_z f = 0
        float fz[NL];
#pragma unroll
        for (int l = 0; l < NL; ++l) fz[l] = 0.f;
        flow_out(zc1 - 1, fz, false);
    }
}

template <int NL>
cudaError_t launch_flow_all(const AlmArgs &a, cudaStream_t st) {
    const int nch = (a.nz + a.zchunk - 1) / a.zchunk;
    dim3 g((a.nx + 31) / 32, (a.ny + kAlmAllTY - 1) / kAlmAllTY, nch);
    alm_flow_all_kernel<NL><<<g, 32 * kAlmAllTY + 64, 0, st>>>(a);
    return cudaGetLastError();
}

// Pass 2, every label of a voxel column per thread, z-march: div of the NEW flows, then p_L, p_S, u_L
// in that order (p_L uses the old p_S; u uses the new p_S).  Residual max|u' - u| fused.
template <int NL>
__global__ void __launch_bounds__(128) alm_potential_kernel(const AlmArgs a) {
    const int x = blockIdx.x * 32 + (threadIdx.x & 31);
    const int y = blockIdx.y * 4 + (threadIdx.x >> 5);
    const bool valid = x < a.nx && y < a.ny;   // no early return: the residual reduction is warp-wide
    const int64_t P = (int64_t)a.pitch * a.ny;
    const int64_t qps = (int64_t)3 * NL * P, ups = (int64_t)NL * P;
    const int pix = valid ? y * a.pitch + x : 0;
    const int zc0 = blockIdx.z * a.zchunk2, zc1 = valid ? min(zc0 + a.zchunk2, a.nz) : zc0;
    const float invK = 1.0f / NL;
    float qzp[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) qzp[l] = zc0 > 0 ? ld(a.q_out + (int64_t)(zc0 - 1) * qps + (2 * NL + l) * P + pix) : 0.f;
    float resid = 0.f;
    for (int z = zc0; z < zc1; ++z) {
        const float *qb = a.q_out + (int64_t)z * qps + pix;
        const int64_t o = (int64_t)z * ups + pix;
        const float ps_old = ld(a.pS + (int64_t)z * P + pix);
        float dq[NL], pn[NL], uo[NL];
        float acc = 0.f;
#pragma unroll
        for (int l = 0; l < NL; ++l) {
            const float qx = ld(qb + l * P), qy = ld(qb + (NL + l) * P), qz = ld(qb + (2 * NL + l) * P);
            const float qxm = x > 0 ? ld(qb + l * P - 1) : 0.f;
            const float qym = y > 0 ? ld(qb + (NL + l) * P - a.pitch) : 0.f;
            dq[l] = ((qx - qxm) + (qy - qym)) + (qz - qzp[l]);
            qzp[l] = qz;
            uo[l] = ld(a.u + o + l * P);
            pn[l] = fminf(load_D(a.D, o + l * P, a.d_bf16), (ps_old - dq[l]) + uo[l] * a.inv_c);
            acc += (pn[l] + dq[l]) - uo[l] * a.inv_c;
        }
        const float ps = acc * invK + invK * a.inv_c;
        a.pS[(int64_t)z * P + pix] = ps;
#pragma unroll
        for (int l = 0; l < NL; ++l) {
            const float un = uo[l] - a.c * ((dq[l] - ps) + pn[l]);
            a.p[o + l * P] = pn[l];
            a.u[o + l * P] = un;
            resid = fmaxf(resid, fabsf(un - uo[l]));
        }
    }
    if (a.check) {
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) resid = fmaxf(resid, __shfl_xor_sync(0xffffffffu, resid, s));
        if ((threadIdx.x & 31) == 0 && resid > 0.f) atomicMax(a.resid_bits, __float_as_uint(resid));
    }
}

// ------------------------------------------------------------------------------------------------
// DAG / HMF explicit-flow ALM (Eq. 11): every node v != S has u_v, p_v, q_v; residuals
//   r_v = div q_v + p_v - sum_{P in parents(v)} w_(P,v) p_P        (source row: p_S)
// pass 1 (per node): q_v <- Proj(q_v + tau grad(r_v - u_v / c))                       [alm_dag_flow_kernel]
// pass 2 (per voxel, nodes in topological order, the block-coordinate maxima of L_c):  [alm_dag_potential]
//   p_S  = ((1 - sum_c w u_c) / c + sum_c w (r_c + w p_S)) / sum_c w^2        (c: children of S)
//   p_v  = ((u_v - sum_c w u_c) / c - (div q_v - sum_P w p_P) + sum_c w (r_c + w p_v)) / (1 + sum_c w^2)
//   p_L  = min(D_L, u_L / c - div q_L + sum_P w p_P)                            (end labels)
//   u_v -= c r_v                                                                 (all v, new p)

// pass 1: one node per CTA z-slice; f = r_v - u_v / c on the tile + halo, q' = Proj(q + tau grad f)
__global__ void __launch_bounds__(32 * kAlmTY + 64) alm_dag_flow_kernel(const AlmArgs a) {
    constexpr int TY = kAlmTY, RS = 33, PS = (TY + 1) * RS;
    __shared__ float F[3 * PS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool is_main = warp < TY;
    int lx, ly;
    if (is_main) {
        lx = lane; ly = warp;
    } else {
        const int h = (warp - TY) * 32 + lane;
        if (h < 32) { lx = h; ly = TY; }
        else if (h < 32 + TY) { lx = 32; ly = h - 32; }
        else { lx = -1; ly = 0; }
    }
    const int nch = (a.nz + a.zchunk - 1) / a.zchunk;
    const int v = blockIdx.z / nch, chunk = blockIdx.z - v * nch;
    const int x = blockIdx.x * 32 + lx, y = blockIdx.y * TY + ly;
    const bool active = lx >= 0 && x < a.nx && y < a.ny;
    const int64_t P = (int64_t)a.pitch * a.ny;
    const int NV = a.NV, NLab = a.NL;
    const int64_t qps = (int64_t)3 * NV * P;
    const int pix = active ? y * a.pitch + x : 0;
    const int sme = ly * RS + (lx < 0 ? 0 : lx);
    const int zc0 = chunk * a.zchunk, zc1 = min(zc0 + a.zchunk, a.nz);
    const bool has_above = zc1 < a.nz;
    const float cx = x < a.nx - 1 ? a.tau : 0.f, cy = y < a.ny - 1 ? a.tau : 0.f;
    float qzp = 0.f;
    if (active && zc0 > 0) qzp = ld(a.q_in + (int64_t)(zc0 - 1) * qps + (2 * NV + v) * P + pix);
    float qcx = 0.f, qcy = 0.f, qcz = 0.f;
    for (int p = zc0; p <= zc1; ++p) {
        if (p == zc1 && !has_above) break;
        float *Fp = F + (p % 3) * PS;
        float f = 0.f, qx = 0.f, qy = 0.f, qz = 0.f;
        if (active) {
            const float *qb = a.q_in + (int64_t)p * qps + pix;
            qx = ld(qb + v * P);
            qy = ld(qb + (NV + v) * P);
            qz = ld(qb + (2 * NV + v) * P);
            const float qxm = x > 0 ? ld(qb + v * P - 1) : 0.f;
            const float qym = y > 0 ? ld(qb + (NV + v) * P - a.pitch) : 0.f;
            const float dq = ((qx - qxm) + (qy - qym)) + (qz - qzp);
            const float *pb = a.p + (int64_t)p * NV * P + pix;
            float inflow = a.W[0][v] * ld(a.pS + (int64_t)p * P + pix);
            for (int i = 0; i < a.NI; ++i)
                if (a.W[1 + i][v] != 0.f) inflow = fmaf(a.W[1 + i][v], ld(pb + i * P), inflow);
            const float uv = v < a.NI ? ld(a.u_int + ((int64_t)p * a.NI + v) * P + pix)
                                      : ld(a.u + ((int64_t)p * NLab + (v - a.NI)) * P + pix);
            f = ((dq + ld(pb + v * P)) - inflow) - uv * a.inv_c;
            qzp = qz;
        }
        if (lx >= 0) Fp[sme] = f;
        __syncthreads();
        if (is_main && active && p > zc0) {
            const int z = p - 1;
            const float *Fz = F + (z % 3) * PS;
            const float fc = Fz[sme];
            const float gx = Fz[sme + 1] - fc, gy = Fz[sme + RS] - fc, gz = f - fc;
            const float sv = cap_at(a, v, z, pix, P);
            float hx = fmaf(cx, gx, qcx), hy = fmaf(cy, gy, qcy), hz = fmaf(a.tau, gz, qcz);
            project(a.cap, sv, hx, hy, hz);
            float *qo = a.q_out + (int64_t)z * qps + pix;
            qo[v * P] = hx;
            qo[(NV + v) * P] = hy;
            qo[(2 * NV + v) * P] = hz;
        }
        qcx = qx; qcy = qy; qcz = qz;
    }
    if (!has_above && is_main && active) {
        const int z = zc1 - 1;
        const float *Fz = F + (z % 3) * PS;
        const float fc = Fz[sme];
        const float gx = Fz[sme + 1] - fc, gy = Fz[sme + RS] - fc;
        const float sv = cap_at(a, v, z, pix, P);
        float hx = fmaf(cx, gx, qcx), hy = fmaf(cy, gy, qcy), hz = qcz;
        project(a.cap, sv, hx, hy, hz);
        float *qo = a.q_out + (int64_t)z * qps + pix;
        qo[v * P] = hx;
        qo[(NV + v) * P] = hy;
        qo[(2 * NV + v) * P] = hz;
    }
}

// pass 2: per voxel column over a short z-chunk (a.zchunk2 planes: parallelism over the whole volume),
// node arrays in registers (NVT = NV non-source nodes, fully unrolled)
template <int NVT>
__global__ void __launch_bounds__(128) alm_dag_potential_kernel(const AlmArgs a) {
    const int x = blockIdx.x * 32 + (threadIdx.x & 31);
    const int y = blockIdx.y * 4 + (threadIdx.x >> 5);
    const bool valid = x < a.nx && y < a.ny;
    const int64_t P = (int64_t)a.pitch * a.ny;
    constexpr int NV = NVT;
    const int NI = a.NI, NLab = a.NL;
    const int64_t qps = (int64_t)3 * NV * P;
    const int pix = valid ? y * a.pitch + x : 0;
    const int zc0 = blockIdx.z * a.zchunk2, zc1 = valid ? min(zc0 + a.zchunk2, a.nz) : zc0;
    float qzp[NVT];
#pragma unroll
    for (int v = 0; v < NVT; ++v)
        qzp[v] = (v < NV && zc0 > 0) ? ld(a.q_out + (int64_t)(zc0 - 1) * qps + (2 * NV + v) * P + pix) : 0.f;
    float resid = 0.f;
    for (int z = zc0; z < zc1; ++z) {
        const float *qb = a.q_out + (int64_t)z * qps + pix;
        float dq[NVT], pv[NVT], uv[NVT];
#pragma unroll
        for (int v = 0; v < NVT; ++v) {
            if (v >= NV) { dq[v] = pv[v] = uv[v] = 0.f; continue; }
            const float qx = ld(qb + v * P), qy = ld(qb + (NV + v) * P), qz = ld(qb + (2 * NV + v) * P);
            const float qxm = x > 0 ? ld(qb + v * P - 1) : 0.f;
            const float qym = y > 0 ? ld(qb + (NV + v) * P - a.pitch) : 0.f;
            dq[v] = ((qx - qxm) + (qy - qym)) + (qz - qzp[v]);
            qzp[v] = qz;
            pv[v] = ld(a.p + ((int64_t)z * NV + v) * P + pix);
            uv[v] = v < NI ? ld(a.u_int + ((int64_t)z * NI + v) * P + pix)
                           : ld(a.u + ((int64_t)z * NLab + (v - NI)) * P + pix);
        }
        float ps = ld(a.pS + (int64_t)z * P + pix);
        // inflow of position c with the current p: sum_P w_(P,c) p_P
        auto inflow = [&](int c) {
            float acc = a.W[0][c] * ps;
#pragma unroll
            for (int i = 0; i < NVT; ++i)
                if (i < NI && a.W[1 + i][c] != 0.f) acc = fmaf(a.W[1 + i][c], pv[i], acc);
            return acc;
        };
        auto r_of = [&](int c) { return (dq[c] + pv[c]) - inflow(c); };
        // source
        {
            float sw2 = 0.f, wu = 0.f, acc = 0.f;
#pragma unroll
            for (int c = 0; c < NVT; ++c) {
                const float w = c < NV ? a.W[0][c] : 0.f;
                if (w != 0.f) {
                    sw2 = fmaf(w, w, sw2);
                    wu = fmaf(w, uv[c], wu);
                    acc = fmaf(w, fmaf(w, ps, r_of(c)), acc);
                }
            }
            ps = ((1.f - wu) * a.inv_c + acc) / sw2;
        }
        // internal nodes (topological), then end labels
#pragma unroll
        for (int v = 0; v < NVT; ++v) {
            if (v >= NV) continue;
            if (v < NI) {
                float sw2 = 0.f, wu = 0.f, acc = 0.f;
#pragma unroll
                for (int c = 0; c < NVT; ++c) {
                    const float w = c < NV ? a.W[1 + v][c] : 0.f;
                    if (w != 0.f) {
                        sw2 = fmaf(w, w, sw2);
                        wu = fmaf(w, uv[c], wu);
                        acc = fmaf(w, fmaf(w, pv[v], r_of(c)), acc);
                    }
                }
                pv[v] = (((uv[v] - wu) * a.inv_c - (dq[v] - inflow(v))) + acc) / (1.f + sw2);
            } else {
                pv[v] = fminf(load_D(a.D, ((int64_t)z * NLab + (v - NI)) * P + pix, a.d_bf16),
                              (uv[v] * a.inv_c - dq[v]) + inflow(v));
            }
        }
        a.pS[(int64_t)z * P + pix] = ps;
        float res[NVT];
#pragma unroll
        for (int v = 0; v < NVT; ++v) res[v] = v < NV ? r_of(v) : 0.f;
#pragma unroll
        for (int v = 0; v < NVT; ++v) {
            if (v >= NV) continue;
            const float un = uv[v] - a.c * res[v];
            a.p[((int64_t)z * NV + v) * P + pix] = pv[v];
            if (v < NI) a.u_int[((int64_t)z * NI + v) * P + pix] = un;
            else a.u[((int64_t)z * NLab + (v - NI)) * P + pix] = un;
            if (v >= NI) resid = fmaxf(resid, fabsf(un - uv[v]));
        }
    }
    if (a.check) {
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) resid = fmaxf(resid, __shfl_xor_sync(0xffffffffu, resid, s));
        if ((threadIdx.x & 31) == 0 && resid > 0.f) atomicMax(a.resid_bits, __float_as_uint(resid));
    }
}

// DAG start: u_L = 1/|L|, u_v = sum_c w u_c (reverse topological), p = 0, p_S = min_L D_L
__global__ void alm_dag_init_kernel(const AlmArgs a) {
    const int64_t P = (int64_t)a.pitch * a.ny;
    const int64_t V = (int64_t)a.nx * a.ny * a.nz;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t z = i / ((int64_t)a.nx * a.ny);
        const int r = (int)(i - z * (int64_t)a.nx * a.ny);
        const int y = r / a.nx, x = r - y * a.nx;
        const int64_t pix = (int64_t)y * a.pitch + x;
        float m = FLT_MAX;
        for (int l = 0; l < a.NL; ++l) m = fminf(m, load_D(a.D, (z * a.NL + l) * P + pix, a.d_bf16));
        a.pS[z * P + pix] = m;
        float uv[16];
        for (int v = 0; v < a.NV; ++v) uv[v] = v >= a.NI ? 1.0f / (float)a.NL : 0.f;
        for (int v = a.NI - 1; v >= 0; --v) {
            float acc = 0.f;
            for (int c = 0; c < a.NV; ++c) acc = fmaf(a.W[1 + v][c], uv[c], acc);
            uv[v] = acc;
        }
        for (int v = 0; v < a.NV; ++v) {
            a.p[(z * a.NV + v) * P + pix] = 0.f;
            if (v < a.NI) a.u_int[(z * a.NI + v) * P + pix] = uv[v];
        }
    }
}

// p_S = min_L D_L, p_L = p_S (the standard start; u = 1/K and q = 0 are set by the caller).
__global__ void alm_init_kernel(const AlmArgs a) {
    const int64_t P = (int64_t)a.pitch * a.ny;
    const int64_t V = (int64_t)a.nx * a.ny * a.nz;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t z = i / ((int64_t)a.nx * a.ny);
        const int r = (int)(i - z * (int64_t)a.nx * a.ny);
        const int y = r / a.nx, x = r - y * a.nx;
        const int64_t o = z * a.NL * P + (int64_t)y * a.pitch + x;
        float m = FLT_MAX;
        for (int l = 0; l < a.NL; ++l) m = fminf(m, load_D(a.D, o + l * P, a.d_bf16));
        a.pS[z * P + (int64_t)y * a.pitch + x] = m;
        for (int l = 0; l < a.NL; ++l) a.p[o + l * P] = m;
    }
}

template <int NL>
cudaError_t launch_pot(const AlmArgs &a, cudaStream_t st) {
    dim3 grid((a.nx + 31) / 32, (a.ny + 3) / 4, (a.nz + a.zchunk2 - 1) / a.zchunk2);
    alm_potential_kernel<NL><<<grid, 128, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_alm_init(const AlmArgs &a, cudaStream_t st) {
    if (a.dag) alm_dag_init_kernel<<<1184, 256, 0, st>>>(a);
    else alm_init_kernel<<<1184, 256, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_alm_iteration(const AlmArgs &a, cudaStream_t st) {
    const int nch = (a.nz + a.zchunk - 1) / a.zchunk;
    if (a.dag) {
        dim3 g1((a.nx + 31) / 32, (a.ny + kAlmTY - 1) / kAlmTY, nch * a.NV);
        alm_dag_flow_kernel<<<g1, 32 * kAlmTY + 64, 0, st>>>(a);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        dim3 g2((a.nx + 31) / 32, (a.ny + 3) / 4, (a.nz + a.zchunk2 - 1) / a.zchunk2);
        switch (a.NV) {
#define PF_DAGPOT(n) case n: alm_dag_potential_kernel<n><<<g2, 128, 0, st>>>(a); break;
            PF_DAGPOT(3) PF_DAGPOT(4) PF_DAGPOT(5) PF_DAGPOT(6) PF_DAGPOT(7) PF_DAGPOT(8) PF_DAGPOT(9)
            PF_DAGPOT(10) PF_DAGPOT(11) PF_DAGPOT(12) PF_DAGPOT(13) PF_DAGPOT(14) PF_DAGPOT(15) PF_DAGPOT(16)
#undef PF_DAGPOT
            default: return cudaErrorInvalidValue;
        }
        return cudaGetLastError();
    }
    cudaError_t e;
    switch (a.NL) {   // pass 1: all labels of a point per thread (K <= 8: the smem ring stays <= 28.5 KB)
#define PF_FLOWALL(n) case n: e = launch_flow_all<n>(a, st); break;
        PF_FLOWALL(2) PF_FLOWALL(3) PF_FLOWALL(4) PF_FLOWALL(5) PF_FLOWALL(6) PF_FLOWALL(7) PF_FLOWALL(8)
#undef PF_FLOWALL
        default: {
            dim3 g1((a.nx + 31) / 32, (a.ny + kAlmTY - 1) / kAlmTY, nch * a.NL);
            alm_flow_kernel<<<g1, 32 * kAlmTY + 64, 0, st>>>(a);
            e = cudaGetLastError();
        }
    }
    if (e != cudaSuccess) return e;
    switch (a.NL) {
        case 2: return launch_pot<2>(a, st);
        case 3: return launch_pot<3>(a, st);
        case 4: return launch_pot<4>(a, st);
        case 5: return launch_pot<5>(a, st);
        case 6: return launch_pot<6>(a, st);
        case 7: return launch_pot<7>(a, st);
        case 8: return launch_pot<8>(a, st);
        case 9: return launch_pot<9>(a, st);
        case 10: return launch_pot<10>(a, st);
        case 11: return launch_pot<11>(a, st);
        case 12: return launch_pot<12>(a, st);
        case 13: return launch_pot<13>(a, st);
        case 14: return launch_pot<14>(a, st);
        case 15: return launch_pot<15>(a, st);
        case 16: return launch_pot<16>(a, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace pf
