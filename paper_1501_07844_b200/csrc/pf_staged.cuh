// pf_staged.cuh -- TMA-staged, persistent version of the fused pseudo-flow iteration (sm_100a).
//
// Same arithmetic and same per-voxel order as pf_iter_kernel (see pf_kernels.cuh for the
// step-by-step mapping to Alg. 1 / Alg. 2 / Alg. 3; the shared math is in pf_math.cuh), different
// data movement:
//   * persistent CTAs (one per SM) walk work items = (32 x TY tile, z-chunk) in a static
//     round-robin order, so the tiles in flight at any time are spatial neighbours and their
//     shared halo lines are served from L2;
//   * every z-plane of the tile is fetched by ONE thread as 3-4 TMA box loads
//     (cp.async.bulk.tensor.4d) into a 2-deep shared-memory ring guarded by mbarriers: q over
//     x in [x0-4, x0+36) x y in [y0-1, y0+TY] (the -x/-y neighbours for div and the +1 halo
//     points), u and D over [x0, x0+36) x [y0, y0+TY], S over the tile.  Out-of-range box
//     elements are zero-filled by the TMA unit, which is exactly q^k(-1) = 0 (reading R4);
//   * plane p+2 is in flight while plane p is computed; q(p) and S(p) of the own voxel are kept
//     in registers (two alternating sets) until the flow step of plane p runs one plane later;
//   * OSTAGE: the new u and q are staged in shared memory and written by TMA bulk-tensor stores
//     with an evict-first L2 policy (no per-thread 64-bit address arithmetic, no L2 pollution);
//     OSTAGE 1 double-buffers the flow staging tile, OSTAGE 2 (many nodes, tight shared memory) has a
//     single one whose reuse is guarded by an mbarrier that thread 0 arrives on once the previous
//     store has read it;
//   * G = 2 (Potts with many labels): the labels of a row of 32 voxels are split over a warp pair;
//     the only per-voxel couplings of the label update -- m = min_L d_L and a = sum_L u~_L -- are
//     exchanged through shared memory under a 64-thread named barrier.  The sum is always formed
//     as (first half) + (second half) (also for G = 1, see label_update), so G does not change a bit.
#pragma once
#include <cuda.h>

#include "pf_kernels.cuh"
#include "pf_tma.cuh"

namespace pf {

struct StagedArgs {
    CUtensorMap tm_q;   // input q, 4-D (x, y, channel = k*NF+f, plane+1) over the NF flow-carrying nodes
    CUtensorMap tm_u;   // input u, 4-D (x, y, l, plane+1)
    CUtensorMap tm_D;   // D, 4-D (x, y, l, plane)
    CUtensorMap tm_S;   // S field, 4-D (x, y, channel, plane); unused when s_ch == 0
    CUtensorMap tm_uo;  // output u, store box (32, TY, NL)        [OSTAGE]
    CUtensorMap tm_qo;  // output q, store box (32, TY, 3*NF)      [OSTAGE]
    const float *q_in;  // plane 0 of input q (chunk-start q^z(zc0-1) read)
    float *u_out;
    float *q_out;
    int nx, ny, pitch, nzl, zg0, nzg;
    int zchunk, tiles_x, tiles, items;
    int s_ch;     // 0: scalar capacities, 1: shared field (x g.s[f]), NF: field per flow node
    int cap, shift, check;
    unsigned int tx_bytes;
    float inv_c, ctau;
    unsigned int *resid_bits;
    unsigned long long *err_voxel;
    GraphConst g;
};

__host__ __device__ constexpr int round32(int n) { return (n + 31) / 32 * 32; }

template <int NI, int NL, int TY, int OSTAGE, int MODEL, int G>
struct StagedLayout {
    static constexpr int NV = NI + NL;
    static constexpr int NF = Model<MODEL, NI, NL>::NF;   // flow-carrying nodes
    static constexpr int QW = 40, UW = 36, SW = 32;
    static constexpr int QROWS = TY + 2, UROWS = TY + 1;
    static constexpr int QSZ = round32(3 * NF * QROWS * QW);  // floats per stage
    static constexpr int USZ = round32(NL * UROWS * UW);
    static constexpr int RS = 33, RPS = (TY + 1) * RS, RING = NF * RPS;
    static constexpr int UOSZ = OSTAGE ? round32(NL * TY * 32) : 0;       // output staging (per buffer)
    static constexpr int QOSZ = OSTAGE ? round32(3 * NF * TY * 32) : 0;
    static constexpr int QOB = OSTAGE == 1 ? 2 : 1;                         // flow staging buffers
    static constexpr int XSZ = G > 1 ? round32(2 * (TY + 2) * G * 32) : 0;  // m / a exchange (G = 2)
    static constexpr int kThreads = 32 * G * (TY + 2);
    // runtime part: the S staging ring holds s_ch channels (0, 1 or NF)
    __host__ __device__ static constexpr int ssz(int s_ch) { return round32(s_ch * TY * SW); }
    __host__ __device__ static constexpr int off_U() { return 2 * QSZ; }
    __host__ __device__ static constexpr int off_D() { return 2 * QSZ + 2 * USZ; }
    __host__ __device__ static constexpr int off_S() { return 2 * QSZ + 4 * USZ; }
    __host__ __device__ static constexpr int off_R(int s_ch) { return off_S() + 2 * ssz(s_ch); }
    __host__ __device__ static constexpr int off_Uo(int s_ch) { return off_R(s_ch) + round32(3 * RING); }
    __host__ __device__ static constexpr int off_Qo(int s_ch) { return off_Uo(s_ch) + 2 * UOSZ; }
    __host__ __device__ static constexpr int off_X(int s_ch) { return off_Qo(s_ch) + QOB * QOSZ; }
    __host__ __device__ static constexpr int floats(int s_ch) { return off_X(s_ch) + XSZ; }
    __host__ __device__ static constexpr int bytes(int s_ch) { return floats(s_ch) * 4 + 32; }
};

__device__ __forceinline__ void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Flow step + projection of the thread's NFG flow nodes (channels f0 .. f0+NFG-1) at one voxel.
template <int NFG, int NF, int CAP, int OSTAGE, int TY>
__device__ __forceinline__ void flow_out_staged(const StagedArgs &a, const float *Rz, int f0, int roff, int rps,
                                                int rs, const float (&Mn)[NFG], bool has_z, int x, int y, int zg,
                                                const float (&qc)[3][NFG], const float (&svc)[NFG], float *qo,
                                                int64_t P) {
    const bool gxv = x < a.nx - 1, gyv = y < a.ny - 1, gzv = has_z && (zg < a.nzg - 1);
    const int Pi = OSTAGE ? TY * 32 : (int)P;  // channel stride: smem staging tile, or global (fits 32 bits)
#pragma unroll
    for (int v = 0; v < NFG; ++v) {
        const int f = f0 + v;
        const float mc = Rz[f * rps + roff];
        const float gx = gxv ? Rz[f * rps + roff + 1] - mc : 0.f;
        const float gy = gyv ? Rz[f * rps + roff + rs] - mc : 0.f;
        const float gz = gzv ? Mn[v] - mc : 0.f;
        float hx = qc[0][v], hy = qc[1][v], hz = qc[2][v];
        flow_step<CAP>(a.ctau, gx, gy, gz, svc[v], hx, hy, hz);
        if (OSTAGE) {
            qo[f * Pi] = hx;
            qo[(NF + f) * Pi] = hy;
            qo[(2 * NF + f) * Pi] = hz;
        } else {
            st_stream(qo + f * Pi, hx);
            st_stream(qo + (NF + f) * Pi, hy);
            st_stream(qo + (2 * NF + f) * Pi, hz);
        }
    }
}

template <int NI, int NL, int TY, int OSTAGE, int MODEL, int G>
__global__ void __launch_bounds__(32 * G *(TY + 2), 1) pf_iter_staged(const __grid_constant__ StagedArgs a) {
    using L = StagedLayout<NI, NL, TY, OSTAGE, MODEL, G>;
    constexpr int NF = L::NF;
    static_assert(G == 1 || (MODEL == 0 && NI == 0 && NL % G == 0), "label split only for Potts");
    constexpr int NLG = NL / G;   // end labels of this thread's group
    constexpr int NFG = NF / G;   // flow nodes of this thread's group
    constexpr int QW = L::QW, UW = L::UW, SW = L::SW, QROWS = L::QROWS, UROWS = L::UROWS;
    constexpr int QCS = QROWS * QW;   // q channel stride in smem
    constexpr int UCS = UROWS * UW;
    constexpr int RS = L::RS, RPS = L::RPS, RING = L::RING;
    extern __shared__ __align__(128) float sm[];
    float *Qs = sm;
    float *Us = sm + L::off_U();
    float *Ds = sm + L::off_D();
    float *Ss = sm + L::off_S();
    float *R = sm + L::off_R(a.s_ch);
    float *Uo = sm + L::off_Uo(a.s_ch);
    float *Qo = sm + L::off_Qo(a.s_ch);
    float *X = sm + L::off_X(a.s_ch);
    const int SSZ = L::ssz(a.s_ch);
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm + L::floats(a.s_ch));

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool is_main = warp < G * TY;
    const int grp = warp % G;
    int lx, ly, xr;  // tile coordinates of the thread's point; exchange row
    if (is_main) {
        lx = lane; ly = warp / G; xr = ly;
    } else if ((warp - G * TY) / G == 0) {  // bottom halo row
        lx = lane; ly = TY; xr = TY;
    } else {                                 // right halo column
        lx = (lane < TY) ? 32 : -1; ly = (lane < TY) ? lane : 0; xr = TY + 1;
    }
    const int l0 = grp * NLG, f0 = grp * NFG;  // first label / flow node of the group
    const int64_t P = (int64_t)a.pitch * a.ny;
    const int64_t qps = (int64_t)3 * NF * P;
    const int64_t ups = (int64_t)NL * P;
    const float k2 = kLog2e * a.inv_c;

    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_init(&bars[2], 1);  // OSTAGE 2: flow staging tile free
        fence_mbar_init();
        prefetch_tmap(&a.tm_q);
        prefetch_tmap(&a.tm_u);
        prefetch_tmap(&a.tm_D);
        if (a.s_ch) prefetch_tmap(&a.tm_S);
    }
    __syncthreads();

    auto issue = [&](int plane, int stage, int x0, int y0) {
        mbar_arrive_expect_tx(&bars[stage], a.tx_bytes);
        tma_load_4d(Qs + stage * L::QSZ, &a.tm_q, &bars[stage], x0 - 4, y0 - 1, 0, plane + 1);
        tma_load_4d(Us + stage * L::USZ, &a.tm_u, &bars[stage], x0, y0, 0, plane + 1);
        tma_load_4d(Ds + stage * L::USZ, &a.tm_D, &bars[stage], x0, y0, 0, plane);
        if (a.s_ch) tma_load_4d(Ss + stage * SSZ, &a.tm_S, &bars[stage], x0, y0, 0, plane);
    };
    const uint64_t pol_out = OSTAGE ? policy_evict_first() : 0;

    float resid = 0.f;
    int kbase = 0;   // planes consumed so far by this CTA (ring position / mbarrier parity)
    for (int item = blockIdx.x; item < a.items; item += gridDim.x) {
        const int chunk = item / a.tiles, tile = item - chunk * a.tiles;
        const int x0 = (tile % a.tiles_x) * 32, y0 = (tile / a.tiles_x) * TY;
        const int zc0 = chunk * a.zchunk, zc1 = min(zc0 + a.zchunk, a.nzl);
        const bool has_above = (a.zg0 + zc1) < a.nzg;
        const int pend = has_above ? zc1 : zc1 - 1;
        const int x = x0 + (lx < 0 ? 0 : lx), y = y0 + ly;
        const bool valid = (lx >= 0) && x < a.nx && y < a.ny;
        const int pix = valid ? y * a.pitch + x : 0;
        const int qoff = (ly + 1) * QW + (lx < 0 ? 0 : lx) + 4;
        const int uoff = ly * UW + (lx < 0 ? 0 : lx);
        const int roff = ly * RS + (lx < 0 ? 0 : lx);

        __syncthreads();  // previous item's readers of the ring / stage buffers are done
        if (tid == 0) {
            fence_proxy_async();
            issue(zc0, kbase & 1, x0, y0);
            if (zc0 + 1 <= pend) issue(zc0 + 1, (kbase + 1) & 1, x0, y0);
        }
        // q of the plane below the chunk (its z-component enters div of the first plane).  Two register
        // sets alternate between "current plane" and "plane awaiting its flow step" (no copies).
        float qA[3][NFG], qB[3][NFG];
        float sA[NFG], sB[NFG];
#pragma unroll
        for (int v = 0; v < NFG; ++v) { qA[0][v] = 0.f; qA[1][v] = 0.f; qA[2][v] = 0.f; sA[v] = 0.f; }
        if (valid && (a.zg0 + zc0) > 0) {
            const float *qb = a.q_in + (int64_t)(zc0 - 1) * qps + (2 * NF + f0) * P + pix;
#pragma unroll
            for (int v = 0; v < NFG; ++v) qA[2][v] = __ldg(qb + v * P);
        }

        auto plane_step = [&](const int p, float (&qc)[3][NFG], float (&svc)[NFG], float (&qn)[3][NFG],
                              float (&svn)[NFG]) {
            const int k = kbase + (p - zc0);
            const int st = k & 1;
            mbar_wait(&bars[st], (k >> 1) & 1);
            const float *Qb = Qs + st * L::QSZ;
            const float *Ub = Us + st * L::USZ;
            const float *Db = Ds + st * L::USZ;
            float *Rp = R + (p % 3) * RING;
            float Mv[NFG];
#pragma unroll
            for (int v = 0; v < NFG; ++v) svn[v] = 0.f;
            // ---------------- stage A(p): div, excess, label update, masses (tile + halo)
            float dq[NFG];
            float Dv[NLG], uold[NLG], ut[NLG], un[NLG];
            float dlab[G == 1 ? NI + NL : NLG];   // end-label excesses (G = 1: positions NI..)
            if (lx >= 0) {
#pragma unroll
                for (int v = 0; v < NFG; ++v) {
                    const int f = f0 + v;
                    const float qx = Qb[f * QCS + qoff];
                    const float qxm = Qb[f * QCS + qoff - 1];
                    const float qy = Qb[(NF + f) * QCS + qoff];
                    const float qym = Qb[(NF + f) * QCS + qoff - QW];
                    const float qz = Qb[(2 * NF + f) * QCS + qoff];
                    dq[v] = ((qx - qxm) + (qy - qym)) + (qz - qc[2][v]);
                    qn[0][v] = qx; qn[1][v] = qy; qn[2][v] = qz;
                }
#pragma unroll
                for (int l = 0; l < NLG; ++l) {
                    Dv[l] = Db[(l0 + l) * UCS + uoff];
                    uold[l] = Ub[(l0 + l) * UCS + uoff];
                }
            }
            float sum = 1.f;
            if constexpr (G == 1) {
                if (lx >= 0) {
                    label_excess<MODEL, NI, NL>(dq, Dv, dlab, a.g.w);
                    sum = label_update<NI, NL>(dlab, uold, ut, un, a.shift, k2);
                }
            } else {
                // Potts, labels l0 .. l0+NLG-1: d_L = D_L + div q_L; m and a exchanged with the partner warp
                float *xm = X + (xr * G) * 32 + lane;
                float *xa = X + ((TY + 2) * G + xr * G) * 32 + lane;
                float mpart = 0.f;
                if (lx >= 0) {
#pragma unroll
                    for (int l = 0; l < NLG; ++l) dlab[l] = Dv[l] + dq[l];
                    mpart = dlab[0];
#pragma unroll
                    for (int l = 1; l < NLG; ++l) mpart = fminf(mpart, dlab[l]);
                }
                if (a.shift == 0) {
                    xm[grp * 32] = mpart;
                    named_bar(1 + xr, 32 * G);
                    mpart = fminf(xm[0], xm[32]);
                } else {
                    mpart = 0.f;
                }
                float spart = 0.f;
                if (lx >= 0) {
#pragma unroll
                    for (int l = 0; l < NLG; ++l) {
                        ut[l] = uold[l] * ex2_approx((mpart - dlab[l]) * k2);
                        spart += ut[l];
                    }
                }
                xa[grp * 32] = spart;
                named_bar(1 + xr, 32 * G);
                sum = xa[0] + xa[32];
                const float inv = __frcp_rn(sum);
#pragma unroll
                for (int l = 0; l < NLG; ++l) {
                    const float nu = ut[l] * inv;
                    un[l] = nu < FLT_MIN ? 0.f : nu;
                }
            }
            if (lx >= 0) {
                if (is_main && valid && p < zc1) {
                    if (grp == 0 && (!(sum > 0.f) || !(sum <= FLT_MAX))) {
                        const unsigned long long vox = ((unsigned long long)(a.zg0 + p) * a.ny + y) * a.nx + x;
                        atomicMin(a.err_voxel, vox);
                    }
                    if (OSTAGE) {
                        float *uo = Uo + (p & 1) * L::UOSZ + ly * 32 + lx;
#pragma unroll
                        for (int l = 0; l < NLG; ++l) uo[(l0 + l) * TY * 32] = un[l];
                    } else {
                        float *uo = a.u_out + (int64_t)p * ups + pix;
#pragma unroll
                        for (int l = 0; l < NLG; ++l) st_stream(uo + (l0 + l) * (int)P, un[l]);
                    }
#pragma unroll
                    for (int l = 0; l < NLG; ++l) resid = fmaxf(resid, fabsf(un[l] - uold[l]));
                }
                if constexpr (G == 1) {
                    node_masses<MODEL, NI, NL>(ut, Mv, a.g.w);
                } else {
#pragma unroll
                    for (int l = 0; l < NLG; ++l) Mv[l] = ut[l];
                }
#pragma unroll
                for (int v = 0; v < NFG; ++v) Rp[(f0 + v) * RPS + roff] = Mv[v];
                if (is_main) {
                    const float *Sb = Ss + st * SSZ + ly * SW + lx;
                    if (a.s_ch == 0) {
#pragma unroll
                        for (int v = 0; v < NFG; ++v) svn[v] = a.g.s[f0 + v];
                    } else if (a.s_ch == 1) {  // shared field x per-node factor (1 for a plain shared field)
                        const float sv = Sb[0];
#pragma unroll
                        for (int v = 0; v < NFG; ++v) svn[v] = sv * a.g.s[f0 + v];
                    } else {
#pragma unroll
                        for (int v = 0; v < NFG; ++v) svn[v] = Sb[(f0 + v) * TY * SW];
                    }
                }
            }
            if (OSTAGE) {
                fence_proxy_async();                // staged outputs -> visible to the TMA (async proxy)
                if (tid == 0) bulk_wait_read_all(); // stores of the buffers about to be rewritten have read them
            }
            __syncthreads();  // ring slot p complete; stage st fully consumed; staged outputs complete
            if (tid == 0) {
                if (p + 2 <= pend) {
                    fence_proxy_async();
                    issue(p + 2, st, x0, y0);
                }
                if (OSTAGE) {
                    if (p < zc1) tma_store_4d(&a.tm_uo, Uo + (p & 1) * L::UOSZ, x0, y0, 0, p + 1, pol_out);
                    if (p - 2 >= zc0)
                        tma_store_4d(&a.tm_qo, Qo + (OSTAGE == 1 ? (p & 1) : 0) * L::QOSZ, x0, y0, 0, p - 1, pol_out);
                    bulk_commit();
                }
                if (OSTAGE == 2) {  // the single flow staging tile may be rewritten once the store has read it
                    bulk_wait_read_all();
                    mbar_arrive(&bars[2]);
                }
            }
            // ---------------- stage B(p-1): flow step + projection of plane p-1
            if (OSTAGE == 2 && is_main && p > zc0) mbar_wait(&bars[2], k & 1);
            if (is_main && valid && p > zc0) {
                const int z = p - 1;
                const float *Rz = R + (z % 3) * RING;
                float *qo = OSTAGE ? Qo + (OSTAGE == 1 ? (z & 1) : 0) * L::QOSZ + ly * 32 + lx
                                   : a.q_out + (int64_t)z * qps + pix;
                if (a.cap == 0)
                    flow_out_staged<NFG, NF, 0, OSTAGE, TY>(a, Rz, f0, roff, RPS, RS, Mv, true, x, y, a.zg0 + z, qc,
                                                            svc, qo, P);
                else
                    flow_out_staged<NFG, NF, 1, OSTAGE, TY>(a, Rz, f0, roff, RPS, RS, Mv, true, x, y, a.zg0 + z, qc,
                                                            svc, qo, P);
            }
        };
        int p = zc0;
        for (; p + 1 <= pend; p += 2) {
            plane_step(p, qA, sA, qB, sB);
            plane_step(p + 1, qB, sB, qA, sA);
        }
        const bool last_in_B = p <= pend;
        if (last_in_B) plane_step(p, qA, sA, qB, sB);
        // last plane of the volume: no plane above, nabla_z = 0
        auto tail_step = [&](const float (&qc)[3][NFG], const float (&svc)[NFG]) {
            const int z = zc1 - 1;
            const float *Rz = R + (z % 3) * RING;
            float *qo = OSTAGE ? Qo + (OSTAGE == 1 ? (z & 1) : 0) * L::QOSZ + ly * 32 + lx
                               : a.q_out + (int64_t)z * qps + pix;
            float Mdummy[NFG];
#pragma unroll
            for (int v = 0; v < NFG; ++v) Mdummy[v] = 0.f;
            if (a.cap == 0)
                flow_out_staged<NFG, NF, 0, OSTAGE, TY>(a, Rz, f0, roff, RPS, RS, Mdummy, false, x, y, a.zg0 + z,
                                                        qc, svc, qo, P);
            else
                flow_out_staged<NFG, NF, 1, OSTAGE, TY>(a, Rz, f0, roff, RPS, RS, Mdummy, false, x, y, a.zg0 + z,
                                                        qc, svc, qo, P);
        };
        if (!has_above) {
            if (OSTAGE == 1) {  // the store issued at the last plane step may still be reading the tail's buffer
                if (tid == 0) bulk_wait_read_all();
                __syncthreads();
            } else if (OSTAGE == 2) {  // single tile: store the last stepped plane before the tail rewrites it
                fence_proxy_async();
                __syncthreads();
                if (tid == 0) {
                    if (pend - 1 >= zc0) tma_store_4d(&a.tm_qo, Qo, x0, y0, 0, pend, pol_out);
                    bulk_commit();
                    bulk_wait_read_all();
                }
                __syncthreads();
            }
            if (is_main && valid) {
                if (last_in_B) tail_step(qB, sB);
                else tail_step(qA, sA);
            }
        }
        if (OSTAGE) {  // flush the item's last staged flow planes
            fence_proxy_async();
            __syncthreads();
            if (tid == 0) {
                for (int z = OSTAGE == 1 ? max(zc0, pend - 1) : zc1 - 1; z < zc1; ++z)
                    tma_store_4d(&a.tm_qo, Qo + (OSTAGE == 1 ? (z & 1) : 0) * L::QOSZ, x0, y0, 0, z + 1, pol_out);
                bulk_commit();
                bulk_wait_read_all();
            }
        }
        kbase += pend - zc0 + 1;
    }
    if (OSTAGE && tid == 0) bulk_wait_all();
    if (a.check) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) resid = fmaxf(resid, __shfl_xor_sync(0xffffffffu, resid, o));
        if (lane == 0 && resid > 0.f) atomicMax(a.resid_bits, __float_as_uint(resid));
    }
}

struct StagedKernelInfo {
    const void *func;
    int threads;
    int smem_bytes;  // with s_ch = 0; add 2 * round32(s_ch * tile_y * 32) floats for an S field
    int tile_y;
    int ostage;      // 1: outputs staged in smem and written by TMA stores
    int groups;      // label groups per row (G)
};

bool staged_kernel_lookup(int NI, int NL, int MODEL, StagedKernelInfo *info);

}  // namespace pf
