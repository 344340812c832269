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
//   * OSTAGE: the new u and q are staged in shared memory and written by TMA bulk-tensor stores with an
//     evict-first L2 policy (no per-thread 64-bit address arithmetic, no L2 pollution).  u always as
//     one double-buffered tile per plane, issued by thread 0 at the plane barrier.  q: OSTAGE 1
//     double-buffers the flow tile the same way; OSTAGE 2 (many nodes, tight shared memory) has ONE
//     flow row per main warp, which the warp hands to the TMA unit itself at the end of its flow step.
//     Bulk-store groups are per thread, so lane 0 only waits for its own previous row store -- issued a
//     whole stage-A phase earlier -- and no CTA-wide barrier or single-thread drain sits on the
//     critical path (a single CTA-wide flow tile stalled every plane on the store's shared-memory read).
//     OSTAGE 0 stores straight from registers.
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
    unsigned long long *ticket;       // monotone work-item ticket counter (never reset)
    unsigned long long ticket_base;   // its value at the start of this launch
    GraphConst g;
};

__host__ __device__ constexpr int round32(int n) { return (n + 31) / 32 * 32; }

template <int NI, int NL, int TY, int OSTAGE, int MODEL, int G>
struct StagedLayout {
    static_assert(G == 1, "one label group per voxel row");
    static_assert(OSTAGE >= 0 && OSTAGE <= 2, "OSTAGE: 0 direct, 1 tile stores, 2 tile u + per-warp q rows");
    static constexpr int NV = NI + NL;
    static constexpr int NF = Model<MODEL, NI, NL>::NF;   // flow-carrying nodes
    static constexpr int QW = 40, UW = 36, SW = 32;
    static constexpr int QROWS = TY + 2, UROWS = TY + 1;
    static constexpr int QSZ = round32(3 * NF * QROWS * QW);  // floats per stage
    static constexpr int USZ = round32(NL * UROWS * UW);
    static constexpr int RS = 33, RPS = (TY + 1) * RS, RING = NF * RPS;
    static constexpr int UOSZ = OSTAGE ? round32(NL * TY * 32) : 0;       // u staging [l][row][32], x2
    static constexpr int QOSZ = OSTAGE ? round32(3 * NF * TY * 32) : 0;   // q staging: OSTAGE 1 [ch][row][32] x2,
    static constexpr int QOB = OSTAGE == 1 ? 2 : 1;                         //            OSTAGE 2 [row][ch][32] x1
    static constexpr int kThreads = 32 * (TY + 2);
    // runtime part: the S staging ring holds s_ch channels (0, 1 or NF)
    __host__ __device__ static constexpr int ssz(int s_ch) { return round32(s_ch * TY * SW); }
    __host__ __device__ static constexpr int off_U() { return 2 * QSZ; }
    __host__ __device__ static constexpr int off_D() { return 2 * QSZ + 2 * USZ; }
    __host__ __device__ static constexpr int off_S() { return 2 * QSZ + 4 * USZ; }
    __host__ __device__ static constexpr int off_R(int s_ch) { return off_S() + 2 * ssz(s_ch); }
    __host__ __device__ static constexpr int off_Uo(int s_ch) { return off_R(s_ch) + round32(3 * RING); }
    __host__ __device__ static constexpr int off_Qo(int s_ch) { return off_Uo(s_ch) + 2 * UOSZ; }
    __host__ __device__ static constexpr int floats(int s_ch) { return off_Qo(s_ch) + QOB * QOSZ; }
    __host__ __device__ static constexpr int bytes(int s_ch) { return floats(s_ch) * 4 + 32; }
};

// Flow step + projection of the thread's NF flow nodes at one voxel (P:148 / P:298).  qo: the thread's
// slot in the staging row (channel stride 32) or its global address (channel stride P).
template <int NF, int CAP, int OSTAGE>
__device__ __forceinline__ void flow_out_staged(const StagedArgs &a, const float *Rz, int roff, int rps, int rs,
                                                const float (&Mn)[NF], bool has_z, int x, int y, int zg,
                                                const float (&qc)[3][NF], const float (&svc)[NF], float *qo,
                                                int Pi /* channel stride: staging, or global (fits 32 bits) */) {
    const bool gxv = x < a.nx - 1, gyv = y < a.ny - 1, gzv = has_z && (zg < a.nzg - 1);
#pragma unroll
    for (int f = 0; f < NF; ++f) {
        const float mc = Rz[f * rps + roff];
        const float gx = gxv ? Rz[f * rps + roff + 1] - mc : 0.f;
        const float gy = gyv ? Rz[f * rps + roff + rs] - mc : 0.f;
        const float gz = gzv ? Mn[f] - mc : 0.f;
        float hx = qc[0][f], hy = qc[1][f], hz = qc[2][f];
        flow_step<CAP>(a.ctau, gx, gy, gz, svc[f], hx, hy, hz);
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

// Per-warp staged output row: lane 0 waits until this warp's previous bulk store from the same row has
// read it.  `since` = bulk groups this warp committed after that store (the u and q rows alternate, so
// it is 0 or 1 except across item boundaries); waiting for all but the newest group is enough when
// since >= 1 and never waits for the other row's just-issued store.
__device__ __forceinline__ void stage_row_acquire(int lane, int since) {
    if (lane == 0) {
        if (since >= 1) bulk_wait_read_but1();
        else bulk_wait_read_all();
    }
    __syncwarp();
}

// ... and hands the written row (plane coordinate cz of the tensor map) to the TMA unit.
__device__ __forceinline__ void stage_row_release(int lane, const CUtensorMap *map, const float *row, int x0, int y,
                                                  int cz, uint64_t pol) {
    fence_proxy_async();  // this thread's generic-proxy writes -> visible to the async proxy
    __syncwarp();
    if (lane == 0) {
        tma_store_4d(map, row, x0, y, 0, cz, pol);
        bulk_commit();
    }
}

template <int NI, int NL, int TY, int OSTAGE, int MODEL, int G>
__global__ void __launch_bounds__(32 * (TY + 2), 1) pf_iter_staged(const __grid_constant__ StagedArgs a) {
    using L = StagedLayout<NI, NL, TY, OSTAGE, MODEL, G>;
    constexpr int NF = L::NF;
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
    const int SSZ = L::ssz(a.s_ch);
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm + L::floats(a.s_ch));

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool is_main = warp < TY;
    int lx, ly;  // tile coordinates of the thread's point
    if (is_main) {
        lx = lane; ly = warp;
    } else if (warp == TY) {  // bottom halo row
        lx = lane; ly = TY;
    } else {                  // right halo column
        lx = (lane < TY) ? 32 : -1; ly = (lane < TY) ? lane : 0;
    }
    const int64_t P = (int64_t)a.pitch * a.ny;
    const int64_t qps = (int64_t)3 * NF * P;
    const int64_t ups = (int64_t)NL * P;
    const float k2 = kLog2e * a.inv_c;
    float *qo_row = Qo + ly * 3 * NF * 32 + lane;   // OSTAGE 2, main warps: the thread's flow staging slots

    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
        prefetch_tmap(&a.tm_q);
        prefetch_tmap(&a.tm_u);
        prefetch_tmap(&a.tm_D);
        if (a.s_ch) prefetch_tmap(&a.tm_S);
        if (OSTAGE) {
            prefetch_tmap(&a.tm_uo);
            prefetch_tmap(&a.tm_qo);
        }
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
    int since_q = 1 << 20;  // bulk groups this thread committed after its last q row store (OSTAGE 2)
    int kbase = 0;   // planes consumed so far by this CTA (ring position / mbarrier parity)
    // Dynamic work queue: a CTA takes the next ticket when it starts an item, so the items in flight are
    // always a window of ~gridDim consecutive tiles and the halo lines one tile loads from HBM are still in
    // L2 when its neighbours read them (a static round-robin lets CTAs drift apart by whole items on
    // many-item volumes, which sent ~40 % extra halo traffic to HBM on 768^2 planes).  Every launch
    // consumes exactly items + gridDim tickets (one failed grab per CTA), so the host knows the base.
    __shared__ int s_item;
    auto grab = [&]() -> int {
        const unsigned long long t = atomicAdd(a.ticket, 1ull) - a.ticket_base;
        return t < (unsigned long long)a.items ? (int)t : a.items;
    };
    if (tid == 0) s_item = grab();
    __syncthreads();
    for (int item = s_item; item < a.items; item = s_item) {
        const int chunk = item / a.tiles, tile = item - chunk * a.tiles;
        const int x0 = (tile % a.tiles_x) * 32, y0 = (tile / a.tiles_x) * TY;
        const int zc0 = chunk * a.zchunk, zc1 = min(zc0 + a.zchunk, a.nzl);
        const bool has_above = (a.zg0 + zc1) < a.nzg;
        const int pend = has_above ? zc1 : zc1 - 1;
        const int x = x0 + (lx < 0 ? 0 : lx), y = y0 + ly;
        const bool valid = (lx >= 0) && x < a.nx && y < a.ny;
        const bool row_out = is_main && y < a.ny;   // warp-uniform: this warp owns an output row
        const int pix = valid ? y * a.pitch + x : 0;
        const int qoff = (ly + 1) * QW + (lx < 0 ? 0 : lx) + 4;
        const int uoff = ly * UW + (lx < 0 ? 0 : lx);
        const int roff = ly * RS + (lx < 0 ? 0 : lx);

        __syncthreads();  // previous item's readers of the ring / stage buffers (and of s_item) are done
        if (tid == 0) {
            s_item = grab();  // next item; read by all threads after this item's plane barriers
            fence_proxy_async();
            issue(zc0, kbase & 1, x0, y0);
            if (zc0 + 1 <= pend) issue(zc0 + 1, (kbase + 1) & 1, x0, y0);
        }
        // q of the plane below the chunk (its z-component enters div of the first plane).  Two register
        // sets alternate between "current plane" and "plane awaiting its flow step" (no copies).
        float qA[3][NF], qB[3][NF];
        float sA[NF], sB[NF];
#pragma unroll
        for (int v = 0; v < NF; ++v) { qA[0][v] = 0.f; qA[1][v] = 0.f; qA[2][v] = 0.f; sA[v] = 0.f; }
        if (valid && (a.zg0 + zc0) > 0) {
            const float *qb = a.q_in + (int64_t)(zc0 - 1) * qps + (2 * NF) * P + pix;
#pragma unroll
            for (int v = 0; v < NF; ++v) qA[2][v] = __ldg(qb + v * P);
        }

        // flow step + projection of plane z (stage B); Mn = M(z+1) at the voxel (unused when !has_z)
        auto stage_b = [&](const int z, const float (&Mn)[NF], bool has_z, const float (&qc)[3][NF],
                           const float (&svc)[NF]) {
            const float *Rz = R + (z % 3) * RING;
            if (OSTAGE == 2) {
                if (row_out) {
                    stage_row_acquire(lane, since_q);
                    if (valid) {
                        if (a.cap == 0)
                            flow_out_staged<NF, 0, 1>(a, Rz, roff, RPS, RS, Mn, has_z, x, y, a.zg0 + z, qc, svc,
                                                      qo_row, 32);
                        else
                            flow_out_staged<NF, 1, 1>(a, Rz, roff, RPS, RS, Mn, has_z, x, y, a.zg0 + z, qc, svc,
                                                      qo_row, 32);
                    }
                    stage_row_release(lane, &a.tm_qo, Qo + ly * 3 * NF * 32, x0, y, z + 1, pol_out);
                    since_q = 0;
                }
            } else if (is_main && valid) {
                float *qo = OSTAGE ? Qo + (z & 1) * L::QOSZ + ly * 32 + lx : a.q_out + (int64_t)z * qps + pix;
                const int Pi = OSTAGE ? TY * 32 : (int)P;
                if (a.cap == 0)
                    flow_out_staged<NF, 0, OSTAGE>(a, Rz, roff, RPS, RS, Mn, has_z, x, y, a.zg0 + z, qc, svc, qo, Pi);
                else
                    flow_out_staged<NF, 1, OSTAGE>(a, Rz, roff, RPS, RS, Mn, has_z, x, y, a.zg0 + z, qc, svc, qo, Pi);
            }
        };

        auto plane_step = [&](const int p, float (&qc)[3][NF], float (&svc)[NF], float (&qn)[3][NF],
                              float (&svn)[NF]) {
            const int k = kbase + (p - zc0);
            const int st = k & 1;
            mbar_wait(&bars[st], (k >> 1) & 1);
            const float *Qb = Qs + st * L::QSZ;
            const float *Ub = Us + st * L::USZ;
            const float *Db = Ds + st * L::USZ;
            float *Rp = R + (p % 3) * RING;
            float Mv[NF];
#pragma unroll
            for (int v = 0; v < NF; ++v) svn[v] = 0.f;
            // ---------------- stage A(p): div, excess, label update, masses (tile + halo)
            float dq[NF];
            float Dv[NL], uold[NL], ut[NL], un[NL];
            float dlab[NI + NL];   // end-label excesses at positions NI..
            float sum = 1.f;
            if (lx >= 0) {
#pragma unroll
                for (int f = 0; f < NF; ++f) {
                    const float qx = Qb[f * QCS + qoff];
                    const float qxm = Qb[f * QCS + qoff - 1];
                    const float qy = Qb[(NF + f) * QCS + qoff];
                    const float qym = Qb[(NF + f) * QCS + qoff - QW];
                    const float qz = Qb[(2 * NF + f) * QCS + qoff];
                    dq[f] = ((qx - qxm) + (qy - qym)) + (qz - qc[2][f]);
                    qn[0][f] = qx; qn[1][f] = qy; qn[2][f] = qz;
                }
#pragma unroll
                for (int l = 0; l < NL; ++l) {
                    Dv[l] = Db[l * UCS + uoff];
                    uold[l] = Ub[l * UCS + uoff];
                }
                label_excess<MODEL, NI, NL>(dq, Dv, dlab, a.g.w);
                sum = label_update<NI, NL>(dlab, uold, ut, un, a.shift, k2);
            }
            if (lx >= 0) {
                if (p < zc1) {
                    if (OSTAGE) {
                        if (is_main && valid) {
                            float *uo = Uo + (p & 1) * L::UOSZ + ly * 32 + lx;
#pragma unroll
                            for (int l = 0; l < NL; ++l) uo[l * TY * 32] = un[l];
                        }
                    } else if (is_main && valid) {
                        float *uo = a.u_out + (int64_t)p * ups + pix;
#pragma unroll
                        for (int l = 0; l < NL; ++l) st_stream(uo + l * (int)P, un[l]);
                    }
                    if (is_main && valid) {
                        if (!(sum > 0.f) || !(sum <= FLT_MAX)) {
                            const unsigned long long vox = ((unsigned long long)(a.zg0 + p) * a.ny + y) * a.nx + x;
                            atomicMin(a.err_voxel, vox);
                        }
#pragma unroll
                        for (int l = 0; l < NL; ++l) resid = fmaxf(resid, fabsf(un[l] - uold[l]));
                    }
                }
                node_masses<MODEL, NI, NL>(ut, Mv, a.g.w);
#pragma unroll
                for (int v = 0; v < NF; ++v) Rp[v * RPS + roff] = Mv[v];
                if (is_main) {
                    const float *Sb = Ss + st * SSZ + ly * SW + lx;
                    if (a.s_ch == 0) {
#pragma unroll
                        for (int v = 0; v < NF; ++v) svn[v] = a.g.s[v];
                    } else if (a.s_ch == 1) {  // shared field x per-node factor (1 for a plain shared field)
                        const float sv = Sb[0];
#pragma unroll
                        for (int v = 0; v < NF; ++v) svn[v] = sv * a.g.s[v];
                    } else {
#pragma unroll
                        for (int v = 0; v < NF; ++v) svn[v] = Sb[v * TY * SW];
                    }
                }
            }
            if (OSTAGE) {
                fence_proxy_async();                // staged u -> visible to the TMA (async proxy)
                if (tid == 0) bulk_wait_read_all(); // stores of the buffers about to be rewritten have read them
            }
            __syncthreads();  // ring slot p complete; stage st fully consumed; staged u complete
            if (tid == 0) {
                if (p + 2 <= pend) {
                    fence_proxy_async();
                    issue(p + 2, st, x0, y0);
                }
                if (OSTAGE) {
                    if (p < zc1) tma_store_4d(&a.tm_uo, Uo + (p & 1) * L::UOSZ, x0, y0, 0, p + 1, pol_out);
                    if (OSTAGE == 1 && p - 2 >= zc0)
                        tma_store_4d(&a.tm_qo, Qo + (p & 1) * L::QOSZ, x0, y0, 0, p - 1, pol_out);
                    bulk_commit();
                    ++since_q;
                }
            }
            // ---------------- stage B(p-1): flow step + projection of plane p-1
            if (p > zc0) stage_b(p - 1, Mv, true, qc, svc);
        };
        int p = zc0;
        for (; p + 1 <= pend; p += 2) {
            plane_step(p, qA, sA, qB, sB);
            plane_step(p + 1, qB, sB, qA, sA);
        }
        const bool last_in_B = p <= pend;
        if (last_in_B) plane_step(p, qA, sA, qB, sB);
        // last plane of the volume: no plane above, nabla_z = 0
        if (!has_above) {
            if (OSTAGE == 1) {  // the store issued at the last plane step may still be reading the tail's buffer
                if (tid == 0) bulk_wait_read_all();
                __syncthreads();
            }
            float Mdummy[NF];
#pragma unroll
            for (int v = 0; v < NF; ++v) Mdummy[v] = 0.f;
            if (last_in_B) stage_b(zc1 - 1, Mdummy, false, qB, sB);
            else stage_b(zc1 - 1, Mdummy, false, qA, sA);
        }
        if (OSTAGE == 1) {  // flush the item's last staged flow planes
            fence_proxy_async();
            __syncthreads();
            if (tid == 0) {
                for (int z = max(zc0, pend - 1); z < zc1; ++z)
                    tma_store_4d(&a.tm_qo, Qo + (z & 1) * L::QOSZ, x0, y0, 0, z + 1, pol_out);
                bulk_commit();
            }
        }
        // the next item rewrites the u (and OSTAGE 1 flow) tiles: their stores must have read them
        // (ordered before the other threads by the barrier at the top of the next item)
        if (OSTAGE && tid == 0) bulk_wait_read_all();
        kbase += pend - zc0 + 1;
    }
    if (OSTAGE && lane == 0) bulk_wait_all();
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
