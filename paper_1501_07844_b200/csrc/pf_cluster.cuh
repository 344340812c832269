// pf_cluster.cuh -- cluster-split version of the fused Potts iteration (Alg. 1) for many labels.
//
// Why: with K = 16 labels one CTA per tile cannot stage more than a 32 x 4 tile in 227 KB of shared
// memory (the flow staging alone is 2 x 3K x (TY+2) x 40 floats), and 32 x 4 tiles leave the SM with 6-12
// warps and a 50 % halo overhead.  Here a CLUSTER of two CTAs (two SMs) shares one 32 x TY tile: CTA rank r
// stages, updates and stores only the labels [r K/2, (r+1) K/2), i.e. each SM does the work of a K/2-label
// problem on a TY = 8 tile.  The Potts label update couples the labels of a voxel only through
//   m(x) = min_L d_L(x)   and   a(x) = sum_L u~_L(x)        (Eq. 7; reading R1)
// so per plane each CTA writes its half's shift m_h, maximum T_h and sum s_h (label_half, pf_math.cuh; u is
// stored as lambda = log2 u) of every point of the tile (+halo) into the partner's shared memory with one
// 16-byte st.async (DSMEM), each exchange completing a transaction-counted mbarrier of the receiver (no
// cluster-wide barrier per plane).  Both CTAs then combine the two triples exactly as label_update's split
// form does (label_halves_combine), so the result is bitwise that of the one-CTA kernels.  Everything else -- the TMA z-march, the M ring, the
// flow step of plane p-1, the staged TMA stores, the ticket queue (one ticket per cluster) -- is the
// staged kernel's (pf_staged.cuh), restricted to the CTA's labels.
#pragma once
#include "pf_staged.cuh"

// Early refill of the input stage (experiments): every warp but warp 0 signals "stage read" on named barrier
// kStageBar right after its shared-memory reads of the plane (bar.arrive, no wait); warp 0 waits for them
// (bar.sync) -- 1: after its label_half, 2: after the exchange wait -- and thread 0 then issues the loads of plane
// p + 2 instead of at the plane barrier.
#ifndef PF_EARLY_ISSUE
#define PF_EARLY_ISSUE 2
#endif

namespace pf {

constexpr int kStageBar = 14;

__device__ __forceinline__ void named_arrive(int id, int nthreads) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// address of the same shared-memory word in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_to_rank(const void *p, uint32_t rank) {
    uint32_t out;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(smem_u32(p)), "r"(rank));
    return out;
}

__device__ __forceinline__ void st_cluster(uint32_t addr, float v) {
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void st_cluster_s32(uint32_t addr, int v) {
    asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// asynchronous 4-byte store into the partner CTA's shared memory; completion is counted on the partner's
// mbarrier (complete_tx) -- no memory fence on the producer side (a barrier.cluster.arrive.release after
// plain st.shared::cluster stores spent 40 % of all stall samples in MEMBAR/ERRBAR)
__device__ __forceinline__ void st_async_f32(uint32_t addr, float v, uint32_t mbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(addr),
                 "r"(__float_as_uint(v)), "r"(mbar)
                 : "memory");
}

// the (m_h, T_h, s_h) triple of one point as ONE 16-byte st.async (4th word unused)
__device__ __forceinline__ void st_async_f32x4(uint32_t addr, float v0, float v1, float v2, uint32_t mbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(addr),
                 "r"(__float_as_uint(v0)), "r"(__float_as_uint(v1)), "r"(__float_as_uint(v2)), "r"(0u), "r"(mbar)
                 : "memory");
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int NL, int TY, int DBF>
struct ClusterLayout {
    static constexpr int NLC = NL / 2;     // labels (= flow nodes, Potts) of one CTA
    static constexpr int NLCP = (NLC + 1) & ~1;   // q-stage k-block stride in channels: 128-byte aligned TMA dst
    using L = StagedLayout<0, NLCP, TY, 1, 0, 1>;
    static constexpr int XPTS = round32((TY + 1) * 33);   // exchange slots: tile + halo points
    __host__ __device__ static constexpr int off_X(int s_ch) { return L::floats(s_ch); }
    __host__ __device__ static constexpr int floats(int s_ch) { return off_X(s_ch) + 8 * XPTS; }   // (m, T, s, -) x 2
    __host__ __device__ static constexpr int bytes(int s_ch) { return floats(s_ch) * 4 + 32; }   // + 4 mbarriers
};

// tm_q / tm_u / tm_D / tm_uo / tm_qo boxes have NL/2 channels here; q channel of (k, label) = k*NL + label.
template <int NL, int TY, int DBF, int UH>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(32 * (TY + 2), 1)
    pf_iter_cluster(const __grid_constant__ StagedArgs a) {
    using CL = ClusterLayout<NL, TY, DBF>;
    using L = typename CL::L;
    constexpr int NLC = CL::NLC, NLCP = CL::NLCP, NF = NL;
    constexpr int QW = L::QW, UW = L::UW, SW = L::SW, QROWS = L::QROWS, UROWS = L::UROWS;
    constexpr int QCS = QROWS * QW, UCS = UROWS * UW;
    constexpr int RS = L::RS, RPS = L::RPS, RING = L::RING;
    static_assert(NL % 2 == 0 && NLC <= 8, "cluster split: even K <= 16");
    extern __shared__ __align__(128) float sm[];
    float *Qs = sm;
    float *Us = sm + L::off_U();
    float *Ds = sm + L::off_D();
    float *Ss = sm + L::off_S();
    float *R = sm + L::off_R(a.s_ch);
    float *Uo = sm + L::off_Uo(a.s_ch);
    float *Qo = sm + L::off_Qo(a.s_ch);
    // partner's (m_h, T_h, s_h) per point, written remotely; double-buffered by plane parity because the
    // partner may run up to one plane ahead (its sends for plane k+1 need only OUR sends for plane k)
    float *X2 = sm + CL::off_X(a.s_ch);       // [parity][XPTS][(m_h, T_h, s_h, -)]
    const int SSZ = L::ssz(a.s_ch);
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm + CL::floats(a.s_ch));

    const uint32_t rank = cluster_rank(), other = rank ^ 1u;
    const int lb = (int)rank * NLC;           // first (global) label of this CTA
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool is_main = warp < TY;
    int lx, ly;
    if (is_main) {
        lx = lane; ly = warp;
    } else if (warp == TY) {
        lx = lane; ly = TY;
    } else {
        lx = (lane < TY) ? 32 : -1; ly = (lane < TY) ? lane : 0;
    }
    const int64_t P = (int64_t)a.pitch * a.ny;
    const int64_t qps = (int64_t)3 * NF * P;
    const float k2 = kLog2e * a.inv_c;
    const int xpt = ly * 33 + (lx < 0 ? 0 : lx);             // this point's exchange slot
    const uint32_t x_remote = map_to_rank(X2 + 4 * xpt, other);
    const uint32_t barx_remote = map_to_rank(&bars[2], other);   // partner's "(m_h, T_h, s_h) received" mbarriers
    constexpr uint32_t kXBuf = 16u * CL::XPTS;                     // byte stride of the parity buffers
    constexpr uint32_t kXBytes = 16u * (32 * TY + 32 + TY);       // one 16-byte triple per tile + halo point

    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_init(&bars[2], 1);
        mbar_init(&bars[3], 1);
        fence_mbar_init();
        prefetch_tmap(&a.tm_q);
        prefetch_tmap(&a.tm_u);
        prefetch_tmap(&a.tm_D);
        if (a.s_ch) prefetch_tmap(&a.tm_S);
        prefetch_tmap(&a.tm_uo);
        prefetch_tmap(&a.tm_qo);
    }
    __syncthreads();

    // inputs of plane step `seq` (plane `plane` of the tile at (x0, y0)) into stage seq & 1, S slot seq & 3
    auto issue = [&](int plane, int seq, int x0, int y0) {
        const int stage = seq & 1;
        mbar_arrive_expect_tx(&bars[stage], a.tx_bytes);
#pragma unroll
        for (int k = 0; k < 3; ++k)
            tma_load_4d(Qs + stage * L::QSZ + k * NLCP * QCS, &a.tm_q, &bars[stage], x0 - 4, y0 - 1, k * NF + lb,
                        plane + 1);
        tma_load_4d(Us + stage * L::USZ, &a.tm_u, &bars[stage], x0, y0, lb, plane + 1);
        tma_load_4d(Ds + stage * L::USZ, &a.tm_D, &bars[stage], x0, y0, lb, plane);
        if (a.s_ch) tma_load_4d(Ss + (seq & 3) * SSZ, &a.tm_S, &bars[stage], x0, y0, 0, plane);
    };
    const uint64_t pol_out = policy_evict_first();

    float resid = 0.f;
    int kbase = 0;
    // One ticket per cluster: rank 0 grabs it and publishes it to both CTAs before a cluster barrier.  The
    // (n+1)-th item of the cluster is taken at the start of its n-th, so the refills of the n-th item's last two
    // plane steps can already load the (n+1)-th item's first two planes (no pipeline bubble between items; the
    // plane steps carry a sequence number k across items: stage k & 1, S slot k & 3).
    __shared__ int s_item[2];
    if (blockIdx.x == 0 && tid == 0) *a.ticket_next = 0ull;   // the next launch's counter (see pf_staged.cuh)
    auto grab_publish = [&](int slot) {
        if (rank == 0 && tid == 0) {
            const unsigned long long t = atomicAdd(a.ticket, 1ull);
            const int it = t < (unsigned long long)(a.items - a.item_begin) ? a.item_begin + (int)t : a.items;
            s_item[slot] = it;
            st_cluster_s32(map_to_rank(&s_item[slot], 1), it);
        }
    };
    grab_publish(0);
    cluster_sync_all();
    int nit = 0, prev_steps = 0;
    for (int item = s_item[0]; item < a.items; item = s_item[(++nit) & 1]) {
        const ItemGeom cg = item_geom(a, item, TY);
        const int x0 = cg.x0, y0 = cg.y0, zc0 = cg.zc0, zc1 = cg.zc1, pend = cg.pend;
        const bool has_above = cg.has_above;
        const int x = x0 + (lx < 0 ? 0 : lx), y = y0 + ly;
        const bool valid = (lx >= 0) && x < a.nx && y < a.ny;
        const int pix = valid ? y * a.pitch + x : 0;
        const int qoff = (ly + 1) * QW + (lx < 0 ? 0 : lx) + 4;
        const int uoff = ly * UW + (lx < 0 ? 0 : lx);
        const int roff = ly * RS + (lx < 0 ? 0 : lx);

        // next item (its slot was last read two items ago); after the barrier both CTAs see it, and both have
        // finished the previous item's readers of the ring / staging buffers
        grab_publish((nit + 1) & 1);
        cluster_sync_all();
        const int nxt = s_item[(nit + 1) & 1];
        const ItemGeom ng = item_geom(a, nxt < a.items ? nxt : a.item_begin, TY);
        const int nsteps_next = nxt < a.items ? ng.steps() : 0;
        if (tid == 0) {   // the item's first planes the previous item's last steps did not prefetch
            fence_proxy_async();
            const int n0 = min(prev_steps >= 2 ? 0 : 2 - prev_steps, cg.steps());
            for (int i = 0; i < n0; ++i) issue(zc0 + i, kbase + i, x0, y0);
        }
        float qA[3][NLC], qB[3][NLC];
#pragma unroll
        for (int v = 0; v < NLC; ++v) { qA[0][v] = 0.f; qA[1][v] = 0.f; qA[2][v] = 0.f; }
        if (valid && (a.zg0 + zc0) > 0) {
            const float *qb = a.q_in + (int64_t)(zc0 - 1) * qps + (2 * NF + lb) * P + pix;
#pragma unroll
            for (int v = 0; v < NLC; ++v) qA[2][v] = __ldg(qb + v * P);
        }

        auto stage_b = [&](const int z, const float (&Mn)[NLC], bool has_z, const float (&qc)[3][NLC]) {
            if (!(is_main && valid)) return;
            const float *Rz = R + (z % 3) * RING;
            const float *Sz = Ss + ((kbase + z - zc0) & 3) * SSZ + ly * SW + lx;
            const float cx = x < a.nx - 1 ? a.ctau : 0.f, cy = y < a.ny - 1 ? a.ctau : 0.f;
            const float cz = (has_z && a.zg0 + z < a.nzg - 1) ? a.ctau : 0.f;
            const float sb = a.s_ch == 1 ? Sz[0] : 1.f;
            float *qo = Qo + (z & 1) * L::QOSZ + ly * 32 + lx;   // [k][v][row][32]
#pragma unroll
            for (int v = 0; v < NLC; ++v) {
                const float mc = Rz[v * RPS + roff];
                const float gx = Rz[v * RPS + roff + 1] - mc;
                const float gy = Rz[v * RPS + roff + RS] - mc;
                const float gz = Mn[v] - mc;
                float hx = qc[0][v], hy = qc[1][v], hz = qc[2][v];
                const float sv = sb * a.g.s[lb + v];
                if (a.cap == 0) flow_step3<0>(cx, cy, cz, gx, gy, gz, sv, hx, hy, hz);
                else flow_step3<1>(cx, cy, cz, gx, gy, gz, sv, hx, hy, hz);
                qo[v * TY * 32] = hx;
                qo[(NLC + v) * TY * 32] = hy;
                qo[(2 * NLC + v) * TY * 32] = hz;
            }
        };
        auto store_q = [&](int z) {   // thread 0: the three k-blocks of the flow tile of plane z
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const float *blk = Qo + (z & 1) * L::QOSZ + k * NLC * TY * 32;
                tma_store_4d(&a.tm_qo, blk, x0, y0, k * NF + lb, z + 1, pol_out);
                // fused halo exchange (pf_staged.cuh): plane 0 -> below, q^z of the last plane -> above
                if (a.link_below && z == 0) tma_store_4d(&a.tm_qo_nb, blk, x0, y0, k * NF + lb, a.nb_plane, pol_out);
                if (k == 2 && a.link_above && z == a.nzl - 1)
                    tma_store_4d(&a.tm_qz_nb, blk, x0, y0, k * NF + lb, 0, pol_out);
            }
        };

        auto plane_step = [&](const int p, float (&qc)[3][NLC], float (&qn)[3][NLC]) {
            const int k = kbase + (p - zc0);
            const int st = k & 1;
            mbar_wait(&bars[st], (k >> 1) & 1);
            const float *Qb = Qs + st * L::QSZ;
            const float *Ub = Us + st * L::USZ;
            const float *Db = Ds + st * L::USZ;
            float *Rp = R + (p % 3) * RING;
            float dl[NLC], uold[NLC], ut[NLC], rr[NLC];   // uold: log2 state; ut: masses u~
            // this CTA's half of the labels: (m_h, T_h, s_h) and r_L = t_L - T_h, e_L = 2^r_L (label_half)
            float mh = 0.f, th = 0.f, sh = 1.f;
            if (lx >= 0) {
#pragma unroll
                for (int v = 0; v < NLC; ++v) {
                    const float qx = Qb[v * QCS + qoff];
                    const float qxm = Qb[v * QCS + qoff - 1];
                    const float qy = Qb[(NLCP + v) * QCS + qoff];
                    const float qym = Qb[(NLCP + v) * QCS + qoff - QW];
                    const float qz = Qb[(2 * NLCP + v) * QCS + qoff];
                    const float dq = ((qx - qxm) + (qy - qym)) + (qz - qc[2][v]);
                    qn[0][v] = qx; qn[1][v] = qy; qn[2][v] = qz;
                    float Dv;
                    if constexpr (DBF) Dv = bf16_to_f32(reinterpret_cast<const uint16_t *>(Db)[v * (UROWS * 40) +
                                                                                              ly * 40 + (lx < 0 ? 0 : lx)]);
                    else Dv = Db[v * UCS + uoff];
                    dl[v] = Dv + dq;                        // Potts: d_L = D_L + div q_L
                    if constexpr (UH) uold[v] = __half2float(reinterpret_cast<const __half *>(Ub)[v * (UROWS * 40) +
                                                                                                  ly * 40 + (lx < 0 ? 0 : lx)]);
                    else uold[v] = Ub[v * UCS + uoff];
                }
                label_half<NLC>(dl, uold, rr, ut, a.shift, k2, mh, th, sh);
            }
            if (PF_EARLY_ISSUE && warp != 0) named_arrive(kStageBar, 32 * (TY + 2));
            // refill of stage st with step k + 2: this item's plane p + 2, else the next item's first planes
            auto refill = [&]() {
                fence_proxy_async();
                if (p + 2 <= pend) issue(p + 2, k + 2, x0, y0);
                else if (p + 1 - pend < nsteps_next) issue(ng.zc0 + (p + 1 - pend), k + 2, ng.x0, ng.y0);
            };
            auto early_issue = [&]() {
                if (warp == 0) {
                    named_bar(kStageBar, 32 * (TY + 2));
                    if (tid == 0) refill();
                }
            };
            if (PF_EARLY_ISSUE == 1) early_issue();
            // ---- ONE exchange of (m_h, T_h, s_h) with the partner CTA (label_update's split form, pf_math.cuh)
            const int xb = k & 1;   // exchange buffer / mbarrier of this plane; phase = (k >> 1) & 1
            if (tid == 0) mbar_arrive_expect_tx(&bars[2 + xb], kXBytes);   // arm (bytes may already be in)
            if (lx >= 0) {
                st_async_f32x4(x_remote + xb * kXBuf, mh, th, sh, barx_remote + xb * 8u);
            }
            mbar_wait(&bars[2 + xb], (k >> 1) & 1);
            if (PF_EARLY_ISSUE == 2) early_issue();
            float sum = 1.f;
            if (lx >= 0) {
                const float4 xo = reinterpret_cast<const float4 *>(X2)[xb * CL::XPTS + xpt];
                float ch, gh;
                sum = rank == 0 ? label_halves_combine(mh, th, sh, xo.x, xo.y, xo.z, 0, a.shift, k2, ch, gh)
                                : label_halves_combine(xo.x, xo.y, xo.z, mh, th, sh, 1, a.shift, k2, ch, gh);
#pragma unroll
                for (int v = 0; v < NLC; ++v) ut[v] *= gh;
                if (p < zc1 && is_main && valid) {
                    if (rank == 0 && label_sum_bad(sum)) {
                        const unsigned long long vox = ((unsigned long long)(a.zg0 + p) * a.ny + y) * a.nx + x;
                        atomicMin(a.err_voxel, vox);
                    }
                    float *uo = Uo + (p & 1) * L::UOSZ + ly * 32 + lx;
                    __half *uoh = reinterpret_cast<__half *>(Uo + (p & 1) * L::UOSZ) + ly * 32 + lx;
#pragma unroll
                    for (int v = 0; v < NLC; ++v) {
                        float ln = rr[v] + ch;
                        if constexpr (UH) {   // stored as binary16: the residual sees the stored value
                            ln = round_state_half(ln);
                            uoh[v * TY * 32] = __float2half_rn(ln);
                        } else {
                            uo[v * TY * 32] = ln;
                        }
                        if (a.check) resid = fmaxf(resid, fabsf(u_of_log2(ln) - u_of_log2(uold[v])));
                    }
                }
#pragma unroll
                for (int v = 0; v < NLC; ++v) Rp[v * RPS + roff] = ut[v];   // Potts: M_L = u~_L
            }
            fence_proxy_async();
            if (tid == 0) bulk_wait_read_all();
            __syncthreads();   // ring slot p complete; stage st consumed; staged u complete
            if (tid == 0) {
                if (!PF_EARLY_ISSUE) refill();
                if (p < zc1) {
                    tma_store_4d(&a.tm_uo, Uo + (p & 1) * L::UOSZ, x0, y0, lb, p + 1, pol_out);
                    if (a.link_below && p == 0)
                        tma_store_4d(&a.tm_uo_nb, Uo + (p & 1) * L::UOSZ, x0, y0, lb, a.nb_plane, pol_out);
                }
                if (p - 2 >= zc0) store_q(p - 2);
                bulk_commit();
            }
            if (p > zc0) stage_b(p - 1, ut, true, qc);
        };
        int p = zc0;
        for (; p + 1 <= pend; p += 2) {
            plane_step(p, qA, qB);
            plane_step(p + 1, qB, qA);
        }
        const bool last_in_B = p <= pend;
        if (last_in_B) plane_step(p, qA, qB);
        if (!has_above) {
            if (tid == 0) bulk_wait_read_all();
            __syncthreads();
            float Mdummy[NLC];
#pragma unroll
            for (int v = 0; v < NLC; ++v) Mdummy[v] = 0.f;
            if (last_in_B) stage_b(zc1 - 1, Mdummy, false, qB);
            else stage_b(zc1 - 1, Mdummy, false, qA);
        }
        fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
            for (int z = max(zc0, pend - 1); z < zc1; ++z) store_q(z);
            bulk_commit();
            bulk_wait_read_all();
        }
        kbase += cg.steps();
        prev_steps = cg.steps();
    }
    if (lane == 0) bulk_wait_all();
    cluster_sync_all();   // no CTA leaves while its partner may still write into its shared memory
    if (a.check) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) resid = fmaxf(resid, __shfl_xor_sync(0xffffffffu, resid, o));
        if (lane == 0 && resid > 0.f) atomicMax(a.resid_bits, __float_as_uint(resid));
    }
}

bool cluster_kernel_lookup(int NL, int DBF, int UH, StagedKernelInfo *info);

}  // namespace pf
