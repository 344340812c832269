// pf_tb2.cuh -- temporal blocking: TWO iterations of the pseudo-flow while-loop per HBM pass (SURVEY 8(f3),
// pf_config.tblock = 2), for Potts models with few labels (K <= 4) on whole volumes.
//
// Why only there: iteration t + 1 of an output tile needs iteration t's flows on the tile grown by one point and
// its masses on the tile grown by two, so iteration t runs redundantly on a halo ring and its results have to
// stay on chip for three planes.  With K labels the state of one (x, y) point is 4K floats, and on sm_100's
// 227 KB per CTA the two staged input planes, the four rings and the staged outputs fit for K <= 4 (K = 4:
// ~150 KB); for the configs' K = 8 / 9-node graphs the same layout needs ~370 KB.
//
// Geometry (relative to the tile origin x0, y0; output tile W = 28 columns x TY rows, so that the widest region
// is 31 points and one warp covers a row -- lane = x_rel + 1, warp = y_rel + 1):
//   R_A0 = [-1, 30) x [-1, TY+2)  iteration t   stage A (div, excess, label update, masses M^t)
//   R_B0 = [-1, 29) x [-1, TY+1)  iteration t   stage B (q^{t+1}: needs M^t at x, x+e_x, x+e_y)
//   R_A1 = [ 0, 29) x [ 0, TY+1)  iteration t+1 stage A (needs q^{t+1} at x, x-e_x, x-e_y)
//   R_B1 = [ 0, 28) x [ 0, TY)    iteration t+1 stage B -> the tile's output u^{t+2}, q^{t+2}
// Inputs (q^t over [-2, 30) x [-2, TY+2), u^t and D over R_A0, S over R_B0) arrive by TMA boxes that start at
// x0 - 4 (16-byte aligned: x0 is a multiple of 28).  Each CTA marches z; at plane step p it runs
//   A_t(p) | B_t(p-1) | A_{t+1}(p-1) | B_{t+1}(p-2)
// separated by CTA barriers.  q^{t+1} of the thread's own point lives in registers (two planes), its x / y
// components are also published in a one-plane exchange buffer for the +e_x / +e_y neighbours' divergence.
// Every per-point arithmetic step is pf_math.cuh's, in the one-iteration kernels' order, so two iterations
// here are bitwise two launches of pf_iter_staged (tests/test_gpu_tblock.py).  Out-of-volume points of R_B0
// get q^{t+1} = 0 (the TMA zero fill of q^k(-1) = 0 in the one-iteration kernels, reading R4).
#pragma once
#include "pf_staged.cuh"

namespace pf {

template <int K, int TY>
struct TB2Layout {
    static constexpr int W = 28;                      // output columns
    static constexpr int BW = 36;                     // input box width: x in [x0-4, x0+32)
    static constexpr int QR = TY + 4, UR = TY + 3, SR = TY + 2;   // q / u, D / S box rows
    static constexpr int QSZ = round32(3 * K * QR * BW), USZ = round32(K * UR * BW);
    static constexpr int STG = QSZ + 2 * USZ;        // q, u, D of one plane
    static constexpr int SSZ = round32(SR * BW);      // one S ring slot (shared field)
    static constexpr int NS = 8;                      // S ring slots (planes p-2 .. p+2 live)
    static constexpr int MS = 32;                     // ring row stride
    static constexpr int M0 = round32(K * (TY + 3) * MS);   // M^t ring slot over R_A0
    static constexpr int XQ = round32(K * (TY + 2) * MS);   // q^{t+1} x / y exchange over R_B0
    static constexpr int M1 = round32(K * (TY + 1) * MS);   // M^{t+1} ring slot over R_A1
    static constexpr int UO = round32(K * TY * W), QO = round32(3 * K * TY * W);   // output staging
    static constexpr int kThreads = 32 * (TY + 3);
    __host__ __device__ static constexpr int off_S() { return 2 * STG; }
    __host__ __device__ static constexpr int off_M0() { return off_S() + NS * SSZ; }
    __host__ __device__ static constexpr int off_X() { return off_M0() + 3 * M0; }
    __host__ __device__ static constexpr int off_M1() { return off_X() + 2 * XQ; }
    __host__ __device__ static constexpr int off_Uo() { return off_M1() + 3 * M1; }
    __host__ __device__ static constexpr int off_Qo() { return off_Uo() + 2 * UO; }
    __host__ __device__ static constexpr int floats() { return off_Qo() + 2 * QO; }
    __host__ __device__ static constexpr int bytes() { return floats() * 4 + 64; }
};

// Flow step + projection of one point's K flows (Eq. 8; R5, R14) from ring values: mc = M(x), mx = M(x+e_x),
// my = M(x+e_y), mz = M(x+e_z); coefficients already folded with the volume boundaries.
template <int K, int CAP>
__device__ __forceinline__ void tb_flow(float cx, float cy, float cz, const float *R, int off, int kstride, int rowstride,
                                        const float (&mz)[K], const float (&sv)[K], const float (&qin)[3][K],
                                        float (&qout)[3][K]) {
#pragma unroll
    for (int v = 0; v < K; ++v) {
        const float mc = R[v * kstride + off];
        const float gx = R[v * kstride + off + 1] - mc;
        const float gy = R[v * kstride + off + rowstride] - mc;
        const float gz = mz[v] - mc;
        float hx = qin[0][v], hy = qin[1][v], hz = qin[2][v];
        flow_step3<CAP>(cx, cy, cz, gx, gy, gz, sv[v], hx, hy, hz);
        qout[0][v] = hx; qout[1][v] = hy; qout[2][v] = hz;
    }
}

// two CTAs per SM for K = 2 (~80 KB of shared memory, <= 93 registers)
template <int K, int TY, int CAP>
__global__ void __launch_bounds__(32 * (TY + 3), K == 2 ? 2 : 1) pf_iter_tb2(const __grid_constant__ StagedArgs a) {
    using L = TB2Layout<K, TY>;
    constexpr int W = L::W, BW = L::BW, MS = L::MS;
    constexpr int QCS = L::QR * BW, UCS = L::UR * BW;
    extern __shared__ __align__(128) float sm[];
    float *Stg = sm;                       // 2 x (q, u, D)
    float *Ss = sm + L::off_S();
    float *M0 = sm + L::off_M0();
    float *Xq = sm + L::off_X();           // [x / y component][K][TY+2][32]
    float *M1 = sm + L::off_M1();
    float *Uo = sm + L::off_Uo();
    float *Qo = sm + L::off_Qo();
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm + L::floats());

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int xr = lane - 1, yr = warp - 1;                 // point of this thread relative to (x0, y0)
    const bool inA0 = lane < 31;
    const bool inB0 = inA0 && xr < 29 && yr < TY + 1;
    const bool inA1 = xr >= 0 && xr < 29 && yr >= 0 && yr < TY + 1;
    const bool inB1 = xr >= 0 && xr < 28 && yr >= 0 && yr < TY;
    const int qoff = (yr + 2) * BW + xr + 4;                // q stage (rows from y0-2, columns from x0-4)
    const int uoff = (yr + 1) * BW + xr + 4;                // u / D / S stages (rows from y0-1)
    const int m0off = (yr + 1) * MS + (xr + 1);             // M^t ring, exchange buffer (from (-1, -1))
    const int m1off = yr * MS + xr;                         // M^{t+1} ring (from (0, 0))
    const int ooff = yr * W + xr;                           // output staging [c][row][W]
    const int64_t P = (int64_t)a.pitch * a.ny;
    const int64_t qps = (int64_t)3 * K * P;
    const float k2 = kLog2e * a.inv_c;
    const int top = a.nzg - 1;                              // whole volume: local plane = global plane

    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
        prefetch_tmap(&a.tm_q);
        prefetch_tmap(&a.tm_u);
        prefetch_tmap(&a.tm_D);
        if (a.s_ch) prefetch_tmap(&a.tm_S);
        prefetch_tmap(&a.tm_uo);
        prefetch_tmap(&a.tm_qo);
    }
    __syncthreads();
    auto issue = [&](int plane, int stage, int x0, int y0) {
        mbar_arrive_expect_tx(&bars[stage], a.tx_bytes);
        float *S0 = Stg + stage * L::STG;
        tma_load_4d(S0, &a.tm_q, &bars[stage], x0 - 4, y0 - 2, 0, plane + 1);
        tma_load_4d(S0 + L::QSZ, &a.tm_u, &bars[stage], x0 - 4, y0 - 1, 0, plane + 1);
        tma_load_4d(S0 + L::QSZ + L::USZ, &a.tm_D, &bars[stage], x0 - 4, y0 - 1, 0, plane);
        if (a.s_ch) tma_load_4d(Ss + (plane & (L::NS - 1)) * L::SSZ, &a.tm_S, &bars[stage], x0 - 4, y0 - 1, 0, plane);
    };
    const uint64_t pol_out = policy_evict_first();

    float resid = 0.f;
    int kbase = 0;
    if (blockIdx.x == 0 && tid == 0) *a.ticket_next = 0ull;
    __shared__ int s_item;
    auto grab = [&]() -> int {
        const unsigned long long t = atomicAdd(a.ticket, 1ull);
        return t < (unsigned long long)a.items ? (int)t : a.items;
    };
    if (tid == 0) s_item = grab();
    __syncthreads();
    for (int item = s_item; item < a.items; item = s_item) {
        const int chunk = item / a.tiles, tile = item - chunk * a.tiles;
        const int x0 = (tile % a.tiles_x) * W, y0 = (tile / a.tiles_x) * TY;
        const int zc0 = chunk * a.zchunk, zc1 = min(zc0 + a.zchunk, a.nzl);
        const int a0 = zc0 > 0 ? zc0 - 1 : 0;               // iteration t also on the plane below the chunk
        const int aE = min(zc1 + 1, top);                   // ... and on up to two planes above it
        const int bE = min(zc1, top);
        const int pLast = zc1 + 1;                           // last plane step (B_{t+1}(zc1 - 1))
        const int x = x0 + xr, y = y0 + yr;
        const bool inside = inA0 && x >= 0 && x < a.nx && y >= 0 && y < a.ny;
        const int64_t pix = inside ? (int64_t)y * a.pitch + x : 0;
        const float cx = x < a.nx - 1 ? a.ctau : 0.f, cy = y < a.ny - 1 ? a.ctau : 0.f;

        __syncthreads();   // the previous item's readers of the rings / stages (and of s_item) are done
        if (tid == 0) {
            s_item = grab();
            fence_proxy_async();
            issue(a0, kbase & 1, x0, y0);
            if (a0 + 1 <= aE) issue(a0 + 1, (kbase + 1) & 1, x0, y0);
        }
        // register state: q^t, q^{t+1}, lambda^{t+1}, D of the own point, two alternating sets each
        float qtA[3][K], qtB[3][K], q1A[3][K], q1B[3][K], uA[K], uB[K], DA[K], DB[K];
#pragma unroll
        for (int v = 0; v < K; ++v) {
            qtA[0][v] = qtA[1][v] = qtA[2][v] = 0.f;
            q1A[0][v] = q1A[1][v] = q1A[2][v] = 0.f;
            q1B[0][v] = q1B[1][v] = q1B[2][v] = 0.f;
        }
        if (inside && a0 > 0) {   // q^t_z of the plane below the first computed plane (0 below the volume)
            const float *qb = a.q_in + (int64_t)(a0 - 1) * qps + 2 * K * P + pix;
#pragma unroll
            for (int v = 0; v < K; ++v) qtA[2][v] = __ldg(qb + v * P);
        }
        auto sval = [&](int plane, float (&sv)[K]) {   // capacities of the own point at `plane`
            const float sb = a.s_ch ? Ss[(plane & (L::NS - 1)) * L::SSZ + uoff] : 1.f;
#pragma unroll
            for (int v = 0; v < K; ++v) sv[v] = sb * a.g.s[v];
        };
        // thread 0, at the first barrier of step p: the TMA stores of the outputs staged in step p - 1
        auto store_outputs = [&](int pu, int pq) {
            if (pu >= zc0 && pu < zc1) tma_store_4d(&a.tm_uo, Uo + (pu & 1) * L::UO, x0, y0, 0, pu + 1, pol_out);
            if (pq >= zc0 && pq < zc1) tma_store_4d(&a.tm_qo, Qo + (pq & 1) * L::QO, x0, y0, 0, pq + 1, pol_out);
            bulk_commit();
        };

        auto step = [&](const int p, float (&qtP)[3][K], float (&qtN)[3][K], float (&q1P)[3][K], float (&q1N)[3][K],
                        float (&uP)[K], float (&uN)[K], float (&DP)[K], float (&DN)[K]) {
            const bool doAt = p <= aE;
            const bool doBt = p - 1 >= a0 && p - 1 <= bE;
            const bool doA1 = p - 1 >= zc0 && p - 1 <= bE;
            const bool doB1 = p - 2 >= zc0 && p - 2 < zc1;
            float Mt[K], M1v[K];
            // ---------------- A_t(p) on R_A0
            if (doAt) {
                const int k = kbase + (p - a0);
                const int st = k & 1;
                mbar_wait(&bars[st], (k >> 1) & 1);
                const float *Qb = Stg + st * L::STG, *Ub = Qb + L::QSZ, *Db = Ub + L::USZ;
                if (inA0) {
                    float dq[K], Dv[K], lam[K], ut[K], ln[K], d[K];
#pragma unroll
                    for (int v = 0; v < K; ++v) {
                        const float qx = Qb[v * QCS + qoff], qxm = Qb[v * QCS + qoff - 1];
                        const float qy = Qb[(K + v) * QCS + qoff], qym = Qb[(K + v) * QCS + qoff - BW];
                        const float qz = Qb[(2 * K + v) * QCS + qoff];
                        dq[v] = ((qx - qxm) + (qy - qym)) + (qz - qtP[2][v]);
                        qtN[0][v] = qx; qtN[1][v] = qy; qtN[2][v] = qz;
                        Dv[v] = Db[v * UCS + uoff];
                        lam[v] = Ub[v * UCS + uoff];
                    }
                    label_excess<0, 0, K>(dq, Dv, d, a.g.w);
                    const float sum = label_update<0, K>(d, lam, ut, ln, a.shift, k2);
#pragma unroll
                    for (int v = 0; v < K; ++v) {
                        uN[v] = ln[v];
                        DN[v] = Dv[v];
                        Mt[v] = ut[v];
                        M0[(p % 3) * L::M0 + v * (TY + 3) * MS + m0off] = ut[v];
                    }
                    if (inB1 && inside && p >= zc0 && p < zc1) {
                        if (label_sum_bad(sum)) atomicMin(a.err_voxel, ((unsigned long long)p * a.ny + y) * a.nx + x);
                        if (a.check == 1) resid = resid_log2<K>(ln, lam, resid);
                    }
                }
            }
            if (tid == 0) bulk_wait_read_all();   // the staging buffers this step rewrites have been read
            __syncthreads();                      // M^t(p) complete; the stage of plane p consumed
            if (tid == 0) {
                if (doAt && p + 2 <= aE) {
                    fence_proxy_async();
                    issue(p + 2, (kbase + (p - a0)) & 1, x0, y0);
                }
                store_outputs(p - 2, p - 3);   // staged in step p - 1
            }
            // ---------------- B_t(p-1) on R_B0: q^{t+1}(p-1)
            if (doBt && inB0) {
                if (inside) {
                    const float cz = p - 1 < top ? a.ctau : 0.f;
                    float mz[K], sv[K];
#pragma unroll
                    for (int v = 0; v < K; ++v) mz[v] = p - 1 < top ? Mt[v] : 0.f;
                    sval(p - 1, sv);
                    tb_flow<K, CAP>(cx, cy, cz, M0 + ((p - 1) % 3) * L::M0, m0off, (TY + 3) * MS, MS, mz, sv, qtP, q1N);
                } else {
#pragma unroll
                    for (int v = 0; v < K; ++v) q1N[0][v] = q1N[1][v] = q1N[2][v] = 0.f;
                }
#pragma unroll
                for (int v = 0; v < K; ++v) {
                    Xq[v * (TY + 2) * MS + m0off] = q1N[0][v];
                    Xq[L::XQ + v * (TY + 2) * MS + m0off] = q1N[1][v];
                }
            }
            __syncthreads();   // exchange complete
            // ---------------- A_{t+1}(p-1) on R_A1
            if (doA1 && inA1) {
                float dq[K], ut[K], ln[K], d[K];
#pragma unroll
                for (int v = 0; v < K; ++v)
                    dq[v] = ((q1N[0][v] - Xq[v * (TY + 2) * MS + m0off - 1]) +
                             (q1N[1][v] - Xq[L::XQ + v * (TY + 2) * MS + m0off - MS])) + (q1N[2][v] - q1P[2][v]);
                label_excess<0, 0, K>(dq, DP, d, a.g.w);
                const float sum = label_update<0, K>(d, uP, ut, ln, a.shift, k2);
#pragma unroll
                for (int v = 0; v < K; ++v) {
                    M1v[v] = ut[v];
                    M1[((p - 1) % 3) * L::M1 + v * (TY + 1) * MS + m1off] = ut[v];
                }
                if (inB1 && p - 1 < zc1) {
                    float *uo = Uo + ((p - 1) & 1) * L::UO + ooff;
#pragma unroll
                    for (int v = 0; v < K; ++v) uo[v * TY * W] = ln[v];
                    if (inside) {
                        if (label_sum_bad(sum)) atomicMin(a.err_voxel, ((unsigned long long)(p - 1) * a.ny + y) * a.nx + x);
                        if (a.check == 2) resid = resid_log2<K>(ln, uP, resid);
                    }
                }
            }
            // (no barrier: B_{t+1}(p-2) reads the M^{t+1} ring slot of plane p-2, complete since the previous step,
            // and the point's own M^{t+1}(p-1); the exchange buffer is rewritten only after the next step's first
            // barrier)
            // ---------------- B_{t+1}(p-2) on R_B1: q^{t+2}(p-2)
            if (doB1 && inB1) {
                float qo3[3][K];
                if (inside) {
                    const float cz = p - 2 < top ? a.ctau : 0.f;
                    float mz[K], sv[K];
#pragma unroll
                    for (int v = 0; v < K; ++v) mz[v] = p - 2 < top ? M1v[v] : 0.f;
                    sval(p - 2, sv);
                    tb_flow<K, CAP>(cx, cy, cz, M1 + ((p - 2) % 3) * L::M1, m1off, (TY + 1) * MS, MS, mz, sv, q1P, qo3);
                } else {
#pragma unroll
                    for (int v = 0; v < K; ++v) qo3[0][v] = qo3[1][v] = qo3[2][v] = 0.f;
                }
                float *qo = Qo + ((p - 2) & 1) * L::QO + ooff;
#pragma unroll
                for (int v = 0; v < K; ++v) {
                    qo[v * TY * W] = qo3[0][v];
                    qo[(K + v) * TY * W] = qo3[1][v];
                    qo[(2 * K + v) * TY * W] = qo3[2][v];
                }
            }
            fence_proxy_async();   // staged outputs -> visible to the async proxy before next step's stores
        };
        int p = a0;
        for (; p + 1 <= pLast; p += 2) {
            step(p, qtA, qtB, q1A, q1B, uA, uB, DA, DB);
            step(p + 1, qtB, qtA, q1B, q1A, uB, uA, DB, DA);
        }
        if (p <= pLast) step(p, qtA, qtB, q1A, q1B, uA, uB, DA, DB);
        __syncthreads();
        if (tid == 0) {
            bulk_wait_read_all();
            store_outputs(pLast - 1, pLast - 2);   // staged in the last step
            bulk_wait_read_all();
        }
        kbase += aE - a0 + 1;
    }
    if (tid == 0) bulk_wait_all();
    if (a.check) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) resid = fmaxf(resid, __shfl_xor_sync(0xffffffffu, resid, o));
        if (lane == 0 && resid > 0.f) atomicMax(a.resid_bits, __float_as_uint(resid));
    }
}

bool tb2_kernel_lookup(int K, int CAP, StagedKernelInfo *info);

}  // namespace pf
