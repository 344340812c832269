// pf_staged.cuh -- TMA-staged, persistent version of the fused pseudo-flow iteration (sm_100a).
//
// Same arithmetic and same per-voxel order as pf_iter_kernel (see pf_kernels.cuh for the
// step-by-step mapping to Alg. 1 / Alg. 2 / Alg. 3; the shared math is in pf_math.cuh), different
// data movement:
//   * persistent CTAs (one per SM) take work items = (32 x TY tile, z-chunk) from a device-side
//     ticket queue, so the tiles in flight at any time are a window of consecutive (neighbouring)
//     tiles and their shared halo lines are served from L2;
//   * every z-plane of the tile is fetched by ONE thread as 3-4 TMA box loads
//     (cp.async.bulk.tensor.4d) into a 2-deep shared-memory ring guarded by mbarriers: q over
//     x in [x0-4, x0+36) x y in [y0-1, y0+TY] (the -x/-y neighbours for div and the +1 halo
//     points), u and D over [x0, x0+36) x [y0, y0+TY], S over the tile.  Out-of-range box
//     elements are zero-filled by the TMA unit, which is exactly q^k(-1) = 0 (reading R4);
//   * plane p+2 is in flight while plane p is computed; q(p) of the own voxel is kept in registers
//     (two alternating sets) until the flow step of plane p runs one plane later; S(p) stays in a
//     4-slot shared ring (slot p mod 4) until then;
//   * OSTAGE: the new u and q are staged in shared memory and written by TMA bulk-tensor stores with an
//     evict-first L2 policy (no per-thread 64-bit address arithmetic, no L2 pollution).  u always as
//     one double-buffered tile per plane, issued by thread 0 at the plane barrier.  q: OSTAGE 1
//     double-buffers the flow tile the same way; OSTAGE 2 (many nodes, tight shared memory) has ONE
//     flow row per main warp, which the warp hands to the TMA unit itself at the end of its flow step.
//     Bulk-store groups are per thread, so lane 0 only waits for its own previous row store -- issued a
//     whole stage-A phase earlier -- and no CTA-wide barrier or single-thread drain sits on the
//     critical path (a single CTA-wide flow tile stalled every plane on the store's shared-memory read).
//     OSTAGE 0 stores straight from registers;
//   * G = 2 (Potts with many labels): the labels of a row of 32 voxels are split over a warp pair, which
//     doubles the warps per SM at the same shared-memory footprint and halves the registers per thread;
//     the only per-voxel couplings of the label update -- m = min_L d_L and a = sum_L u~_L -- are
//     combined from per-half (shift, sum) pairs exchanged once through shared memory under a 64-thread named
//     barrier -- label_update's split form (pf_math.cuh), so G does not change a bit.
//   * u is stored as lambda = log2 u (pf_math.cuh label_update; reading R18): the u stages, the staged u tile
//     and the output hold log2 values.
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
    CUtensorMap tm_uo;  // output u, store box (32, TY, NL)                                   [OSTAGE]
    CUtensorMap tm_qo;  // output q, store box (32, TY, 3*NF) [OSTAGE 1] or (32, 1, NF/G)   [OSTAGE 2]
    // fused halo exchange (pf_link_slabs): the boundary planes of the new state are also TMA-stored into
    // the neighbouring slabs' halo planes (peer memory); tile stores only (OSTAGE 1 / cluster kernel)
    CUtensorMap tm_uo_nb;   // below neighbour's new u     (box as tm_uo), halo plane coordinate nb_plane
    CUtensorMap tm_qo_nb;   // below neighbour's new q     (box as tm_qo)
    CUtensorMap tm_qz_nb;   // above neighbour's new q     (box: the z-component block), coordinate 0
    int link_below, link_above, nb_plane;
    const float *q_in;  // plane 0 of input q (chunk-start q^z(zc0-1) read)
    float *u_out;
    float *q_out;
    int nx, ny, pitch, nzl, zg0, nzg;
    int zchunk, tiles_x, tiles;
    int strip;          // tile order inside a z-chunk: column strips of `strip` tiles, row-major inside a strip
    int item_begin, items;  // this launch runs items [item_begin, items)
    // z-chunks: item / tiles < nb: boundary chunk = the single plane bplane[item / tiles] (planes next to
    // a neighbouring slab, computed first so their halo exchange overlaps the rest); otherwise interior
    // chunk c = item / tiles - nb: planes [zlo + c*zchunk, min(zlo + (c+1)*zchunk, zhi))
    int nb, bplane0, bplane1, zlo, zhi;
    int s_ch;     // 0: scalar capacities, 1: shared field (x g.s[f]), NF: field per flow node
    int cap, shift, check;
    int fastproj;       // 1: flow_step3's plain projection is exact for this launch (see pf_math.cuh)
    unsigned int tx_bytes;
    float inv_c, ctau;
    unsigned int *resid_bits;
    unsigned long long *err_voxel;
    unsigned long long *ticket;        // this launch's work-item ticket counter (0 at launch start)
    unsigned long long *ticket_next;   // the other counter: zeroed here for the next launch (launches alternate)
    GraphConst g;
};

__host__ __device__ constexpr int round32(int n) { return (n + 31) / 32 * 32; }

// Tile origin of the t-th tile of a z-chunk.  Tiles are taken in column strips of `strip` tiles (the last
// strip may be narrower), row-major inside a strip; strip < 0: row groups of -strip tile rows, column-major inside
// a group.  The default is one strip of full rows (narrower strips and row groups, which bring a tile's
// y-neighbour closer in the ticket order, measured slower: pf_api.cu choose_chunking).
__device__ __forceinline__ void tile_origin(const StagedArgs &a, int t, int ty_rows, int &x0, int &y0) {
    const int tiles_y = a.tiles / a.tiles_x;
    if (a.strip < 0) {   // row groups of h tile rows, column-major inside a group: a tile's y-neighbour inside the
        const int h = -a.strip;                     // group is the next ticket, its x-neighbour h tickets away
        const int gblk = h * a.tiles_x, gidx = t / gblk;
        const int hh = min(h, tiles_y - gidx * h);
        const int r = t - gidx * gblk, cx = r / hh;
        x0 = cx * 32;
        y0 = (gidx * h + (r - cx * hh)) * ty_rows;
        return;
    }
    const int sblk = a.strip * tiles_y;           // tiles per full strip
    const int sidx = t / sblk;
    const int w = min(a.strip, a.tiles_x - sidx * a.strip);
    const int r = t - sidx * sblk;
    const int ty = r / w;
    x0 = (sidx * a.strip + (r - ty * w)) * 32;
    y0 = ty * ty_rows;
}

// Geometry of one work item: tile origin, the chunk's planes [zc0, zc1) and the last plane step pend (zc1 when a
// plane above exists: its stage A gives the masses M(zc1) the flow step of plane zc1 - 1 needs).
struct ItemGeom {
    int x0, y0, zc0, zc1, pend;
    bool has_above;
    __device__ __forceinline__ int steps() const { return pend - zc0 + 1; }
};

__device__ __forceinline__ ItemGeom item_geom(const StagedArgs &a, int item, int ty_rows) {
    ItemGeom g;
    const int chunk = item / a.tiles, tile = item - chunk * a.tiles;
    tile_origin(a, tile, ty_rows, g.x0, g.y0);
    g.zc0 = chunk < a.nb ? (chunk == 0 ? a.bplane0 : a.bplane1) : a.zlo + (chunk - a.nb) * a.zchunk;
    g.zc1 = chunk < a.nb ? g.zc0 + 1 : min(g.zc0 + a.zchunk, a.zhi);
    g.has_above = (a.zg0 + g.zc1) < a.nzg;
    g.pend = g.has_above ? g.zc1 : g.zc1 - 1;
    return g;
}

// NSTG: input stages in flight (2: one plane of look-ahead; 3: two, where shared memory allows -- short tiles).
// SR: S ring slots covering the planes p - 1 .. p + NSTG.
template <int NI, int NL, int TY, int OSTAGE, int MODEL, int G, int NSTG_ = 2>
struct StagedLayout {
    static_assert(OSTAGE >= 0 && OSTAGE <= 2, "OSTAGE: 0 direct, 1 tile stores, 2 tile u + per-warp q rows");
    static constexpr int NSTG = NSTG_, SR = NSTG_ == 2 ? 4 : 8;
    static constexpr int NV = NI + NL;
    static constexpr int NF = Model<MODEL, NI, NL>::NF;   // flow-carrying nodes
    static constexpr int QW = 40, UW = 36, SW = 32;
    static constexpr int QROWS = TY + 2, UROWS = TY + 1;
    static constexpr int QSZ = round32(3 * NF * QROWS * QW);  // floats per stage
    static constexpr int USZ = round32(NL * UROWS * UW);
    static constexpr int RS = 33, RPS = (TY + 1) * RS, RING = NF * RPS;
    static constexpr int UOSZ = OSTAGE ? round32(NL * TY * 32) : 0;       // u staging [l][row][32], x2
    static constexpr int QOSZ = OSTAGE ? round32(3 * NF * TY * 32) : 0;   // q staging: OSTAGE 1 [ch][row][32] x2,
    static constexpr int QOB = OSTAGE == 1 ? 2 : 1;                         //   OSTAGE 2 [row][grp][k][f][32] x1
    static constexpr int XSZ = G > 1 ? round32(3 * (TY + 2) * G * 32) : 0;  // (m_h, T_h, s_h) exchange (G = 2)
    static constexpr int kThreads = 32 * G * (TY + 2);
    // runtime part: the S staging ring holds s_ch channels (0, 1 or NF)
    __host__ __device__ static constexpr int ssz(int s_ch) { return round32(s_ch * TY * SW); }
    __host__ __device__ static constexpr int off_U() { return NSTG * QSZ; }
    __host__ __device__ static constexpr int off_D() { return NSTG * (QSZ + USZ); }
    __host__ __device__ static constexpr int off_S() { return NSTG * (QSZ + 2 * USZ); }
    __host__ __device__ static constexpr int off_R(int s_ch) { return off_S() + SR * ssz(s_ch); }
    __host__ __device__ static constexpr int off_Uo(int s_ch) { return off_R(s_ch) + round32(3 * RING); }
    __host__ __device__ static constexpr int off_Qo(int s_ch) { return off_Uo(s_ch) + 2 * UOSZ; }
    __host__ __device__ static constexpr int off_X(int s_ch) { return off_Qo(s_ch) + QOB * QOSZ; }
    __host__ __device__ static constexpr int floats(int s_ch) { return off_X(s_ch) + XSZ; }
    __host__ __device__ static constexpr int bytes(int s_ch) { return floats(s_ch) * 4 + 32; }
};

__device__ __forceinline__ void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Flow step + projection of the thread's NFG flow nodes (channels f0 .. f0+NFG-1) at one voxel (P:148,
// P:298).  qo: the thread's slot for channel (k = 0, node f0) in the staging buffer or in global memory;
// Pf / Pk: the stride between consecutive nodes / between the k-components there.
// Sz: the voxel's S slot of plane z (shared field, or node 0 of per-node fields; stride TY*32 per node).
// Boundaries (nabla_k M = 0 at the last index) are folded into per-axis step coefficients computed once
// per voxel; M is finite at every point the kernel computes (also outside the volume, from the TMA zero
// fill), so q - 0 * g == q there.  Capacity: S_f = sb * g.s[f] with sb = 1 (scalars), the shared field
// (g.s = 1 for a plain shared field, the node factors for a scaled one), or the node's own field.
template <int NFG, int CAP, int OSTAGE, int TY>
__device__ __forceinline__ void flow_out_staged(const StagedArgs &a, const float *Rz, int f0, int roff, int rps,
                                                int rs, const float (&Mn)[NFG], bool has_z, int x, int y, int zg,
                                                const float (&qc)[3][NFG], const float *Sz, float *qo,
                                                int Pf, int Pk) {
    const float cx = x < a.nx - 1 ? a.ctau : 0.f, cy = y < a.ny - 1 ? a.ctau : 0.f;
    const float cz = (has_z && zg < a.nzg - 1) ? a.ctau : 0.f;
    auto one = [&](int v, float sv) {
        const int f = f0 + v;
        const float mc = Rz[f * rps + roff];
        const float gx = Rz[f * rps + roff + 1] - mc;
        const float gy = Rz[f * rps + roff + rs] - mc;
        const float gz = Mn[v] - mc;
        float hx = qc[0][v], hy = qc[1][v], hz = qc[2][v];
        if (a.fastproj) flow_step3<CAP, false>(cx, cy, cz, gx, gy, gz, sv, hx, hy, hz);
        else flow_step3<CAP, true>(cx, cy, cz, gx, gy, gz, sv, hx, hy, hz);
        if (OSTAGE) {
            qo[v * Pf] = hx;
            qo[v * Pf + Pk] = hy;
            qo[v * Pf + 2 * Pk] = hz;
        } else {
            st_stream(qo + v * Pf, hx);
            st_stream(qo + v * Pf + Pk, hy);
            st_stream(qo + v * Pf + 2 * Pk, hz);
        }
    };
    if (a.s_ch <= 1) {
        const float sb = a.s_ch == 1 ? Sz[0] : 1.f;
#pragma unroll
        for (int v = 0; v < NFG; ++v) one(v, sb * a.g.s[f0 + v]);
    } else {
#pragma unroll
        for (int v = 0; v < NFG; ++v) one(v, Sz[(f0 + v) * TY * 32]);
    }
}

// Per-warp staged output row (OSTAGE 2): lane 0 waits until this warp's previous bulk store from the
// row has read it.  `since` = bulk groups lane 0 committed after that store (thread 0 also commits the
// CTA's u tiles); waiting for all but the newest group is enough when since >= 1 and never waits for
// a just-issued u store.
__device__ __forceinline__ void stage_row_acquire(int lane, int since) {
    if (lane == 0) {
        if (since >= 1) bulk_wait_read_but1();
        else bulk_wait_read_all();
    }
    __syncwarp();
}

// DBF: D stored as bf16 (pf_config.d_bf16; the D stage then holds rows of 40 bf16).
// UH: lambda = log2 u stored as binary16 (pf_config.u_half; the u stage then holds rows of 40 halves, the u
// staging tile halves [l][row][32]).
template <int NI, int NL, int TY, int OSTAGE, int MODEL, int G, int DBF, int UH, uint64_t MASK, int NSTG_ = 2>
__global__ void __launch_bounds__(32 * G *(TY + 2), 1) pf_iter_staged(const __grid_constant__ StagedArgs a) {
    using L = StagedLayout<NI, NL, TY, OSTAGE, MODEL, G, NSTG_>;
    constexpr int NSTG = L::NSTG, SR = L::SR;
    constexpr int NF = L::NF;
    static_assert(G == 1 || (G == 2 && MODEL == 0 && NI == 0 && NL % 2 == 0), "label split: Potts, two halves");
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
    // OSTAGE 2: this warp's flow staging row, [k][v][32] for its NFG nodes
    float *qo_row = Qo + (ly * G + grp) * 3 * NFG * 32;

    if (tid == 0) {
        for (int i = 0; i < NSTG; ++i) mbar_init(&bars[i], 1);
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
        if (a.s_ch) tma_load_4d(Ss + (plane & (SR - 1)) * SSZ, &a.tm_S, &bars[stage], x0, y0, 0, plane);
    };
    const uint64_t pol_out = OSTAGE ? policy_evict_first() : 0;

    float resid = 0.f;
    int since_q = 1 << 20;  // bulk groups this thread committed after its last q row store (OSTAGE 2)
    int kbase = 0;          // planes consumed so far by this CTA (ring position / mbarrier parity)
    // Dynamic work queue: a CTA takes the next ticket when it starts an item, so the items in flight are
    // always a window of ~gridDim consecutive tiles and the halo lines one tile loads from HBM are still in
    // L2 when its neighbours read them (a static round-robin lets CTAs drift apart by whole items on
    // many-item volumes, which sent ~40 % extra halo traffic to HBM on 768^2 planes).  Two counters
    // alternate between launches; each launch zeroes the one the next launch uses, so a launch's
    // parameters do not depend on history and a sequence of launches can be replayed as a CUDA graph.
    if (blockIdx.x == 0 && tid == 0) *a.ticket_next = 0ull;
    __shared__ int s_item;
    auto grab = [&]() -> int {
        const unsigned long long t = atomicAdd(a.ticket, 1ull);
        return t < (unsigned long long)(a.items - a.item_begin) ? a.item_begin + (int)t : a.items;
    };
    if (tid == 0) s_item = grab();
    __syncthreads();
    for (int item = s_item; item < a.items; item = s_item) {
        const int chunk = item / a.tiles, tile = item - chunk * a.tiles;
        int x0, y0;
        tile_origin(a, tile, TY, x0, y0);
        const int zc0 = chunk < a.nb ? (chunk == 0 ? a.bplane0 : a.bplane1) : a.zlo + (chunk - a.nb) * a.zchunk;
        const int zc1 = chunk < a.nb ? zc0 + 1 : min(zc0 + a.zchunk, a.zhi);
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
            for (int i = 0; i < NSTG && zc0 + i <= pend; ++i) issue(zc0 + i, (kbase + i) % NSTG, x0, y0);
        }
        // q of the plane below the chunk (its z-component enters div of the first plane).  Two register
        // sets alternate between "current plane" and "plane awaiting its flow step" (no copies).
        float qA[3][NFG], qB[3][NFG];
#pragma unroll
        for (int v = 0; v < NFG; ++v) { qA[0][v] = 0.f; qA[1][v] = 0.f; qA[2][v] = 0.f; }
        if (valid && (a.zg0 + zc0) > 0) {
            const float *qb = a.q_in + (int64_t)(zc0 - 1) * qps + (2 * NF + f0) * P + pix;
#pragma unroll
            for (int v = 0; v < NFG; ++v) qA[2][v] = __ldg(qb + v * P);
        }

        // flow step + projection of plane z (stage B); Mn = M(z+1) at the voxel (unused when !has_z)
        auto stage_b = [&](const int z, const float (&Mn)[NFG], bool has_z, const float (&qc)[3][NFG]) {
            const float *Rz = R + (z % 3) * RING;
            const float *Sz = Ss + (z & (SR - 1)) * SSZ + ly * SW + lx;
            if (OSTAGE == 2) {
                if (row_out) {
                    stage_row_acquire(lane, since_q);
                    if (valid) {
                        if (a.cap == 0)
                            flow_out_staged<NFG, 0, 1, TY>(a, Rz, f0, roff, RPS, RS, Mn, has_z, x, y, a.zg0 + z, qc,
                                                           Sz, qo_row + lx, 32, NFG * 32);
                        else
                            flow_out_staged<NFG, 1, 1, TY>(a, Rz, f0, roff, RPS, RS, Mn, has_z, x, y, a.zg0 + z, qc,
                                                           Sz, qo_row + lx, 32, NFG * 32);
                    }
                    fence_proxy_async();  // this thread's staged flows -> visible to the async proxy
                    __syncwarp();
                    if (lane == 0) {
#pragma unroll
                        for (int kk = 0; kk < 3; ++kk)
                            tma_store_4d(&a.tm_qo, qo_row + kk * NFG * 32, x0, y, kk * NF + f0, z + 1, pol_out);
                        bulk_commit();
                    }
                    since_q = 0;
                }
            } else if (is_main && valid) {
                float *qo = OSTAGE ? Qo + (z & 1) * L::QOSZ + f0 * TY * 32 + ly * 32 + lx
                                   : a.q_out + (int64_t)z * qps + f0 * P + pix;
                const int Pf = OSTAGE ? TY * 32 : (int)P;
                if (a.cap == 0)
                    flow_out_staged<NFG, 0, OSTAGE, TY>(a, Rz, f0, roff, RPS, RS, Mn, has_z, x, y, a.zg0 + z, qc, Sz,
                                                        qo, Pf, NF * Pf);
                else
                    flow_out_staged<NFG, 1, OSTAGE, TY>(a, Rz, f0, roff, RPS, RS, Mn, has_z, x, y, a.zg0 + z, qc, Sz,
                                                        qo, Pf, NF * Pf);
            }
        };

        // thread 0, OSTAGE 1: the flow tile of plane z to this slab's new state, and with linked slabs
        // plane 0 to the below neighbour's upper halo plane, q^z of the last plane to the above
        // neighbour's lower halo plane (the fused halo exchange)
        auto store_q = [&](int z) {
            tma_store_4d(&a.tm_qo, Qo + (z & 1) * L::QOSZ, x0, y0, 0, z + 1, pol_out);
            if (a.link_below && z == 0) tma_store_4d(&a.tm_qo_nb, Qo + (z & 1) * L::QOSZ, x0, y0, 0, a.nb_plane, pol_out);
            if (a.link_above && z == a.nzl - 1)
                tma_store_4d(&a.tm_qz_nb, Qo + (z & 1) * L::QOSZ + 2 * NF * TY * 32, x0, y0, 2 * NF, 0, pol_out);
        };

        auto plane_step = [&](const int p, float (&qc)[3][NFG], float (&qn)[3][NFG]) {
            const int k = kbase + (p - zc0);
            const int st = k % NSTG;
            mbar_wait(&bars[st], (k / NSTG) & 1);
            const float *Qb = Qs + st * L::QSZ;
            const float *Ub = Us + st * L::USZ;
            const float *Db = Ds + st * L::USZ;
            float *Rp = R + (p % 3) * RING;
            float Mv[NFG];
            // ---------------- stage A(p): div, excess, label update, masses (tile + halo)
            float dq[NFG];
            float Dv[NLG], uold[NLG], ut[NLG], un[NLG];   // uold / un: log2 states; ut: masses u~
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
                if constexpr (DBF) {
                    const uint16_t *Dh = reinterpret_cast<const uint16_t *>(Db);
                    const int doff = ly * 40 + (lx < 0 ? 0 : lx);
#pragma unroll
                    for (int l = 0; l < NLG; ++l) Dv[l] = bf16_to_f32(Dh[(l0 + l) * (UROWS * 40) + doff]);
                } else {
#pragma unroll
                    for (int l = 0; l < NLG; ++l) Dv[l] = Db[(l0 + l) * UCS + uoff];
                }
                if constexpr (UH) {
                    const __half *Uh = reinterpret_cast<const __half *>(Ub);
                    const int hoff = ly * 40 + (lx < 0 ? 0 : lx);
#pragma unroll
                    for (int l = 0; l < NLG; ++l) uold[l] = __half2float(Uh[(l0 + l) * (UROWS * 40) + hoff]);
                } else {
#pragma unroll
                    for (int l = 0; l < NLG; ++l) uold[l] = Ub[(l0 + l) * UCS + uoff];
                }
            }
            float sum = 1.f;
            if constexpr (G == 1) {
                if (lx >= 0) {
                    label_excess<MODEL, NI, NL, MASK>(dq, Dv, dlab, a.g.w);
                    sum = label_update<NI, NL>(dlab, uold, ut, un, a.shift, k2);
                }
            } else {
                // Potts, labels l0 .. l0+NLG-1 = half `grp` of the labels (NL >= kHalfSplitNL): the half's
                // (m_h, T_h, s_h), ONE exchange of the three with the partner warp, then label_update's split
                // combine (pf_math.cuh)
                static_assert(G == 2 && NL >= kHalfSplitNL, "label split = label_update's two halves");
                float *xm = X + (xr * G) * 32 + lane;
                float *xt = X + ((TY + 2) * G + xr * G) * 32 + lane;
                float *xs = X + (2 * (TY + 2) * G + xr * G) * 32 + lane;
                float mh = 0.f, th = 0.f, sh = 1.f;
                float rr[NLG];
                if (lx >= 0) {
#pragma unroll
                    for (int l = 0; l < NLG; ++l) dlab[l] = Dv[l] + dq[l];
                    label_half<NLG>(dlab, uold, rr, ut, a.shift, k2, mh, th, sh);
                }
                xm[grp * 32] = mh;
                xt[grp * 32] = th;
                xs[grp * 32] = sh;
                named_bar(1 + xr, 32 * G);
                float ch, gh;
                sum = label_halves_combine(xm[0], xt[0], xs[0], xm[32], xt[32], xs[32], grp, a.shift, k2, ch, gh);
#pragma unroll
                for (int l = 0; l < NLG; ++l) {
                    un[l] = rr[l] + ch;
                    ut[l] *= gh;
                }
            }
            if constexpr (UH) {   // the stored (binary16) state is what the next iteration reads: round once here
#pragma unroll
                for (int l = 0; l < NLG; ++l) un[l] = round_state_half(un[l]);
            }
            if (lx >= 0) {
                if (p < zc1 && is_main && valid) {
                    if (grp == 0 && label_sum_bad(sum)) {
                        const unsigned long long vox = ((unsigned long long)(a.zg0 + p) * a.ny + y) * a.nx + x;
                        atomicMin(a.err_voxel, vox);
                    }
                    if (OSTAGE) {
                        if constexpr (UH) {
                            __half *uo = reinterpret_cast<__half *>(Uo + (p & 1) * L::UOSZ) + l0 * TY * 32 + ly * 32 + lx;
#pragma unroll
                            for (int l = 0; l < NLG; ++l) uo[l * TY * 32] = __float2half_rn(un[l]);
                        } else {
                            float *uo = Uo + (p & 1) * L::UOSZ + l0 * TY * 32 + ly * 32 + lx;
#pragma unroll
                            for (int l = 0; l < NLG; ++l) uo[l * TY * 32] = un[l];
                        }
                    } else if constexpr (UH) {
                        __half *uo = reinterpret_cast<__half *>(a.u_out) + (int64_t)p * ups + l0 * P + pix;
#pragma unroll
                        for (int l = 0; l < NLG; ++l) st_stream_h(uo + l * (int)P, __float2half_rn(un[l]));
                    } else {
                        float *uo = a.u_out + (int64_t)p * ups + l0 * P + pix;
#pragma unroll
                        for (int l = 0; l < NLG; ++l) st_stream(uo + l * (int)P, un[l]);
                    }
                    if (a.check) resid = resid_log2<NLG>(un, uold, resid);
                }
                if constexpr (G == 1) {
                    node_masses<MODEL, NI, NL, MASK>(ut, Mv, a.g.w);
                } else {
#pragma unroll
                    for (int l = 0; l < NLG; ++l) Mv[l] = ut[l];
                }
#pragma unroll
                for (int v = 0; v < NFG; ++v) Rp[(f0 + v) * RPS + roff] = Mv[v];
            }
            if (OSTAGE) {
                fence_proxy_async();                // staged u -> visible to the TMA (async proxy)
                if (tid == 0) bulk_wait_read_all(); // stores of the buffers about to be rewritten have read them
            }
            __syncthreads();  // ring slot p complete; stage st fully consumed; staged u complete
            if (tid == 0) {
                if (p + NSTG <= pend) {   // the slot plane p released: NSTG - 1 planes of look-ahead
                    fence_proxy_async();
                    issue(p + NSTG, st, x0, y0);
                }
                if (OSTAGE) {
                    if (p < zc1) {
                        tma_store_4d(&a.tm_uo, Uo + (p & 1) * L::UOSZ, x0, y0, 0, p + 1, pol_out);
                        if (OSTAGE == 1 && a.link_below && p == 0)   // fused halo exchange: plane 0 -> below
                            tma_store_4d(&a.tm_uo_nb, Uo + (p & 1) * L::UOSZ, x0, y0, 0, a.nb_plane, pol_out);
                    }
                    if (OSTAGE == 1 && p - 2 >= zc0) store_q(p - 2);
                    bulk_commit();
                    ++since_q;
                }
            }
            // ---------------- stage B(p-1): flow step + projection of plane p-1
            if (p > zc0) stage_b(p - 1, Mv, true, qc);
        };
        int p = zc0;
        for (; p + 1 <= pend; p += 2) {
            plane_step(p, qA, qB);
            plane_step(p + 1, qB, qA);
        }
        const bool last_in_B = p <= pend;
        if (last_in_B) plane_step(p, qA, qB);
        // last plane of the volume: no plane above, nabla_z = 0
        if (!has_above) {
            if (OSTAGE == 1) {  // the store issued at the last plane step may still be reading the tail's buffer
                if (tid == 0) bulk_wait_read_all();
                __syncthreads();
            }
            float Mdummy[NFG];
#pragma unroll
            for (int v = 0; v < NFG; ++v) Mdummy[v] = 0.f;
            if (last_in_B) stage_b(zc1 - 1, Mdummy, false, qB);
            else stage_b(zc1 - 1, Mdummy, false, qA);
        }
        if (OSTAGE == 1) {  // flush the item's last staged flow planes
            fence_proxy_async();
            __syncthreads();
            if (tid == 0) {
                for (int z = max(zc0, pend - 1); z < zc1; ++z) store_q(z);
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
    int smem_bytes;  // with s_ch = 0; add 4 * round32(s_ch * tile_y * 32) floats for an S field
    int tile_y;
    int ostage;      // 1: outputs staged in smem and written by TMA stores
    int groups;      // label groups per row (G)
    int s_slots;     // S ring slots (StagedLayout::SR)
};

// mask: the graph's edge mask (edge_on); a kernel specialised for exactly that mask is preferred, else dense rows
bool staged_kernel_lookup(int NI, int NL, int MODEL, int DBF, int UH, uint64_t mask, StagedKernelInfo *info);

}  // namespace pf
