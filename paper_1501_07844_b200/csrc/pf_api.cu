// pf_api.cu -- the C-ABI of include/pf.h: graph compilation (row a10), device state
// and layouts, the per-iteration launch loop (rows a0-a8), labeling (a9), halo
// regions for z-slab decomposition (row e).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <cuda.h>

#include "pf.h"
#include "pf_alm.cuh"
#include "pf_aux.cuh"
#include "pf_kernels.cuh"
#include "pf_staged.cuh"
#include "pf_cluster.cuh"

using namespace pf;

namespace {

thread_local std::string g_last_error;

pf_status fail(pf_status st, const char *fmt, ...) {
    char buf[2048];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return st;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

bool is_device_ptr(const void *p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// --------------------------------------------------------------------------
// Label-graph compilation (reading R9)
// --------------------------------------------------------------------------
struct Compiled {
    int num_nodes = 0, NI = 0, NL = 0, NV = 0;
    bool chain = false;  // Ishikawa chain shape (see pf.h); model 1 also needs zero end-label capacities
    int model = 0;       // 0: Alg. 1/2, 1: Alg. 3 (Ishikawa chain)
    int NF = 0;          // flow-carrying nodes (positions 0..NF-1)
    std::vector<int> pos_of_node;  // node id -> position, S -> -1
    std::vector<int> node_of_pos;
    GraphConst g;
    std::vector<std::vector<float>> W;  // W[pos][leaf slot] path weights
    std::vector<float> w_src;           // weight of the edge S -> position (0: none)
};

pf_status compile_graph(const pf_graph *gr, Compiled *out) {
    if (!gr || gr->num_nodes < 3 || gr->num_edges < 2 || !gr->parent || !gr->child || !gr->weight)
        return fail(PF_ERR_GRAPH, "graph: need >= 3 nodes (S + 2 end labels), >= 2 edges and non-NULL arrays");
    const int n = gr->num_nodes, ne = gr->num_edges;
    std::string errs;
    auto add = [&](const std::string &s) { errs += (errs.empty() ? "" : "; ") + s; };
    std::vector<std::vector<std::pair<int, float>>> kids(n), pars(n);
    bool idx_ok = true;
    for (int e = 0; e < ne; ++e) {
        const int p = gr->parent[e], c = gr->child[e];
        const float w = gr->weight[e];
        if (p < 0 || p >= n || c < 0 || c >= n) {
            add("edge " + std::to_string(e) + " has a node id out of range");
            idx_ok = false;
            continue;
        }
        if (!(w > 0.f) || !std::isfinite(w)) add("edge " + std::to_string(e) + " weight must be > 0");
        if (p == c) add("self-loop at node " + std::to_string(p));
        kids[p].push_back({c, w});
        pars[c].push_back({p, w});
    }
    if (!idx_ok) return fail(PF_ERR_GRAPH, "graph: %s", errs.c_str());
    if (!pars[0].empty()) add("source S (node 0) has parents");
    // Kahn with lowest-id tie-break
    std::vector<int> indeg(n, 0), order;
    for (int v = 0; v < n; ++v) indeg[v] = (int)pars[v].size();
    std::vector<bool> placed(n, false);
    for (int k = 0; k < n; ++k) {
        int pick = -1;
        for (int v = 0; v < n; ++v)
            if (!placed[v] && indeg[v] == 0) { pick = v; break; }
        if (pick < 0) break;
        placed[pick] = true;
        order.push_back(pick);
        for (auto &c : kids[pick]) indeg[c.first]--;
    }
    if ((int)order.size() != n) add("graph has a cycle");
    // reachability from S
    std::vector<bool> reach(n, false);
    std::vector<int> stack{0};
    reach[0] = true;
    while (!stack.empty()) {
        int v = stack.back();
        stack.pop_back();
        for (auto &c : kids[v])
            if (!reach[c.first]) { reach[c.first] = true; stack.push_back(c.first); }
    }
    for (int v = 1; v < n; ++v)
        if (!reach[v]) add("node " + std::to_string(v) + " unreachable from S");
    std::vector<int> leaves, internals;
    for (int v = 1; v < n; ++v) (kids[v].empty() ? leaves : internals).push_back(v);
    if (leaves.size() < 2) add("fewer than 2 end labels");
    if (!errs.empty()) return fail(PF_ERR_GRAPH, "graph: %s", errs.c_str());
    // W_(v, B) by memoised recursion in reverse topological order
    const int NL = (int)leaves.size();
    std::vector<std::vector<double>> Wd(n, std::vector<double>(NL, 0.0));
    for (int k = n - 1; k >= 0; --k) {
        const int v = order[k];
        if (kids[v].empty() && v != 0) {
            Wd[v][std::find(leaves.begin(), leaves.end(), v) - leaves.begin()] = 1.0;
        } else {
            for (auto &c : kids[v])
                for (int l = 0; l < NL; ++l) Wd[v][l] += (double)c.second * Wd[c.first][l];
        }
    }
    for (int l = 0; l < NL; ++l)
        if (std::fabs(Wd[0][l] - 1.0) > 1e-6)
            add("W_(S," + std::to_string(leaves[l]) + ") = " + std::to_string(Wd[0][l]) +
                " != 1 (sum of end labels must equal u_S = 1, reading R9)");
    if (!errs.empty()) return fail(PF_ERR_GRAPH, "graph: %s", errs.c_str());
    const int NI = (int)internals.size();
    // Ishikawa chain: internals in topological order N_1..N_N, S -> {N_1, L_0}, N_i -> {N_{i+1}, L_i},
    // N_N -> L_N, all weights 1, end labels in increasing id order L_0..L_N
    bool chain = NL == NI + 1 && NI >= 1 && kids[0].size() == 2;
    std::vector<int> lev;
    for (int k = 0; k < n && chain; ++k)
        if (order[k] != 0 && !kids[order[k]].empty()) lev.push_back(order[k]);
    auto has_edge = [&](int p, int c) {
        for (auto &e : kids[p])
            if (e.first == c && e.second == 1.f) return true;
        return false;
    };
    if (chain) {
        chain = (int)lev.size() == NI && has_edge(0, lev[0]) && has_edge(0, leaves[0]);
        for (int i = 0; i < NI && chain; ++i) {
            const bool last = i == NI - 1;
            chain = kids[lev[i]].size() == (last ? 1u : 2u) && has_edge(lev[i], leaves[i + 1]) &&
                    (last || has_edge(lev[i], lev[i + 1]));
        }
    }
    if (!chain && (NI > kMaxInternal || NI + NL > kMaxNodes))
        return fail(PF_ERR_UNSUPPORTED, "graph: %d internal + %d end nodes exceeds the compiled kernel set "
                                        "(<= %d internal, <= %d non-source nodes)", NI, NL, kMaxInternal, kMaxNodes);
    if (chain && NL > kMaxNodes)
        return fail(PF_ERR_UNSUPPORTED, "graph: Ishikawa chain with %d labels exceeds %d", NL, kMaxNodes);
    out->chain = chain;
    out->num_nodes = n;
    out->NI = NI;
    out->NL = NL;
    out->NV = NI + NL;
    out->pos_of_node.assign(n, -1);
    out->node_of_pos.clear();
    for (int k = 0; k < n; ++k) {  // internal nodes in topological order
        const int v = order[k];
        if (v != 0 && !kids[v].empty()) {
            out->pos_of_node[v] = (int)out->node_of_pos.size();
            out->node_of_pos.push_back(v);
        }
    }
    for (int v : leaves) {  // end labels in node-id order
        out->pos_of_node[v] = (int)out->node_of_pos.size();
        out->node_of_pos.push_back(v);
    }
    memset(&out->g, 0, sizeof(out->g));
    for (int v = 1; v < n && NI <= kMaxInternal; ++v) {  // dense weights (unused by the chain kernels)
        if (kids[v].empty()) continue;
        const int i = out->pos_of_node[v];
        for (auto &c : kids[v]) out->g.w[i][out->pos_of_node[c.first]] += c.second;
    }
    out->w_src.assign(out->NV, 0.f);
    for (auto &c : kids[0]) out->w_src[out->pos_of_node[c.first]] += c.second;
    out->W.assign(out->NV, std::vector<float>(NL, 0.f));  // W_(v, B), for reports
    for (int p = 0; p < out->NV; ++p)
        for (int l = 0; l < NL; ++l) out->W[p][l] = (float)Wd[out->node_of_pos[p]][l];
    return PF_OK;
}

}  // namespace

struct pf_solver {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    bool poisoned = false;
    int ndim = 3;
    int64_t nx = 0, ny = 0, nz = 0;
    int64_t z0 = 0, z1 = 0, nzl = 0;
    int64_t P = 0;       // channel-plane stride = pitch * ny
    int64_t pitch = 0;   // row pitch (elements), multiple of 4 for TMA
    Compiled gc;
    pf_config cfg{};
    int s_kind = 0;
    // allocations (base pointers) and plane-0 pointers
    float *u_alloc[2] = {nullptr, nullptr}, *q_alloc[2] = {nullptr, nullptr};
    float *D_alloc = nullptr, *S_alloc = nullptr;   // D_alloc: fp32 D (nullptr when D is stored as bf16)
    uint16_t *D16 = nullptr;                          // bf16 D (cfg.d_bf16), same [z][l][y][pitch] layout
    bool alm = false;                                 // PF_METHOD_EXPLICIT_ALM (pf_alm.cu)
    float *p_alloc = nullptr, *pS_alloc = nullptr;    // ALM sink flows [z][l][y][pitch], source flow [z][y][pitch]
    float *uint_alloc = nullptr;                      // ALM on a DAG: u of the internal nodes [z][NI][y][pitch]
    const void *Dptr() const { return D16 ? (const void *)D16 : (const void *)D_alloc; }
    float *u[2] = {nullptr, nullptr}, *q[2] = {nullptr, nullptr};
    int cur = 0;
    int64_t iters = 0;
    unsigned int *d_resid = nullptr;
    unsigned long long *d_err = nullptr;   // [0] error voxel, [1], [2] work-item ticket counters
    int launch_parity = 0;                 // which ticket counter the next staged launch uses
    // fused halo exchange (pf_link_slabs): neighbours and tensor maps of their state buffers
    pf_solver *nb_below = nullptr, *nb_above = nullptr;   // in-process links (pf_link_slabs)
    bool link_below = false, link_above = false;           // in-process or IPC links
    int nb_plane = 0;                                      // below neighbour's upper halo plane coordinate
    CUtensorMap tm_uo_nb[2], tm_qo_nb[2], tm_qz_nb[2];
    // cross-process links (pf_ipc_*): state from cudaMalloc (IPC-exportable), an interprocess event
    // recorded after every iteration, the neighbours' opened buffers and events
    bool ipc = false;
    cudaEvent_t ipc_ev = nullptr;
    std::vector<void *> ipc_opened;
    cudaEvent_t nb_ev[2] = {nullptr, nullptr};
    // CUDA graph of `graph_iters` whole iterations (pf_iterate), replayed when the state matches the
    // capture: same ping-pong buffer, same counter parity, check iterations at the same positions
    cudaGraphExec_t graph = nullptr;
    int graph_iters = 0, graph_cur = 0, graph_parity = 0;
    bool graph_failed = false;
    unsigned int *d_flag = nullptr;
    double *d_energy = nullptr;  // partials + result
    IterKernelInfo kinfo{};
    int zchunk = 0;
    dim3 grid;
    int ctas_per_sm = 0;
    int regs = 0;
    int64_t device_bytes = 0;
    bool last_resid_valid = false;
    int64_t launches = 0;
    // TMA-staged persistent kernel (default) -- see pf_staged.cuh
    bool staged = false;
    bool cluster = false;   // staged work split over a 2-CTA cluster (pf_cluster.cuh; Potts, many labels)
    StagedKernelInfo sinfo{};
    CUtensorMap tm_q[2], tm_u[2], tm_D, tm_S, tm_qo[2], tm_uo[2];
    int staged_smem = 0;
    int s_ch = 0;
    int tiles_x = 0, tiles = 0, items = 0, sgrid = 0;
    // boundary / interior split of the z-chunks (slabs with neighbours; pf_iterate_phase)
    int nb = 0, bplane[2] = {0, 0}, zlo = 0, zhi = 0, items_b = 0;
    int phase_pending = 0;  // 1 after pf_iterate_phase(0) until its phase 1
    unsigned int tx_bytes = 0;
};

namespace {

pf_status cuda_fail(pf_solver *s, cudaError_t e, const char *what) {
    if (s) s->poisoned = true;
    cudaGetLastError();  // clear the (non-sticky) last-error state so it does not leak into other solvers
    return fail(PF_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define CK(expr, what)                                     \
    do {                                                   \
        cudaError_t e__ = (expr);                          \
        if (e__ != cudaSuccess) return cuda_fail(s, e__, what); \
    } while (0)

int64_t ups(const pf_solver *s) { return (int64_t)s->gc.NL * s->P; }
// q always carries 3 components internally (q^z == 0 for 2-D volumes), so the kernels need no ndim branch
int64_t qps(const pf_solver *s) { return (int64_t)3 * s->gc.NF * s->P; }

// Device memory comes from the device's stream-ordered pool, which keeps up to kPoolKeep bytes of freed
// memory for reuse: a solver created right after another one was destroyed (the end-to-end
// create / iterate / get_labeling / destroy cycle) does not pay cudaMalloc / cudaFree again.
constexpr uint64_t kPoolKeep = 64ull << 30;

void pool_setup(int dev) {
    static bool done[64] = {false};
    if (dev < 0 || dev >= 64 || done[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = kPoolKeep;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
    done[dev] = true;
}

void free_all(pf_solver *s) {
    if (s->graph) {
        cudaGraphExecDestroy(s->graph);
        s->graph = nullptr;
    }
    for (void *p : s->ipc_opened) cudaIpcCloseMemHandle(p);
    s->ipc_opened.clear();
    for (int i = 0; i < 2; ++i)
        if (s->nb_ev[i]) { cudaEventDestroy(s->nb_ev[i]); s->nb_ev[i] = nullptr; }
    if (s->ipc_ev) { cudaEventDestroy(s->ipc_ev); s->ipc_ev = nullptr; }
    if (s->ipc) {   // cudaMalloc'd state (exportable); synchronise before the synchronous frees
        cudaStreamSynchronize(s->stream);
        for (int i = 0; i < 2; ++i) {
            if (s->u_alloc[i]) cudaFree(s->u_alloc[i]);
            if (s->q_alloc[i]) cudaFree(s->q_alloc[i]);
            s->u_alloc[i] = s->q_alloc[i] = nullptr;
        }
    }
    void *ptrs[] = {s->u_alloc[0], s->u_alloc[1], s->q_alloc[0], s->q_alloc[1], s->D_alloc, s->S_alloc, s->D16,
                    s->p_alloc, s->pS_alloc, s->uint_alloc,
                    s->d_resid, s->d_err, s->d_flag, s->d_energy};
    for (void *p : ptrs)
        if (p) cudaFreeAsync(p, s->stream);
    cudaGetLastError();
    for (int i = 0; i < 2; ++i) s->u_alloc[i] = s->q_alloc[i] = nullptr;
    s->D_alloc = s->S_alloc = nullptr;
    s->D16 = nullptr;
    s->p_alloc = s->pS_alloc = s->uint_alloc = nullptr;
    s->d_resid = nullptr;
    s->d_err = nullptr;
    s->d_flag = nullptr;
    s->d_energy = nullptr;
}

// ipc: a plain cudaMalloc allocation (pool allocations cannot be exported with cudaIpcGetMemHandle);
// free_all releases those with cudaFree (s->ipc)
pf_status alloc(pf_solver *s, void **p, size_t bytes, const char *what, bool ipc = false) {
    cudaError_t e = ipc ? cudaMalloc(p, bytes) : cudaMallocAsync(p, bytes, s->stream);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(PF_ERR_OOM, "cudaMallocAsync(%zu bytes) for %s failed: %s", bytes, what, cudaGetErrorString(e));
    }
    s->device_bytes += (int64_t)bytes;
    return PF_OK;
}

AlmArgs alm_args(pf_solver *s, int check) {
    AlmArgs a;
    memset(&a, 0, sizeof(a));
    a.q_in = s->q[s->cur];
    a.q_out = s->q[1 - s->cur];
    a.u = s->u[0];
    a.p = s->p_alloc;
    a.pS = s->pS_alloc;
    a.D = s->Dptr();
    a.d_bf16 = s->D16 ? 1 : 0;
    a.S = s->S_alloc;
    a.s_per_node = s->s_kind == PF_S_FIELD_PER_NODE ? 1 : 0;
    a.cap = s->cfg.cap;
    a.check = check;
    a.nx = (int)s->nx;
    a.ny = (int)s->ny;
    a.nz = (int)s->nzl;
    a.pitch = (int)s->pitch;
    a.NL = s->gc.NL;
    a.zchunk = 32;
    a.zchunk2 = s->gc.NI > 0 ? 2 : 8;   // pass-2 chunk: parallelism vs the chunk-start q^z re-read
    a.c = s->cfg.c;
    a.inv_c = 1.0f / s->cfg.c;
    a.tau = s->cfg.tau;
    for (int l = 0; l < s->gc.NV && l < 16; ++l) a.s[l] = s->gc.g.s[l];
    a.resid_bits = s->d_resid;
    if (s->gc.NI > 0) {   // DAG / HMF (Eq. 11)
        a.dag = 1;
        a.NI = s->gc.NI;
        a.NV = s->gc.NV;
        a.u_int = s->uint_alloc;
        const Compiled &g = s->gc;
        for (int j = 0; j < g.NV; ++j) a.W[0][j] = g.w_src[j];
        for (int i = 0; i < g.NI; ++i)
            for (int j = 0; j < g.NV; ++j) a.W[1 + i][j] = g.g.w[i][j];
    }
    return a;
}


pf_status init_state(pf_solver *s) {
    const int64_t nu = (s->nzl + 2) * ups(s), nq = (s->nzl + 2) * qps(s);
    if (s->alm) {  // u = 1/K, q = 0, p_S = min_L D_L, p_L = p_S
        CK(launch_fill(s->u_alloc[0], nu, 1.0f / (float)s->gc.NL, s->stream), "init u");
        for (int i = 0; i < 2; ++i) CK(cudaMemsetAsync(s->q_alloc[i], 0, nq * sizeof(float), s->stream), "init q");
        CK(launch_alm_init(alm_args(s, 0), s->stream), "ALM init");
        s->launches += 2;
        CK(cudaMemsetAsync(s->d_err, 0xff, sizeof(unsigned long long), s->stream), "init err");
        s->cur = 0;
        s->iters = 0;
        return PF_OK;
    }
    for (int i = 0; i < 2; ++i) {
        CK(launch_fill(s->u_alloc[i], nu, 1.0f / (float)s->gc.NL, s->stream), "init u");
        s->launches++;
        CK(cudaMemsetAsync(s->q_alloc[i], 0, nq * sizeof(float), s->stream), "init q");
    }
    CK(cudaMemsetAsync(s->d_err, 0xff, sizeof(unsigned long long), s->stream), "init err");
    s->cur = 0;
    s->iters = 0;
    return PF_OK;
}

// z-chunk length minimising (work items per CTA slot, rounded up) x (planes per item incl. the
// look-ahead plane); `slots` = CTAs resident at once (persistent grid) or SMs (one-shot grid).
int best_chunks(int64_t tiles, int nzl, int64_t slots) {
    int best_n = 1;
    double best_cost = 1e300;
    const int max_n = std::max(1, nzl / 4);
    for (int n = 1; n <= max_n; ++n) {
        const int ch = (nzl + n - 1) / n;
        const int nn = (nzl + ch - 1) / ch;
        const double cost = std::ceil((double)(tiles * nn) / slots) * (ch + 1);
        if (cost < best_cost - 1e-9) { best_cost = cost; best_n = nn; }
    }
    return best_n;
}

void choose_chunking(pf_solver *s) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->device);
    const int nzl = (int)s->nzl;
    const int ty = s->staged ? s->sinfo.tile_y : s->kinfo.tile_y;
    const int gx = (int)((s->nx + kTX - 1) / kTX), gy = (int)((s->ny + ty - 1) / ty);
    const int64_t tiles = (int64_t)gx * gy;
    if (s->staged) {
        const int occ = std::max(1, s->ctas_per_sm);
        const int64_t slots = (int64_t)sms * occ;
        // planes next to a neighbouring slab form their own one-plane chunks, computed first
        s->nb = 0;
        const bool below = s->z0 > 0, above = s->z1 < s->nz;
        if (below) s->bplane[s->nb++] = 0;
        if (above && !(below && nzl == 1)) s->bplane[s->nb++] = nzl - 1;
        s->zlo = below ? 1 : 0;
        s->zhi = std::max(s->zlo, (above ? nzl - 1 : nzl));
        const int nzi = s->zhi - s->zlo;
        const int64_t wslots = s->cluster ? slots / 2 : slots;   // concurrent work items
        int n = nzi > 0 ? best_chunks(tiles, nzi, wslots) : 0;
        // cluster kernel: chunks of <= 32 planes.  Its 74 work slots put a tile's y-neighbour (tiles_x
        // tickets later) about tiles_x / 74 chunk-lengths behind; with 48-plane chunks on 768^2 planes that
        // is ~15 planes, past the ~10 planes of traffic L2 holds, and the y-halo rows came from HBM
        // (ncu: 1.31x algorithmic bytes over 20 back-to-back iterations vs 1.08x with 24-plane chunks;
        // sustained: 32 planes is the fastest, tools/ab.py)
        if (s->cluster && nzi > 32) n = std::max(n, (nzi + 31) / 32);
        if (const char *zc = getenv("PF_ZCHUNK")) {   // experiments (tools/): force the z-chunk length
            const int want = atoi(zc);
            if (want > 0 && nzi > 0) n = (nzi + want - 1) / want;
        }
        s->zchunk = nzi > 0 ? (nzi + n - 1) / n : 1;
        const int nch = nzi > 0 ? (nzi + s->zchunk - 1) / s->zchunk : 0;
        s->tiles_x = gx;
        s->tiles = (int)tiles;
        s->items_b = (int)(tiles * s->nb);
        s->items = (int)(tiles * (s->nb + nch));
        s->sgrid = (int)std::min<int64_t>(slots, (int64_t)s->items * (s->cluster ? 2 : 1));
        s->grid = dim3(s->sgrid, 1, 1);
    } else {
        const int n = best_chunks(tiles, nzl, sms);
        s->zchunk = (nzl + n - 1) / n;
        s->grid = dim3(gx, gy, (nzl + s->zchunk - 1) / s->zchunk);
    }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
    }
    return fn;
}

// 4-D fp32 tensor map over an internal array [plane][channel][y][pitch] (x fastest); elements with
// x >= nx, y outside [0, ny) or plane outside [0, nplanes) read as 0 (TMA out-of-bounds fill).
bool encode4d(CUtensorMap *m, const void *base, int64_t nx, int64_t ny, int64_t pitch, int64_t nch, int64_t nplanes,
              int bx, int by, int bc, bool bf16 = false) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    const int64_t es_b = bf16 ? 2 : 4;
    cuuint64_t dims[4] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nch, (cuuint64_t)nplanes};
    cuuint64_t strides[3] = {(cuuint64_t)(pitch * es_b), (cuuint64_t)(pitch * ny * es_b),
                             (cuuint64_t)(pitch * ny * nch * es_b)};
    cuuint32_t box[4] = {(cuuint32_t)bx, (cuuint32_t)by, (cuuint32_t)bc, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return fn(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void *)base, dims,
              strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

pf_status check_usable(const pf_solver *s) {
    if (!s) return fail(PF_ERR_INVALID, "NULL solver");
    if (s->poisoned) return fail(PF_ERR_STATE, "solver poisoned by an earlier error");
    return PF_OK;
}

pf_status check_numeric(pf_solver *s) {
    unsigned long long v = ~0ull;
    CK(cudaMemcpyAsync(&v, s->d_err, sizeof(v), cudaMemcpyDeviceToHost, s->stream), "read error word");
    CK(cudaStreamSynchronize(s->stream), "sync");
    if (v != ~0ull) {
        s->poisoned = true;
        const unsigned long long nx = (unsigned long long)s->nx, ny = (unsigned long long)s->ny;
        return fail(PF_ERR_NUMERIC, "numerical collapse: a(x) <= 0 or not finite at voxel (x=%llu, y=%llu, z=%llu)",
                    v % nx, (v / nx) % ny, v / (nx * ny));
    }
    return PF_OK;
}

// Copy `nz` planes of one dense volume [z][y][x] (x fastest) into channel `c` of an internal array
// [plane][channel][y][pitch] with `nch` channels (to_internal), or back out of it.
cudaError_t copy_volume(bool to_internal, float *internal_c, int64_t nch, float *dense, int64_t nx, int64_t ny,
                        int64_t pitch, int64_t nz, cudaStream_t st) {
    if (nz <= 0) return cudaSuccess;
    if (pitch == nx) {  // unpadded rows: one contiguous x-y plane per (z, channel) -> large 2-D copy
        const size_t plane = (size_t)(nx * ny) * 4;
        if (to_internal)
            return cudaMemcpy2DAsync(internal_c, plane * nch, dense, plane, plane, (size_t)nz, cudaMemcpyDefault, st);
        return cudaMemcpy2DAsync(dense, plane, internal_c, plane * nch, plane, (size_t)nz, cudaMemcpyDefault, st);
    }
    cudaMemcpy3DParms p;
    memset(&p, 0, sizeof(p));
    cudaPitchedPtr ip = make_cudaPitchedPtr(internal_c, (size_t)pitch * 4, (size_t)nx, (size_t)(ny * nch));
    cudaPitchedPtr dp = make_cudaPitchedPtr(dense, (size_t)nx * 4, (size_t)nx, (size_t)ny);
    p.srcPtr = to_internal ? dp : ip;
    p.dstPtr = to_internal ? ip : dp;
    p.extent = make_cudaExtent((size_t)nx * 4, (size_t)ny, (size_t)nz);
    p.kind = cudaMemcpyDefault;
    return cudaMemcpy3DAsync(&p, st);
}

}  // namespace

extern "C" {

const char *pf_last_error(void) { return g_last_error.c_str(); }

const char *pf_version(void) { return "pf 0.1 (sm_100a)"; }

pf_status pf_create(const pf_dims *dims, const pf_graph *graph, const float *const *D, const pf_smoothness *S,
                    const pf_config *cfg, const pf_slab *slab, pf_solver **out) {
    if (!out) return fail(PF_ERR_INVALID, "out is NULL");
    *out = nullptr;
    if (!dims || !graph || !D || !S || !cfg) return fail(PF_ERR_INVALID, "NULL argument");
    if ((dims->ndim != 2 && dims->ndim != 3) || dims->nx < 1 || dims->ny < 1 || dims->nz < 1 ||
        (dims->ndim == 2 && dims->nz != 1))
        return fail(PF_ERR_INVALID, "dims: ndim must be 2 or 3, extents >= 1, nz == 1 for ndim == 2");
    if (((dims->nx + 3) / 4 * 4) * dims->ny * 3 * kMaxNodes >= (int64_t)1 << 31)
        return fail(PF_ERR_INVALID, "dims: an x-y plane must have < 2^31 / 48 voxels (32-bit channel offsets)");
    if (!(cfg->c > 0.f) || !(cfg->tau > 0.f) || !std::isfinite(cfg->c) || !std::isfinite(cfg->tau))
        return fail(PF_ERR_INVALID, "config: c and tau must be finite and > 0");
    if ((cfg->cap != PF_CAP_L2 && cfg->cap != PF_CAP_LINF) || (cfg->shift != PF_SHIFT_MIN && cfg->shift != PF_SHIFT_NONE) ||
        cfg->check_every < 0)
        return fail(PF_ERR_INVALID, "config: bad cap / shift / check_every");
    int64_t z0 = 0, z1 = dims->nz;
    if (slab) {
        z0 = slab->z_begin;
        z1 = slab->z_end;
        if (z0 < 0 || z1 > dims->nz || z1 <= z0) return fail(PF_ERR_INVALID, "slab: need 0 <= z_begin < z_end <= nz");
    }
    Compiled gc;
    pf_status st = compile_graph(graph, &gc);
    if (st != PF_OK) return st;
    if (S->kind != PF_S_SCALAR_PER_NODE && S->kind != PF_S_SHARED_FIELD && S->kind != PF_S_FIELD_PER_NODE &&
        S->kind != PF_S_SCALED_FIELD)
        return fail(PF_ERR_INVALID, "smoothness: bad kind");
    if (S->kind == PF_S_SCALED_FIELD && (!S->scalars || !S->fields))
        return fail(PF_ERR_INVALID, "smoothness: scaled field needs scalars and fields[0]");
    if (S->kind == PF_S_SCALAR_PER_NODE || S->kind == PF_S_SCALED_FIELD) {
        if (!S->scalars) return fail(PF_ERR_INVALID, "smoothness: scalars is NULL");
        for (int v = 1; v < gc.num_nodes; ++v)
            if (!(S->scalars[v] >= 0.f) || !std::isfinite(S->scalars[v]))
                return fail(PF_ERR_INVALID, "smoothness: S_%d = %g must be finite and >= 0", v, (double)S->scalars[v]);
    } else if (!S->fields) {
        return fail(PF_ERR_INVALID, "smoothness: fields is NULL");
    }
    for (int l = 0; l < gc.NL; ++l)
        if (!D[l]) return fail(PF_ERR_INVALID, "D[%d] is NULL", l);
    // Ishikawa model (Alg. 3): chain shape and identically-zero end-label capacities
    if (gc.chain) {
        bool zero = S->kind == PF_S_SCALAR_PER_NODE || S->kind == PF_S_SCALED_FIELD;
        for (int l = 0; l < gc.NL && zero; ++l) zero = S->scalars[gc.node_of_pos[gc.NI + l]] == 0.f;
        gc.model = zero ? 1 : 0;
    }
    if (gc.model == 0 && (gc.NI > kMaxInternal || gc.NV > kMaxNodes))
        return fail(PF_ERR_UNSUPPORTED, "graph: %d internal + %d end nodes exceeds the compiled kernel set "
                                        "(<= %d internal, <= %d non-source nodes)", gc.NI, gc.NL, kMaxInternal,
                    kMaxNodes);
    gc.NF = gc.model == 1 ? gc.NI : gc.NV;
    if (cfg->method != PF_METHOD_PSEUDO_FLOW && cfg->method != PF_METHOD_EXPLICIT_ALM)
        return fail(PF_ERR_INVALID, "config: bad method");
    const bool alm = cfg->method == PF_METHOD_EXPLICIT_ALM;
    if (alm && (gc.model != 0 || gc.NV > 16 || slab || S->kind == PF_S_SCALED_FIELD))
        return fail(PF_ERR_UNSUPPORTED, "explicit-flow ALM: Potts / HMF / DAG graphs (<= 16 non-source nodes), whole "
                                        "volumes, scalar, shared or per-node capacities only");

    if (cfg->ipc && alm) return fail(PF_ERR_UNSUPPORTED, "config: ipc is for the pseudo-flow kernels");
    pf_solver *s = new pf_solver();
    s->alm = alm;
    s->ipc = cfg->ipc != 0;
    cudaGetDevice(&s->device);
    s->ndim = dims->ndim;
    s->nx = dims->nx;
    s->ny = dims->ny;
    s->nz = dims->nz;
    s->z0 = z0;
    s->z1 = z1;
    s->nzl = z1 - z0;
    // row pitch: 16-byte TMA strides for fp32 (multiple of 4) and, with bf16 D, for bf16 rows (of 8)
    s->pitch = cfg->d_bf16 ? (dims->nx + 7) / 8 * 8 : (dims->nx + 3) / 4 * 4;
    s->P = s->pitch * dims->ny;
    s->gc = gc;
    s->cfg = *cfg;
    s->s_kind = S->kind;
    if (!iter_kernel_lookup(gc.NI, gc.NL, gc.model, &s->kinfo)) {
        delete s;
        return fail(PF_ERR_UNSUPPORTED, "no compiled kernel for %d internal / %d end nodes", gc.NI, gc.NL);
    }
    {
        const char *env = getenv("PF_ITER_KERNEL");
        const bool want_global = env && strcmp(env, "global") == 0;
        s->staged = !alm && !want_global && staged_kernel_lookup(gc.NI, gc.NL, gc.model, cfg->d_bf16 ? 1 : 0, &s->sinfo) && encode_fn() != nullptr;
        // Potts with many labels: the 2-CTA cluster split (scalar / shared capacities; PF_CLUSTER=0 disables)
        const char *cenv = getenv("PF_CLUSTER");
        if (s->staged && gc.model == 0 && gc.NI == 0 && S->kind != PF_S_FIELD_PER_NODE &&
            !(cenv && strcmp(cenv, "0") == 0)) {
            StagedKernelInfo ci{};
            if (cluster_kernel_lookup(gc.NL, cfg->d_bf16 ? 1 : 0, &ci)) {
                s->sinfo = ci;
                s->cluster = true;
            }
        }
        if (s->staged) {
            const int s_ch = (S->kind == PF_S_SHARED_FIELD || S->kind == PF_S_SCALED_FIELD)
                                 ? 1 : (S->kind == PF_S_FIELD_PER_NODE ? gc.NF : 0);
            s->staged_smem = s->sinfo.smem_bytes + 16 * ((s_ch * s->sinfo.tile_y * 32 + 31) / 32 * 32);  // 4 S slots
            int maxsm = 0;
            cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, s->device);
            cudaFuncAttributes fa{};
            cudaFuncGetAttributes(&fa, s->sinfo.func);  // static shared words (work-queue slot) count too
            if (s->staged_smem + (int)fa.sharedSizeBytes > maxsm) s->staged = false;  // e.g. per-node S fields
        }
    }
    cudaError_t e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete s;
        return fail(PF_ERR_CUDA, "cudaStreamCreate: %s", cudaGetErrorString(e));
    }
    s->own_stream = true;
    pool_setup(s->device);
    const int NL = gc.NL, NF = gc.NF;
    const int64_t P = s->P, nzl = s->nzl;
    auto bail = [&](pf_status st2) {
        std::string msg = g_last_error;
        free_all(s);
        cudaStreamSynchronize(s->stream);
        if (s->own_stream) cudaStreamDestroy(s->stream);
        delete s;
        g_last_error = msg;
        return st2;
    };
    // state: planes -1 .. nzl (halo below / above); the ALM updates u in place (one buffer) and stores p, p_S
    for (int i = 0; i < 2; ++i) {
        if (alm && i == 1) {
            s->u_alloc[1] = nullptr;
        } else if ((st = alloc(s, (void **)&s->u_alloc[i], (size_t)((nzl + 2) * NL * P) * sizeof(float), "u", cfg->ipc))
                   != PF_OK) {
            return bail(st);
        }
        if ((st = alloc(s, (void **)&s->q_alloc[i], (size_t)((nzl + 2) * 3 * NF * P) * sizeof(float), "q", cfg->ipc))
            != PF_OK)
            return bail(st);
        s->u[i] = (alm ? s->u_alloc[0] : s->u_alloc[i]) + NL * P;
        s->q[i] = s->q_alloc[i] + (int64_t)3 * NF * P;
    }
    if (alm) {
        const int np = gc.NI > 0 ? gc.NV : NL;   // p of every non-source node (DAG) or of the labels (Potts)
        if ((st = alloc(s, (void **)&s->p_alloc, (size_t)(nzl * np * P) * sizeof(float), "ALM p")) != PF_OK)
            return bail(st);
        if (gc.NI > 0 &&
            (st = alloc(s, (void **)&s->uint_alloc, (size_t)(nzl * gc.NI * P) * sizeof(float), "ALM u_int")) != PF_OK)
            return bail(st);
        if ((st = alloc(s, (void **)&s->pS_alloc, (size_t)(nzl * P) * sizeof(float), "ALM p_S")) != PF_OK)
            return bail(st);
    }
    const int64_t nzD = std::min(z1 + 1, dims->nz) - z0;  // owned + static halo plane above
    if ((st = alloc(s, (void **)&s->D_alloc, (size_t)((nzl + 1) * NL * P) * sizeof(float), "D")) != PF_OK)
        return bail(st);
    const int64_t nS = (S->kind == PF_S_SHARED_FIELD || S->kind == PF_S_SCALED_FIELD)
                           ? 1 : (S->kind == PF_S_FIELD_PER_NODE ? NF : 0);
    if (nS > 0 && (st = alloc(s, (void **)&s->S_alloc, (size_t)(nzl * nS * P) * sizeof(float), "S")) != PF_OK)
        return bail(st);
    if ((st = alloc(s, (void **)&s->d_resid, 64, "resid")) != PF_OK) return bail(st);
    if ((st = alloc(s, (void **)&s->d_err, 64, "err")) != PF_OK) return bail(st);
    e = cudaMemsetAsync(s->d_err, 0, 64, s->stream);
    if (e != cudaSuccess) { cuda_fail(s, e, "zero ticket"); return bail(PF_ERR_CUDA); }
    s->launch_parity = 0;
    if ((st = alloc(s, (void **)&s->d_flag, 64, "flag")) != PF_OK) return bail(st);
    if ((st = alloc(s, (void **)&s->d_energy, (size_t)(2 * kEnergyBlocks + 2) * sizeof(double), "energy")) != PF_OK)
        return bail(st);
    // inputs -> internal layouts (boundary [z][y][x] per label -> [z][l][y][pitch])
    e = cudaMemsetAsync(s->D_alloc, 0, (size_t)((nzl + 1) * NL * P) * sizeof(float), s->stream);
    if (e != cudaSuccess) { cuda_fail(s, e, "zero D"); return bail(PF_ERR_CUDA); }
    for (int l = 0; l < NL; ++l) {
        e = copy_volume(true, s->D_alloc + l * P, NL, (float *)D[l], s->nx, s->ny, s->pitch, nzD, s->stream);
        if (e != cudaSuccess) { cuda_fail(s, e, "upload D"); return bail(PF_ERR_CUDA); }
    }
    if (cfg->d_bf16) {  // bf16 storage: round once on the device, drop the fp32 copy
        const int64_t nD = (nzl + 1) * NL * P;
        if ((st = alloc(s, (void **)&s->D16, (size_t)nD * sizeof(uint16_t), "D (bf16)")) != PF_OK) return bail(st);
        e = launch_f32_to_bf16(s->D_alloc, s->D16, nD, s->stream);
        if (e != cudaSuccess) { cuda_fail(s, e, "D -> bf16"); return bail(PF_ERR_CUDA); }
        s->launches++;
        cudaFreeAsync(s->D_alloc, s->stream);
        s->D_alloc = nullptr;
        s->device_bytes -= nD * (int64_t)sizeof(float);
    }
    if (nS > 0) {
        e = cudaMemsetAsync(s->S_alloc, 0, (size_t)(nzl * nS * P) * sizeof(float), s->stream);
        if (e != cudaSuccess) { cuda_fail(s, e, "zero S"); return bail(PF_ERR_CUDA); }
    }
    if (S->kind == PF_S_SHARED_FIELD || S->kind == PF_S_SCALED_FIELD) {
        if (!S->fields[0]) return bail(fail(PF_ERR_INVALID, "smoothness: fields[0] is NULL"));
        for (int p = 0; p < NF; ++p)  // per-node factor of the shared field
            s->gc.g.s[p] = S->kind == PF_S_SHARED_FIELD ? 1.f : S->scalars[gc.node_of_pos[p]];
        e = copy_volume(true, s->S_alloc, 1, (float *)S->fields[0], s->nx, s->ny, s->pitch, nzl, s->stream);
        if (e != cudaSuccess) { cuda_fail(s, e, "upload S"); return bail(PF_ERR_CUDA); }
    } else if (S->kind == PF_S_FIELD_PER_NODE) {
        for (int p = 0; p < NF; ++p) {
            const int v = gc.node_of_pos[p];
            if (!S->fields[v - 1]) return bail(fail(PF_ERR_INVALID, "smoothness: fields[%d] is NULL", v - 1));
            e = copy_volume(true, s->S_alloc + p * P, NF, (float *)S->fields[v - 1], s->nx, s->ny, s->pitch, nzl,
                            s->stream);
            if (e != cudaSuccess) { cuda_fail(s, e, "upload S"); return bail(PF_ERR_CUDA); }
        }
    } else {
        for (int p = 0; p < NF; ++p) s->gc.g.s[p] = S->scalars[gc.node_of_pos[p]];
    }
    if (nS > 0) {
        cudaMemsetAsync(s->d_flag, 0, 4, s->stream);
        launch_check_nonneg(s->S_alloc, nzl * nS * P, s->d_flag, s->stream);
        s->launches++;
        unsigned int flag = 0;
        cudaMemcpyAsync(&flag, s->d_flag, 4, cudaMemcpyDeviceToHost, s->stream);
        e = cudaStreamSynchronize(s->stream);
        if (e != cudaSuccess) { cuda_fail(s, e, "validate S"); return bail(PF_ERR_CUDA); }
        if (flag) return bail(fail(PF_ERR_INVALID, "smoothness: S must be >= 0 and finite everywhere"));
    }
    if ((st = init_state(s)) != PF_OK) return bail(st);
    // kernel configuration
    {
        const void *fn = s->staged ? s->sinfo.func : s->kinfo.func;
        const int thr = s->staged ? s->sinfo.threads : s->kinfo.threads;
        const int smb = s->staged ? s->staged_smem : s->kinfo.smem_bytes;
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smb);
        if (e != cudaSuccess) { cuda_fail(s, e, "cudaFuncSetAttribute"); return bail(PF_ERR_CUDA); }
        cudaFuncAttributes fa;
        if (cudaFuncGetAttributes(&fa, fn) == cudaSuccess) s->regs = fa.numRegs;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&s->ctas_per_sm, fn, thr, smb);
    }
    if (s->staged) {
        const int ty = s->sinfo.tile_y;
        s->s_ch = (S->kind == PF_S_SHARED_FIELD || S->kind == PF_S_SCALED_FIELD) ? 1
                                                                                   : (S->kind == PF_S_FIELD_PER_NODE ? NF : 0);
        bool ok = true;
        // boxes: the cluster kernel's CTAs stage half of the labels (channel boxes of NL/2, three q loads)
        const int cq = s->cluster ? NL / 2 : 3 * NF, cl = s->cluster ? NL / 2 : NL;
        for (int i = 0; i < 2; ++i) {
            ok = ok && encode4d(&s->tm_q[i], s->q_alloc[i], s->nx, s->ny, s->pitch, (int64_t)3 * NF, nzl + 2, 40,
                                ty + 2, cq);
            ok = ok && encode4d(&s->tm_u[i], s->u_alloc[i], s->nx, s->ny, s->pitch, NL, nzl + 2, 36, ty + 1, cl);
        }
        for (int i = 0; i < 2; ++i) {
            // OSTAGE 2 stores one flow row per warp, OSTAGE 1 the whole tile
            ok = ok && encode4d(&s->tm_qo[i], s->q_alloc[i], s->nx, s->ny, s->pitch, (int64_t)3 * NF, nzl + 2, 32,
                                s->sinfo.ostage == 2 ? 1 : ty,
                                s->sinfo.ostage == 2 ? NF / s->sinfo.groups : (s->cluster ? NL / 2 : 3 * NF));
            ok = ok && encode4d(&s->tm_uo[i], s->u_alloc[i], s->nx, s->ny, s->pitch, NL, nzl + 2, 32, ty, cl);
        }
        if (s->D16)  // bf16 rows: a 40-element (80-byte) box keeps the 16-byte box-width rule
            ok = ok && encode4d(&s->tm_D, s->D16, s->nx, s->ny, s->pitch, NL, nzl + 1, 40, ty + 1, cl, true);
        else
            ok = ok && encode4d(&s->tm_D, s->D_alloc, s->nx, s->ny, s->pitch, NL, nzl + 1, 36, ty + 1, cl);
        if (s->s_ch) ok = ok && encode4d(&s->tm_S, s->S_alloc, s->nx, s->ny, s->pitch, s->s_ch, nzl, 32, ty, s->s_ch);
        else memset(&s->tm_S, 0, sizeof(s->tm_S));
        if (!ok) return bail(fail(PF_ERR_CUDA, "cuTensorMapEncodeTiled failed"));
        s->tx_bytes = (unsigned)(4 * (40 * (ty + 2) * 3 * (s->cluster ? NL / 2 : NF) + 36 * (ty + 1) * cl +
                                      32 * ty * s->s_ch) +
                                 (s->D16 ? 2 * 40 : 4 * 36) * (ty + 1) * cl);
    }
    choose_chunking(s);
    e = cudaStreamSynchronize(s->stream);
    if (e != cudaSuccess) { cuda_fail(s, e, "create"); return bail(PF_ERR_CUDA); }
    *out = s;
    return PF_OK;
}

pf_status pf_reset(pf_solver *s) {
    pf_status st = check_usable(s);
    if (st != PF_OK) return st;
    DeviceGuard dg(s->device);
    // IPC-linked: the neighbours' last kernels (which write into this slab's halo planes) must be done
    // before the re-init, and their next kernels must start after it
    for (int i = 0; i < 2; ++i)
        if (s->nb_ev[i]) CK(cudaStreamWaitEvent(s->stream, s->nb_ev[i], 0), "wait neighbour");
    if ((st = init_state(s)) != PF_OK) return st;
    if (s->ipc_ev) CK(cudaEventRecord(s->ipc_ev, s->stream), "record");
    return PF_OK;
}

pf_status pf_set_stream(pf_solver *s, void *stream) {
    pf_status st = check_usable(s);
    if (st != PF_OK) return st;
    DeviceGuard dg(s->device);
    if (s->own_stream) {
        cudaStreamSynchronize(s->stream);
        cudaStreamDestroy(s->stream);
        s->own_stream = false;
    }
    s->stream = (cudaStream_t)stream;
    return PF_OK;
}

namespace {

// Launch items [ib, ie) of one iteration reading state `cur` (no swap).  ie == ib launches nothing.
pf_status launch_items(pf_solver *s, int ib, int ie, int check) {
    if (s->staged) {
        if (ie <= ib) return PF_OK;
        StagedArgs sa;
        memset(&sa, 0, sizeof(sa));
        sa.tm_D = s->tm_D;
        sa.tm_S = s->tm_S;
        sa.nx = (int)s->nx;
        sa.ny = (int)s->ny;
        sa.pitch = (int)s->pitch;
        sa.nzl = (int)s->nzl;
        sa.zg0 = (int)s->z0;
        sa.nzg = (int)s->nz;
        sa.zchunk = s->zchunk;
        sa.tiles_x = s->tiles_x;
        sa.tiles = s->tiles;
        sa.item_begin = ib;
        sa.items = ie;
        sa.nb = s->nb;
        sa.bplane0 = s->bplane[0];
        sa.bplane1 = s->bplane[1];
        sa.zlo = s->zlo;
        sa.zhi = s->zhi;
        sa.s_ch = s->s_ch;
        sa.cap = s->cfg.cap;
        sa.shift = s->cfg.shift;
        sa.tx_bytes = s->tx_bytes;
        sa.inv_c = 1.0f / s->cfg.c;
        sa.ctau = s->cfg.c * s->cfg.tau;
        sa.resid_bits = s->d_resid;
        sa.err_voxel = s->d_err;
        sa.g = s->gc.g;
        sa.tm_q = s->tm_q[s->cur];
        sa.tm_u = s->tm_u[s->cur];
        sa.tm_qo = s->tm_qo[1 - s->cur];
        sa.tm_uo = s->tm_uo[1 - s->cur];
        sa.q_in = s->q[s->cur];
        sa.u_out = s->u[1 - s->cur];
        sa.q_out = s->q[1 - s->cur];
        sa.check = check;
        if (s->link_below) {
            sa.link_below = 1;
            sa.tm_uo_nb = s->tm_uo_nb[1 - s->cur];
            sa.tm_qo_nb = s->tm_qo_nb[1 - s->cur];
            sa.nb_plane = s->nb_plane;
        }
        if (s->link_above) {
            sa.link_above = 1;
            sa.tm_qz_nb = s->tm_qz_nb[1 - s->cur];
        }
        sa.ticket = s->d_err + 1 + s->launch_parity;
        sa.ticket_next = s->d_err + 2 - s->launch_parity;
        // cluster kernel: 2 CTAs per item and one ticket grab per cluster
        const int per = s->cluster ? 2 : 1;
        const int grid = (int)std::min<int64_t>(s->sgrid / per, ie - ib) * per;
        void *args[] = {(void *)&sa};
        CK(cudaLaunchKernel(s->sinfo.func, dim3(grid), dim3(s->sinfo.threads), args, s->staged_smem, s->stream),
           s->cluster ? "launch pf_iter_cluster" : "launch pf_iter_staged");
        s->launch_parity ^= 1;
    } else {
        IterArgs a;
        memset(&a, 0, sizeof(a));
        a.D = s->Dptr();
        a.d_bf16 = s->D16 ? 1 : 0;
        a.S = s->S_alloc;
        a.nx = (int)s->nx;
        a.ny = (int)s->ny;
        a.pitch = (int)s->pitch;
        a.nzl = (int)s->nzl;
        a.zg0 = (int)s->z0;
        a.nzg = (int)s->nz;
        a.zchunk = s->zchunk;
        a.s_kind = s->s_kind == PF_S_SCALED_FIELD ? 1 : s->s_kind;
        a.cap = s->cfg.cap;
        a.shift = s->cfg.shift;
        a.inv_c = 1.0f / s->cfg.c;
        a.ctau = s->cfg.c * s->cfg.tau;
        a.resid_bits = s->d_resid;
        a.err_voxel = s->d_err;
        a.g = s->gc.g;
        a.check = check;
        a.u_in = s->u[s->cur];
        a.q_in = s->q[s->cur];
        a.u_out = s->u[1 - s->cur];
        a.q_out = s->q[1 - s->cur];
        void *args[] = {(void *)&a};
        CK(cudaLaunchKernel(s->kinfo.func, s->grid, dim3(s->kinfo.threads), args, s->kinfo.smem_bytes, s->stream),
           "launch pf_iter_kernel");
    }
    s->launches++;
    return PF_OK;
}

int check_this_iteration(pf_solver *s) {
    const int64_t it = s->iters + 1;
    return (s->cfg.check_every > 0 && it % s->cfg.check_every == 0) ? 1 : 0;
}

pf_status read_residual(pf_solver *s, bool any_check, float *residual) {
    if (any_check) s->last_resid_valid = true;
    if (!residual) return PF_OK;
    *residual = -1.f;
    pf_status st;
    if ((st = check_numeric(s)) != PF_OK) return st;
    if (any_check) {
        unsigned int bits = 0;
        CK(cudaMemcpyAsync(&bits, s->d_resid, sizeof(bits), cudaMemcpyDeviceToHost, s->stream), "read residual");
        CK(cudaStreamSynchronize(s->stream), "sync");
        float r;
        memcpy(&r, &bits, 4);
        *residual = r;
    }
    return PF_OK;
}

// Plain launch loop of n iterations (bookkeeping advanced as if executed).
pf_status launch_iterations(pf_solver *s, int32_t n, bool *any_check) {
    pf_status st;
    for (int t = 0; t < n; ++t) {
        const int check = check_this_iteration(s);
        if (check) {
            CK(cudaMemsetAsync(s->d_resid, 0, sizeof(unsigned int), s->stream), "reset residual");
            *any_check = true;
        }
        if (s->alm) {
            CK(launch_alm_iteration(alm_args(s, check), s->stream), "ALM iteration");
            s->launches += 2;
        } else if ((st = launch_items(s, 0, s->items, check)) != PF_OK) {
            return st;
        }
        s->cur = 1 - s->cur;
        s->iters += 1;
    }
    return PF_OK;
}

// Iterations per graph: even (ping-pong buffer and counter parity return to their start) and a multiple
// of check_every (the residual resets / checks sit at the same positions in every replay).
int graph_period(const pf_solver *s) {
    const int k = s->cfg.check_every;
    if (k <= 0) return 16;
    return (k % 2) ? 2 * k : k;
}

bool graph_aligned(const pf_solver *s) {
    const int k = s->cfg.check_every;
    return k <= 0 || s->iters % k == 0;
}

// Capture graph_period() iterations into s->graph (the state bookkeeping is restored afterwards: capture
// does not execute).  Captured on a private stream (the solver's may be the legacy default stream).
pf_status capture_graph(pf_solver *s) {
    const int P = graph_period(s);
    cudaStream_t cap = nullptr, real = s->stream;
    if (cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        s->graph_failed = true;
        return PF_OK;
    }
    const int cur0 = s->cur, par0 = s->launch_parity;
    const int64_t it0 = s->iters, l0 = s->launches;
    cudaGraph_t g = nullptr;
    bool ok = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    bool dummy = false;
    if (ok) {
        s->stream = cap;
        const pf_status st = launch_iterations(s, P, &dummy);
        s->stream = real;
        ok = cudaStreamEndCapture(cap, &g) == cudaSuccess && st == PF_OK;
    }
    s->cur = cur0;
    s->launch_parity = par0;
    s->iters = it0;
    s->launches = l0;
    if (ok) ok = cudaGraphInstantiate(&s->graph, g, 0) == cudaSuccess;
    if (g) cudaGraphDestroy(g);
    cudaStreamDestroy(cap);
    cudaGetLastError();
    if (!ok) {
        s->graph = nullptr;
        s->graph_failed = true;
        return PF_OK;
    }
    s->graph_iters = P;
    s->graph_cur = cur0;
    s->graph_parity = par0;
    return PF_OK;
}

}  // namespace

pf_status pf_iterate(pf_solver *s, int32_t n, float *residual) {
    pf_status st = check_usable(s);
    if (st != PF_OK) return st;
    if (n < 0) return fail(PF_ERR_INVALID, "n must be >= 0");
    if (s->link_below || s->link_above) return fail(PF_ERR_STATE, "linked slab: iterate with pf_iterate_linked / pf_ipc_step");
    if (s->phase_pending) return fail(PF_ERR_STATE, "pf_iterate: an iteration split by pf_iterate_phase is open");
    DeviceGuard dg(s->device);
    bool any_check = false;
    // whole periods as CUDA-graph replays (one graph launch instead of P kernel launches + memsets),
    // the rest as plain launches; PF_GRAPHS=0 disables
    static const bool graphs_on = !(getenv("PF_GRAPHS") && strcmp(getenv("PF_GRAPHS"), "0") == 0);
    const int P = graph_period(s);
    while (graphs_on && !s->alm && !s->graph_failed && n >= P && graph_aligned(s)) {
        if (!s->graph && (st = capture_graph(s)) != PF_OK) return st;
        if (!s->graph || s->cur != s->graph_cur || s->launch_parity != s->graph_parity) break;
        CK(cudaGraphLaunch(s->graph, s->stream), "graph launch");
        s->iters += P;
        s->launches += (int64_t)P * (s->cfg.check_every > 0 ? 1 : 1);
        any_check = any_check || s->cfg.check_every > 0;
        n -= P;
    }
    if ((st = launch_iterations(s, n, &any_check)) != PF_OK) return st;
    return read_residual(s, any_check, residual);
}

pf_status pf_run(pf_solver *s, int32_t max_iters, float tol, int32_t *iters_done, float *residual) {
    pf_status st = check_usable(s);
    if (st != PF_OK) return st;
    if (max_iters < 0 || !(tol >= 0.f)) return fail(PF_ERR_INVALID, "max_iters must be >= 0 and tol >= 0");
    if (s->cfg.check_every <= 0) return fail(PF_ERR_INVALID, "pf_run needs check_every > 0 (the residual cadence)");
    int32_t done = 0;
    float r = -1.f;
    while (done < max_iters) {
        // run up to and including the next check iteration; the residual read is the only host sync
        const int64_t k = s->cfg.check_every;
        const int32_t to_check = (int32_t)(k - (s->iters % k));
        const int32_t n = std::min<int32_t>(to_check, max_iters - done);
        float rr = -1.f;
        if ((st = pf_iterate(s, n, &rr)) != PF_OK) return st;
        done += n;
        if (rr >= 0.f) {
            r = rr;
            if (r <= tol) break;
        }
    }
    if (iters_done) *iters_done = done;
    if (residual) *residual = r;
    return PF_OK;
}

pf_status pf_iterate_phase(pf_solver *s, int32_t phase, float *residual) {
    pf_status st = check_usable(s);
    if (st != PF_OK) return st;
    if (phase != 0 && phase != 1) return fail(PF_ERR_INVALID, "phase must be 0 or 1");
    if (s->alm) return fail(PF_ERR_UNSUPPORTED, "pf_iterate_phase: not for the explicit-flow ALM");
    if (s->link_below || s->link_above) return fail(PF_ERR_STATE, "linked slab: iterate with pf_iterate_linked / pf_ipc_step");
    if ((phase == 0) == (s->phase_pending != 0))
        return fail(PF_ERR_STATE, phase == 0 ? "phase 0 issued twice" : "phase 1 without phase 0");
    DeviceGuard dg(s->device);
    const int check = check_this_iteration(s);
    if (phase == 0) {
        if (check) CK(cudaMemsetAsync(s->d_resid, 0, sizeof(unsigned int), s->stream), "reset residual");
        // global-load kernel: no split, the whole iteration runs in phase 0
        if ((st = launch_items(s, 0, s->staged ? s->items_b : 1, check)) != PF_OK) return st;
        s->phase_pending = 1;
        return PF_OK;
    }
    if (s->staged && (st = launch_items(s, s->items_b, s->items, check)) != PF_OK) return st;
    s->phase_pending = 0;
    s->cur = 1 - s->cur;
    s->iters += 1;
    return read_residual(s, check != 0, residual);
}

pf_status pf_get_labeling(pf_solver *s, float *u, uint8_t *argmax) {
    pf_status st = check_usable(s);
    if (st != PF_OK) return st;
    DeviceGuard dg(s->device);
    const int NL = s->gc.NL;
    const int64_t P = s->P, nzl = s->nzl;
    const int64_t V = s->nx * s->ny * nzl;
    if (u) {
        for (int l = 0; l < NL; ++l)
            CK(copy_volume(false, s->u[s->cur] + l * P, NL, u + l * V, s->nx, s->ny, s->pitch, nzl, s->stream),
               "download u");
    }
    if (argmax) {
        const bool dev = is_device_ptr(argmax);
        uint8_t *dst = argmax;
        // stream-ordered scratch from the (retained) pool: cudaMalloc / cudaFree would synchronize the device
        if (!dev) CK(cudaMallocAsync((void **)&dst, (size_t)V, s->stream), "argmax scratch");
        CK(launch_argmax(s->u[s->cur], dst, NL, (int)s->nx, (int)s->ny, (int)s->pitch, nzl, s->stream), "argmax kernel");
        s->launches++;
        if (!dev) {
            CK(cudaMemcpyAsync(argmax, dst, (size_t)V, cudaMemcpyDeviceToHost, s->stream), "download argmax");
            CK(cudaStreamSynchronize(s->stream), "sync");
            cudaFreeAsync(dst, s->stream);
        }
    }
    return check_numeric(s);
}

pf_status pf_get_node_labeling(pf_solver *s, int32_t node, float *u_node) {
    pf_status st = check_usable(s);
    if (st != PF_OK) return st;
    if (!u_node) return fail(PF_ERR_INVALID, "u_node is NULL");
    if (node < 0 || node >= s->gc.num_nodes) return fail(PF_ERR_INVALID, "node %d out of range", node);
    DeviceGuard dg(s->device);
    NodeWeights w;
    memset(&w, 0, sizeof(w));
    const int NL = s->gc.NL;
    for (int l = 0; l < NL && l < 16; ++l)
        w.W[l] = node == 0 ? 1.f : s->gc.W[s->gc.pos_of_node[node]][l];   // W_(S, B) = 1 (reading R9)
    const int64_t V = s->nx * s->ny * s->nzl;
    const bool dev = is_device_ptr(u_node);
    float *dst = u_node;
    if (!dev) CK(cudaMallocAsync((void **)&dst, (size_t)V * sizeof(float), s->stream), "node labeling scratch");
    CK(launch_node_labeling(s->u[s->cur], dst, w, NL, (int)s->nx, (int)s->ny, (int)s->pitch, s->nzl, s->stream),
       "node labeling kernel");
    s->launches++;
    if (!dev) {
        CK(cudaMemcpyAsync(u_node, dst, (size_t)V * sizeof(float), cudaMemcpyDeviceToHost, s->stream), "download");
        CK(cudaStreamSynchronize(s->stream), "sync");
        cudaFreeAsync(dst, s->stream);
    }
    return check_numeric(s);
}

pf_status pf_get_flows(pf_solver *s, float *q) {
    pf_status st = check_usable(s);
    if (st != PF_OK) return st;
    if (!q) return fail(PF_ERR_INVALID, "q is NULL");
    DeviceGuard dg(s->device);
    const int NV = s->gc.NV, NF = s->gc.NF, nd = s->ndim;
    const int64_t P = s->P, nzl = s->nzl;
    const int64_t V = s->nx * s->ny * nzl;
    for (int p = 0; p < NV; ++p) {
        const int v = s->gc.node_of_pos[p];
        for (int k = 0; k < nd; ++k) {
            float *dst = q + ((int64_t)(v - 1) * nd + k) * V;
            if (p >= NF) {  // node without a stored flow (Ishikawa end labels): identically 0
                if (is_device_ptr(dst))
                    CK(cudaMemsetAsync(dst, 0, (size_t)V * sizeof(float), s->stream), "zero flows");
                else
                    memset(dst, 0, (size_t)V * sizeof(float));
                continue;
            }
            CK(copy_volume(false, s->q[s->cur] + ((int64_t)k * NF + p) * P, (int64_t)3 * NF, dst, s->nx, s->ny, s->pitch,
                           nzl, s->stream),
               "download q");
        }
    }
    return check_numeric(s);
}

pf_status pf_get_energy(pf_solver *s, double *primal, double *dual) {
    pf_status st = check_usable(s);
    if (st != PF_OK) return st;
    DeviceGuard dg(s->device);
    EnergyArgs a;
    memset(&a, 0, sizeof(a));
    a.u = s->u[s->cur];
    a.q = s->q[s->cur];
    a.D = s->Dptr();
    a.d_bf16 = s->D16 ? 1 : 0;
    a.S = s->S_alloc;
    a.nx = (int)s->nx;
    a.ny = (int)s->ny;
    a.pitch = (int)s->pitch;
    a.nzl = (int)s->nzl;
    a.zg0 = (int)s->z0;
    a.nzg = (int)s->nz;
    a.ndim = 3;
    a.NI = s->gc.NI;
    a.NL = s->gc.NL;
    a.NV = s->gc.NV;
    a.NF = s->gc.NF;
    a.model = s->gc.model;
    a.s_kind = s->s_kind == PF_S_SCALED_FIELD ? 1 : s->s_kind;
    a.cap = s->cfg.cap;
    a.g = s->gc.g;
    CK(launch_energy(a, s->d_energy + 2, kEnergyBlocks, s->d_energy, s->stream), "energy kernel");
    s->launches += 2;
    double h[2];
    CK(cudaMemcpyAsync(h, s->d_energy, sizeof(h), cudaMemcpyDeviceToHost, s->stream), "download energy");
    CK(cudaStreamSynchronize(s->stream), "sync");
    if (primal) *primal = h[0];
    if (dual) *dual = h[1];
    return check_numeric(s);
}

pf_status pf_iterations(const pf_solver *s, int64_t *done) {
    if (!s || !done) return fail(PF_ERR_INVALID, "NULL argument");
    *done = s->iters;
    return PF_OK;
}

pf_status pf_halo_regions(pf_solver *s, pf_halo *h) {
    pf_status st = check_usable(s);
    if (st != PF_OK) return st;
    if (!h) return fail(PF_ERR_INVALID, "h is NULL");
    memset(h, 0, sizeof(*h));
    const int NV = s->gc.NF;  // flow-carrying nodes
    const int64_t P = s->P, nzl = s->nzl;
    float *u = s->u[s->cur], *q = s->q[s->cur];
    h->bytes_u = ups(s) * (int64_t)sizeof(float);
    h->bytes_q = qps(s) * (int64_t)sizeof(float);
    h->bytes_qz = s->ndim == 3 ? (int64_t)NV * P * (int64_t)sizeof(float) : 0;
    if (s->z0 > 0) {  // neighbour below exists
        h->send_down_u = u;
        h->send_down_q = q;
        if (s->ndim == 3) h->recv_down_qz = q - qps(s) + 2 * NV * P;
    }
    if (s->z1 < s->nz) {  // neighbour above exists
        h->recv_up_u = u + nzl * ups(s);
        h->recv_up_q = q + nzl * qps(s);
        if (s->ndim == 3) h->send_up_qz = q + (nzl - 1) * qps(s) + 2 * NV * P;
    }
    return PF_OK;
}

pf_status pf_exchange_local(pf_solver *const *solvers, int32_t n) {
    if (!solvers || n < 1) return fail(PF_ERR_INVALID, "need >= 1 solver");
    for (int i = 0; i < n; ++i) {
        pf_status st = check_usable(solvers[i]);
        if (st != PF_OK) return st;
    }
    for (int i = 0; i + 1 < n; ++i) {
        pf_solver *lo = solvers[i], *hi = solvers[i + 1];
        if (lo->z1 != hi->z0 || lo->nx != hi->nx || lo->ny != hi->ny || lo->gc.NF != hi->gc.NF)
            return fail(PF_ERR_INVALID, "exchange: solvers %d and %d are not consecutive slabs of one volume", i, i + 1);
    }
    // order: every receiver waits for every sender's pending work, copies on the receiver's stream,
    // then every sender waits for the copies that read its current state.
    std::vector<cudaEvent_t> ev(n);
    for (int i = 0; i < n; ++i) {
        pf_solver *s = solvers[i];
        DeviceGuard dg(s->device);
        CK(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming), "event");
        CK(cudaEventRecord(ev[i], s->stream), "record");
    }
    for (int i = 0; i < n; ++i) {
        pf_solver *s = solvers[i];
        DeviceGuard dg(s->device);
        if (i > 0) CK(cudaStreamWaitEvent(s->stream, ev[i - 1], 0), "wait");
        if (i + 1 < n) CK(cudaStreamWaitEvent(s->stream, ev[i + 1], 0), "wait");
    }
    for (int i = 0; i + 1 < n; ++i) {
        pf_solver *lo = solvers[i], *hi = solvers[i + 1];
        pf_halo hl, hh;
        pf_halo_regions(lo, &hl);
        pf_halo_regions(hi, &hh);
        pf_solver *s = lo;
        {
            DeviceGuard dg(lo->device);
            CK(cudaMemcpyAsync(hl.recv_up_u, hh.send_down_u, hl.bytes_u, cudaMemcpyDefault, lo->stream), "halo u");
            CK(cudaMemcpyAsync(hl.recv_up_q, hh.send_down_q, hl.bytes_q, cudaMemcpyDefault, lo->stream), "halo q");
        }
        s = hi;
        if (hh.bytes_qz) {
            DeviceGuard dg(hi->device);
            CK(cudaMemcpyAsync(hh.recv_down_qz, hl.send_up_qz, hh.bytes_qz, cudaMemcpyDefault, hi->stream), "halo qz");
        }
    }
    for (int i = 0; i < n; ++i) {
        pf_solver *s = solvers[i];
        DeviceGuard dg(s->device);
        CK(cudaEventRecord(ev[i], s->stream), "record");
    }
    for (int i = 0; i < n; ++i) {
        pf_solver *s = solvers[i];
        DeviceGuard dg(s->device);
        if (i > 0) CK(cudaStreamWaitEvent(s->stream, ev[i - 1], 0), "wait");
        if (i + 1 < n) CK(cudaStreamWaitEvent(s->stream, ev[i + 1], 0), "wait");
    }
    for (int i = 0; i < n; ++i) cudaEventDestroy(ev[i]);
    return PF_OK;
}

pf_status pf_link_slabs(pf_solver *const *solvers, int32_t n) {
    if (!solvers || n < 2) return fail(PF_ERR_INVALID, "need >= 2 solvers");
    for (int i = 0; i < n; ++i) {
        pf_status st = check_usable(solvers[i]);
        if (st != PF_OK) return st;
        const pf_solver *s = solvers[i];
        if (!s->staged || !(s->cluster || s->sinfo.ostage == 1))
            return fail(PF_ERR_UNSUPPORTED, "link: solver %d's kernel variant stores no whole tiles (use "
                                            "pf_exchange_local)", i);
        if (s->phase_pending) return fail(PF_ERR_STATE, "link: solver %d has an open split iteration", i);
    }
    for (int i = 0; i + 1 < n; ++i) {
        const pf_solver *lo = solvers[i], *hi = solvers[i + 1];
        if (lo->z1 != hi->z0 || lo->nx != hi->nx || lo->ny != hi->ny || lo->pitch != hi->pitch ||
            lo->gc.NF != hi->gc.NF || lo->gc.NL != hi->gc.NL || lo->cluster != hi->cluster || lo->cur != hi->cur ||
            lo->sinfo.tile_y != hi->sinfo.tile_y)
            return fail(PF_ERR_INVALID, "link: solvers %d and %d are not consecutive slabs of one volume in step", i,
                        i + 1);
    }
    for (int i = 0; i + 1 < n; ++i) {   // peer access between devices (TMA stores into the neighbour's memory)
        const int a = solvers[i]->device, b = solvers[i + 1]->device;
        if (a == b) continue;
        int ok1 = 0, ok2 = 0;
        cudaDeviceCanAccessPeer(&ok1, a, b);
        cudaDeviceCanAccessPeer(&ok2, b, a);
        if (!ok1 || !ok2) return fail(PF_ERR_UNSUPPORTED, "link: no peer access between devices %d and %d", a, b);
        {
            DeviceGuard dg(a);
            if (cudaDeviceEnablePeerAccess(b, 0) != cudaSuccess) cudaGetLastError();   // already enabled is fine
        }
        {
            DeviceGuard dg(b);
            if (cudaDeviceEnablePeerAccess(a, 0) != cudaSuccess) cudaGetLastError();
        }
    }
    for (int i = 0; i < n; ++i) {
        pf_solver *s = solvers[i];
        const int ty = s->sinfo.tile_y, NF = s->gc.NF, NL = s->gc.NL;
        const int cq = s->cluster ? NL / 2 : 3 * NF, cl = s->cluster ? NL / 2 : NL, cz = s->cluster ? NL / 2 : NF;
        bool ok = true;
        s->nb_below = i > 0 ? solvers[i - 1] : nullptr;
        s->nb_above = i + 1 < n ? solvers[i + 1] : nullptr;
        s->link_below = s->nb_below != nullptr;
        s->link_above = s->nb_above != nullptr;
        if (s->nb_below) s->nb_plane = (int)s->nb_below->nzl + 1;
        for (int b = 0; b < 2; ++b) {
            if (s->nb_below) {   // below neighbour's buffers: its upper halo plane receives our plane 0
                const pf_solver *t = s->nb_below;
                ok = ok && encode4d(&s->tm_uo_nb[b], t->u_alloc[b], t->nx, t->ny, t->pitch, NL, t->nzl + 2, 32, ty, cl);
                ok = ok && encode4d(&s->tm_qo_nb[b], t->q_alloc[b], t->nx, t->ny, t->pitch, (int64_t)3 * NF, t->nzl + 2,
                                    32, ty, cq);
            }
            if (s->nb_above) {   // above neighbour's buffers: its lower halo plane receives our last q^z
                const pf_solver *t = s->nb_above;
                ok = ok && encode4d(&s->tm_qz_nb[b], t->q_alloc[b], t->nx, t->ny, t->pitch, (int64_t)3 * NF, t->nzl + 2,
                                    32, ty, cz);
            }
        }
        if (!ok) return fail(PF_ERR_CUDA, "link: cuTensorMapEncodeTiled failed");
    }
    return PF_OK;
}

pf_status pf_iterate_linked(pf_solver *const *solvers, int32_t n, int32_t iters, float *residual) {
    if (!solvers || n < 1 || iters < 0) return fail(PF_ERR_INVALID, "need >= 1 solver and iters >= 0");
    for (int i = 0; i < n; ++i) {
        pf_status st = check_usable(solvers[i]);
        if (st != PF_OK) return st;
        if (i > 0 && solvers[i]->nb_below != solvers[i - 1])
            return fail(PF_ERR_INVALID, "iterate_linked: solvers are not linked in this order");
    }
    // iteration t+1 of a slab starts after iteration t of both neighbours: they write its next halo planes
    // (RAW) and read the buffers its next kernel writes into (WAR)
    std::vector<cudaEvent_t> ev[2];
    for (int e = 0; e < 2; ++e) {
        ev[e].resize(n);
        for (int i = 0; i < n; ++i) {
            pf_solver *s = solvers[i];
            DeviceGuard dg(s->device);
            CK(cudaEventCreateWithFlags(&ev[e][i], cudaEventDisableTiming), "event");
        }
    }
    bool any_check = false;
    pf_status st = PF_OK;
    for (int t = 0; t < iters && st == PF_OK; ++t) {
        std::vector<cudaEvent_t> &prev = ev[(t + 1) & 1], &curv = ev[t & 1];
        for (int i = 0; i < n; ++i) {
            pf_solver *s = solvers[i];
            DeviceGuard dg(s->device);
            if (t > 0) {
                if (i > 0) CK(cudaStreamWaitEvent(s->stream, prev[i - 1], 0), "wait");
                if (i + 1 < n) CK(cudaStreamWaitEvent(s->stream, prev[i + 1], 0), "wait");
            } else {   // the first iteration waits for whatever the neighbours had queued
                if (i > 0) {
                    CK(cudaEventRecord(curv[i - 1], solvers[i - 1]->stream), "record");
                    CK(cudaStreamWaitEvent(s->stream, curv[i - 1], 0), "wait");
                }
                if (i + 1 < n) {
                    CK(cudaEventRecord(curv[i + 1], solvers[i + 1]->stream), "record");
                    CK(cudaStreamWaitEvent(s->stream, curv[i + 1], 0), "wait");
                }
            }
            const int check = check_this_iteration(s);
            if (check) {
                CK(cudaMemsetAsync(s->d_resid, 0, sizeof(unsigned int), s->stream), "reset residual");
                any_check = true;
            }
            if ((st = launch_items(s, 0, s->items, check)) != PF_OK) break;
        }
        for (int i = 0; i < n && st == PF_OK; ++i) {
            pf_solver *s = solvers[i];
            DeviceGuard dg(s->device);
            CK(cudaEventRecord(curv[i], s->stream), "record");
            s->cur = 1 - s->cur;
            s->iters += 1;
        }
    }
    // the neighbours' last kernels wrote this slab's halo planes: later work on its stream waits for them
    if (iters > 0 && st == PF_OK) {
        std::vector<cudaEvent_t> &last = ev[(iters - 1) & 1];
        for (int i = 0; i < n; ++i) {
            pf_solver *s = solvers[i];
            DeviceGuard dg(s->device);
            if (i > 0) CK(cudaStreamWaitEvent(s->stream, last[i - 1], 0), "wait");
            if (i + 1 < n) CK(cudaStreamWaitEvent(s->stream, last[i + 1], 0), "wait");
        }
    }
    float r = -1.f;
    for (int i = 0; i < n && st == PF_OK; ++i) {
        float ri = -1.f;
        st = read_residual(solvers[i], any_check, residual ? &ri : nullptr);
        r = std::max(r, ri);
    }
    for (int e = 0; e < 2; ++e)
        for (int i = 0; i < n; ++i) cudaEventDestroy(ev[e][i]);
    if (residual) *residual = r;
    return st;
}

pf_status pf_ipc_export(pf_solver *s, pf_ipc_slab *out) {
    pf_status st = check_usable(s);
    if (st != PF_OK) return st;
    if (!out) return fail(PF_ERR_INVALID, "out is NULL");
    if (!s->ipc) return fail(PF_ERR_STATE, "ipc_export: create the solver with pf_config.ipc = 1");
    if (!s->staged || !(s->cluster || s->sinfo.ostage == 1))
        return fail(PF_ERR_UNSUPPORTED, "ipc_export: this kernel variant stores no whole tiles");
    DeviceGuard dg(s->device);
    memset(out, 0, sizeof(*out));
    for (int i = 0; i < 2; ++i) {
        CK(cudaIpcGetMemHandle((cudaIpcMemHandle_t *)out->u[i], s->u_alloc[i]), "ipc handle u");
        CK(cudaIpcGetMemHandle((cudaIpcMemHandle_t *)out->q[i], s->q_alloc[i]), "ipc handle q");
    }
    if (!s->ipc_ev) CK(cudaEventCreateWithFlags(&s->ipc_ev, cudaEventDisableTiming | cudaEventInterprocess), "ipc event");
    CK(cudaIpcGetEventHandle((cudaIpcEventHandle_t *)out->event, s->ipc_ev), "ipc event handle");
    CK(cudaEventRecord(s->ipc_ev, s->stream), "record");   // "my initial state is in place"
    out->nx = s->nx;
    out->ny = s->ny;
    out->nzl = s->nzl;
    out->z0 = s->z0;
    out->pitch = s->pitch;
    out->NF = s->gc.NF;
    out->NL = s->gc.NL;
    out->tile_y = s->sinfo.tile_y;
    out->cluster = s->cluster ? 1 : 0;
    out->cur = s->cur;
    return PF_OK;
}

pf_status pf_ipc_link(pf_solver *s, const pf_ipc_slab *below, const pf_ipc_slab *above) {
    pf_status st = check_usable(s);
    if (st != PF_OK) return st;
    if (!s->ipc || !s->ipc_ev) return fail(PF_ERR_STATE, "ipc_link: export first (pf_ipc_export)");
    DeviceGuard dg(s->device);
    const int ty = s->sinfo.tile_y, NF = s->gc.NF, NL = s->gc.NL;
    const int cq = s->cluster ? NL / 2 : 3 * NF, cl = s->cluster ? NL / 2 : NL, cz = s->cluster ? NL / 2 : NF;
    const pf_ipc_slab *nb[2] = {below, above};
    for (int side = 0; side < 2; ++side) {
        const pf_ipc_slab *t = nb[side];
        if (!t) continue;
        const bool adjacent = side == 0 ? t->z0 + t->nzl == s->z0 : t->z0 == s->z1;
        if (!adjacent || t->nx != s->nx || t->ny != s->ny || t->pitch != s->pitch || t->NF != NF || t->NL != NL ||
            t->tile_y != ty || t->cluster != (s->cluster ? 1 : 0) || t->cur != s->cur)
            return fail(PF_ERR_INVALID, "ipc_link: the %s blob is not this slab's neighbour in step",
                        side == 0 ? "below" : "above");
        void *ub[2] = {nullptr, nullptr}, *qb[2] = {nullptr, nullptr};
        for (int b = 0; b < 2; ++b) {
            CK(cudaIpcOpenMemHandle(&ub[b], *(const cudaIpcMemHandle_t *)t->u[b], cudaIpcMemLazyEnablePeerAccess),
               "open ipc u");
            s->ipc_opened.push_back(ub[b]);
            CK(cudaIpcOpenMemHandle(&qb[b], *(const cudaIpcMemHandle_t *)t->q[b], cudaIpcMemLazyEnablePeerAccess),
               "open ipc q");
            s->ipc_opened.push_back(qb[b]);
        }
        CK(cudaIpcOpenEventHandle(&s->nb_ev[side], *(const cudaIpcEventHandle_t *)t->event), "open ipc event");
        bool ok = true;
        for (int b = 0; b < 2; ++b) {
            if (side == 0) {   // below: its upper halo plane receives our plane 0
                ok = ok && encode4d(&s->tm_uo_nb[b], ub[b], t->nx, t->ny, t->pitch, NL, t->nzl + 2, 32, ty, cl);
                ok = ok && encode4d(&s->tm_qo_nb[b], qb[b], t->nx, t->ny, t->pitch, (int64_t)3 * NF, t->nzl + 2, 32,
                                    ty, cq);
            } else {           // above: its lower halo plane receives our last q^z
                ok = ok && encode4d(&s->tm_qz_nb[b], qb[b], t->nx, t->ny, t->pitch, (int64_t)3 * NF, t->nzl + 2, 32,
                                    ty, cz);
            }
        }
        if (!ok) return fail(PF_ERR_CUDA, "ipc_link: cuTensorMapEncodeTiled failed");
        if (side == 0) {
            s->link_below = true;
            s->nb_plane = (int)t->nzl + 1;
        } else {
            s->link_above = true;
        }
    }
    return PF_OK;
}

pf_status pf_ipc_step(pf_solver *s, float *residual) {
    pf_status st = check_usable(s);
    if (st != PF_OK) return st;
    if (!s->ipc || !s->ipc_ev) return fail(PF_ERR_STATE, "ipc_step: export and link first");
    DeviceGuard dg(s->device);
    // the neighbours' latest recorded iteration (the caller's host barrier makes it the previous one)
    for (int i = 0; i < 2; ++i)
        if (s->nb_ev[i]) CK(cudaStreamWaitEvent(s->stream, s->nb_ev[i], 0), "wait neighbour");
    const int check = check_this_iteration(s);
    if (check) CK(cudaMemsetAsync(s->d_resid, 0, sizeof(unsigned int), s->stream), "reset residual");
    if ((st = launch_items(s, 0, s->items, check)) != PF_OK) return st;
    CK(cudaEventRecord(s->ipc_ev, s->stream), "record");
    s->cur = 1 - s->cur;
    s->iters += 1;
    return read_residual(s, check != 0, residual);
}

pf_status pf_get_kernel_info(const pf_solver *s, pf_kernel_info *info) {
    if (!s || !info) return fail(PF_ERR_INVALID, "NULL argument");
    info->tile_x = kTX;
    info->tile_y = s->staged ? s->sinfo.tile_y : s->kinfo.tile_y;
    info->z_chunk = s->zchunk;
    info->threads_per_cta = s->staged ? s->sinfo.threads : s->kinfo.threads;
    info->ctas = (int)(s->grid.x * s->grid.y * s->grid.z);
    info->regs_per_thread = s->regs;
    info->smem_bytes = s->staged ? s->staged_smem : s->kinfo.smem_bytes;
    info->staged = s->staged ? 1 : 0;
    info->work_items = s->staged ? s->items : info->ctas;
    info->ctas_per_sm = s->ctas_per_sm;
    // algorithmic bytes per iteration: per end label u r/w + D r + q r/w,
    // per internal node q r/w, plus the capacity fields
    const int64_t V = s->nx * s->ny * s->nzl;
    // per end label: u r/w + D r (+ its flow r/w unless it carries none); per flow-carrying internal node:
    // its flow r/w
    const int64_t per_leaf = 4 + 4 + (s->D16 ? 2 : 4), per_flow = 8 * s->ndim;
    int64_t b = V * (per_leaf * s->gc.NL + per_flow * s->gc.NF);
    if (s->alm && s->gc.NI == 0)  // pass 1: q r/w, p r, u r (+ p_S r); pass 2: q r, D r, p w, u r/w (+ p_S r/w)
        b = V * ((int64_t)s->gc.NL * (8 * s->ndim + 4 + 4 + 4 * s->ndim + (s->D16 ? 2 : 4) + 4 + 8) + 12);
    else if (s->alm)  // DAG: per node pass 1 q r/w, p r, u r; pass 2 q r, p r/w, u r/w; D per label; p_S r, r/w
        b = V * ((int64_t)s->gc.NV * (8 * s->ndim + 4 + 4 + 4 * s->ndim + 8 + 8) +
                 (int64_t)s->gc.NL * (s->D16 ? 2 : 4) + 12);
    if (s->s_kind == PF_S_SHARED_FIELD || s->s_kind == PF_S_SCALED_FIELD) b += 4 * V;
    if (s->s_kind == PF_S_FIELD_PER_NODE) b += 4 * V * s->gc.NF;
    info->algorithmic_bytes_per_iteration = b;
    info->device_bytes = s->device_bytes;
    info->kernel_launches = s->launches;
    info->model = s->gc.model;
    info->flow_nodes = s->gc.NF;
    return PF_OK;
}

void pf_destroy(pf_solver *s) {
    if (!s) return;
    DeviceGuard dg(s->device);
    free_all(s);
    if (s->stream) cudaStreamSynchronize(s->stream);
    if (s->own_stream) cudaStreamDestroy(s->stream);
    delete s;
}

}  // extern "C"
