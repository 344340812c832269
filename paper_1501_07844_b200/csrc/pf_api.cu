// pf_api.cu -- the C-ABI of include/pf.h: device state and layouts, the per-iteration launch loop
// (rows a0-a8, CUDA-graph replay, convergence stop, split iterations), labeling (a9), energies.
// Graph compilation (a10) is in pf_graph.cu, the z-slab entry points (row e) in pf_slabs.cu.
#include "pf_internal.h"

using namespace pf;
using namespace pfi;

namespace pfi {


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



bool is_device_ptr(const void *p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}


pf_status cuda_fail(pf_solver *s, cudaError_t e, const char *what) {
    if (s) s->poisoned = true;
    cudaGetLastError();  // clear the (non-sticky) last-error state so it does not leak into other solvers
    return fail(PF_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}





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
    if (s->ipc_inbox) { cudaFree(s->ipc_inbox); s->ipc_inbox = nullptr; }
    if (s->ipc) {   // cudaMalloc'd state (exportable); synchronise before the synchronous frees
        cudaStreamSynchronize(s->stream);
        for (int i = 0; i < 2; ++i) {
            if (s->u_alloc[i]) cudaFree(s->u_alloc[i]);
            if (s->q_alloc[i]) cudaFree(s->q_alloc[i]);
            s->u_alloc[i] = s->q_alloc[i] = nullptr;
        }
    }
    void *ptrs[] = {s->u_alloc[0], s->u_alloc[1], s->q_alloc[0], s->q_alloc[1], s->D_alloc, s->S_alloc, s->D16,
                    s->p_alloc, s->pS_alloc, s->uint_alloc, s->M_alloc, s->d_wide,
                    s->d_resid, s->d_err, s->d_flag, s->d_energy};
    for (void *p : ptrs)
        if (p) cudaFreeAsync(p, s->stream);
    cudaGetLastError();
    for (int i = 0; i < 2; ++i) s->u_alloc[i] = s->q_alloc[i] = nullptr;
    s->D_alloc = s->S_alloc = nullptr;
    s->D16 = nullptr;
    s->p_alloc = s->pS_alloc = s->uint_alloc = nullptr;
    s->M_alloc = s->d_wide = nullptr;
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
    // u_L = 1/|L|, stored as lambda = log2 u (reading R18)
    const float lam0 = (float)(-std::log2((double)s->gc.NL));
    for (int i = 0; i < 2; ++i) {
        CK(s->cfg.u_half ? launch_fill_half(s->u_alloc[i], nu, lam0, s->stream)
                         : launch_fill(s->u_alloc[i], nu, lam0, s->stream), "init u");
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
        // tile order (pf_staged.cuh tile_origin): full rows.  Narrower strips (to bring a tile's y-neighbour
        // closer in the ticket order) measured slower on 768-wide planes: C5slab strips of 12 / 8 / 6 / 4 tiles
        // 7.15 / 7.21 / 7.32 / 8.77 ms vs 7.10 (full rows of 24), C4 strips of 5: 2.09 vs 1.73 ms (tools/ab.py).
        // Row groups (PF_STRIP = -h: h tile rows, column-major inside, the y-neighbour one ticket away and the
        // x-neighbour h) also measured slower: C5slab h = 2 / 4 / 8 7.06 / 7.17 / 8.69 vs 7.03 ms, DRAM reads
        // 21.2 / 21.7 / 26.5 vs 21.4 GB per iteration (profiles/r2/cluster_rowgroups.txt): the x-neighbour,
        // whose 256-byte blocks a q row shares, has to stay the adjacent ticket.
        s->strip = gx;
        if (const char *sp = getenv("PF_STRIP")) {   // experiments (tools/ab.py): force the strip width
            const int want = atoi(sp);
            if (want > 0) s->strip = std::min(want, gx);
            if (want < 0) s->strip = want;   // row groups of -want tile rows, column-major inside a group
        }
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

#ifndef PF_L2PROMO_DEFAULT
#define PF_L2PROMO_DEFAULT 3
#endif

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
              int bx, int by, int bc, int dtype) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    const int64_t es_b = dtype ? 2 : 4;
    cuuint64_t dims[4] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nch, (cuuint64_t)nplanes};
    cuuint64_t strides[3] = {(cuuint64_t)(pitch * es_b), (cuuint64_t)(pitch * ny * es_b),
                             (cuuint64_t)(pitch * ny * nch * es_b)};
    cuuint32_t box[4] = {(cuuint32_t)bx, (cuuint32_t)by, (cuuint32_t)bc, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    // L2 promotion of the TMA requests: PF_L2PROMO = 0 (none) / 1 (64 B) / 2 (128 B) / 3 (256 B) overrides the
    // default (experiments, tools/ab.py)
    static const int promo = [] {
        const char *e = getenv("PF_L2PROMO");
        return e && e[0] >= '0' && e[0] <= '3' ? e[0] - '0' : PF_L2PROMO_DEFAULT;
    }();
    const CUtensorMapL2promotion pr = promo == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                      : promo == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                      : promo == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                   : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    return fn(m, dtype == 1 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : dtype == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                                            : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
              4, (void *)base, dims,
              strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, pr,
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

}  // namespace pfi

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
    if (const char *fg = getenv("PF_L2FETCH"))   // experiments: device-wide L2 fetch granularity hint (32 / 64 / 128)
        cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(fg));
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
    // beyond the compiled kernel set: the generic two-pass path (pf_generic.cu), whole volumes, fp32 state
    // (PF_GENERIC=1, tests: any model-0 graph on the generic kernels -- bitwise those of the dense compiled kernels)
    const char *genv = getenv("PF_GENERIC");
    gc.generic = gc.model == 0 && (gc.NI > kMaxInternal || gc.NV > kMaxNodes || (genv && strcmp(genv, "1") == 0));
    if (gc.generic && (slab || cfg->ipc || cfg->u_half || cfg->tblock == 2))
        return fail(PF_ERR_UNSUPPORTED, "graph: %d internal + %d end nodes run on the generic kernels (beyond the "
                                        "compiled set of <= %d internal, <= %d non-source nodes): whole volumes, "
                                        "fp32 label state, no ipc / tblock", gc.NI, gc.NL, kMaxInternal, kMaxNodes);
    gc.NF = gc.model == 1 ? gc.NI : gc.NV;
    if (cfg->method != PF_METHOD_PSEUDO_FLOW && cfg->method != PF_METHOD_EXPLICIT_ALM)
        return fail(PF_ERR_INVALID, "config: bad method");
    const bool alm = cfg->method == PF_METHOD_EXPLICIT_ALM;
    if (alm && (gc.model != 0 || gc.NV > 16 || slab || S->kind == PF_S_SCALED_FIELD))
        return fail(PF_ERR_UNSUPPORTED, "explicit-flow ALM: Potts / HMF / DAG graphs (<= 16 non-source nodes), whole "
                                        "volumes, scalar, shared or per-node capacities only");

    if (cfg->ipc && alm) return fail(PF_ERR_UNSUPPORTED, "config: ipc is for the pseudo-flow kernels");
    if (cfg->u_half != 0 && cfg->u_half != 1) return fail(PF_ERR_INVALID, "config: u_half must be 0 or 1");
    if (cfg->u_half && (alm || cfg->d_bf16))
        return fail(PF_ERR_UNSUPPORTED, "config: u_half is for the pseudo-flow kernels with fp32 D");
    pf_solver *s = new pf_solver();
    s->alm = alm;
    s->ipc = cfg->ipc != 0;
    cudaGetDevice(&s->device);
    cudaDeviceGetAttribute(&s->sms, cudaDevAttrMultiProcessorCount, s->device);
    s->ndim = dims->ndim;
    s->nx = dims->nx;
    s->ny = dims->ny;
    s->nz = dims->nz;
    s->z0 = z0;
    s->z1 = z1;
    s->nzl = z1 - z0;
    // row pitch: 16-byte TMA strides for fp32 (multiple of 4) and, with bf16 D, for bf16 rows (of 8)
    s->pitch = (cfg->d_bf16 || cfg->u_half) ? (dims->nx + 7) / 8 * 8 : (dims->nx + 3) / 4 * 4;
    s->P = s->pitch * dims->ny;
    s->gc = gc;
    s->cfg = *cfg;
    s->s_kind = S->kind;
    if (gc.generic) {
        s->kinfo.func = generic_kernel_func();
        s->kinfo.threads = 256;
        s->kinfo.smem_bytes = 0;
        s->kinfo.tile_y = 8;
    } else if (!iter_kernel_lookup(gc.NI, gc.NL, gc.model, &s->kinfo)) {
        delete s;
        return fail(PF_ERR_UNSUPPORTED, "no compiled kernel for %d internal / %d end nodes", gc.NI, gc.NL);
    }
    {
        const char *env = getenv("PF_ITER_KERNEL");
        const bool want_global = env && strcmp(env, "global") == 0;
        // the graph's edge mask: a kernel specialised for exactly these edges is used when one is compiled in
        // (PF_DENSE_GRAPH=1, experiments: always the dense weight rows)
        uint64_t mask = 0;
        for (int i = 0; i < gc.NI && i < kMaxInternal; ++i)
            for (int j = 0; j < gc.NV && j < kMaxNodes; ++j)
                if (gc.g.w[i][j] != 0.f) mask |= 1ull << (i * 16 + j);
        if (gc.model != 0 || (getenv("PF_DENSE_GRAPH") && strcmp(getenv("PF_DENSE_GRAPH"), "1") == 0)) mask = kDenseMask;
        s->staged = !alm && !want_global && !gc.generic &&
                    staged_kernel_lookup(gc.NI, gc.NL, gc.model, cfg->d_bf16 ? 1 : 0, cfg->u_half ? 1 : 0, mask,
                                         &s->sinfo) &&
                    encode_fn() != nullptr;
        // Potts with many labels: the 2-CTA cluster split (scalar / shared capacities; PF_CLUSTER=0 disables)
        const char *cenv = getenv("PF_CLUSTER");
        if (s->staged && gc.model == 0 && gc.NI == 0 && S->kind != PF_S_FIELD_PER_NODE &&
            !(cenv && strcmp(cenv, "0") == 0)) {
            StagedKernelInfo ci{};
            if (cluster_kernel_lookup(gc.NL, cfg->d_bf16 ? 1 : 0, cfg->u_half ? 1 : 0, &ci)) {
                s->sinfo = ci;
                s->cluster = true;
            }
        }
        if (s->staged) {
            const int s_ch = (S->kind == PF_S_SHARED_FIELD || S->kind == PF_S_SCALED_FIELD)
                                 ? 1 : (S->kind == PF_S_FIELD_PER_NODE ? gc.NF : 0);
            s->staged_smem = s->sinfo.smem_bytes +
                             4 * s->sinfo.s_slots * ((s_ch * s->sinfo.tile_y * 32 + 31) / 32 * 32);   // S ring slots
            int maxsm = 0;
            cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, s->device);
            cudaFuncAttributes fa{};
            cudaFuncGetAttributes(&fa, s->sinfo.func);  // static shared words (work-queue slot) count too
            if (s->staged_smem + (int)fa.sharedSizeBytes > maxsm) s->staged = false;  // e.g. per-node S fields
        }
        if (cfg->u_half && !s->staged) {
            delete s;
            return fail(PF_ERR_UNSUPPORTED, "config: u_half needs the TMA-staged kernels (not the global-load fallback)");
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
        } else if ((st = alloc(s, (void **)&s->u_alloc[i], (size_t)((nzl + 2) * NL * P) * ubytes(s), "u", cfg->ipc))
                   != PF_OK) {
            return bail(st);
        }
        if ((st = alloc(s, (void **)&s->q_alloc[i], (size_t)((nzl + 2) * 3 * NF * P) * sizeof(float), "q", cfg->ipc))
            != PF_OK)
            return bail(st);
        s->u[i] = reinterpret_cast<float *>(reinterpret_cast<char *>(alm ? s->u_alloc[0] : s->u_alloc[i]) +
                                            NL * P * ubytes(s));   // plane 0 (storage: fp32 or binary16)
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
    if (gc.generic) {   // masses scratch of the two-pass generic iteration, and the graph for the energy kernel
        if ((st = alloc(s, (void **)&s->M_alloc, (size_t)(nzl * gc.NV * P) * sizeof(float), "masses (generic)")) != PF_OK)
            return bail(st);
        if ((st = alloc(s, (void **)&s->d_wide, sizeof(GraphWide), "graph (generic)")) != PF_OK) return bail(st);
    }
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
        for (int p = 0; p < NF; ++p) {  // per-node factor of the shared field
            s->gc.gw.s[p] = S->kind == PF_S_SHARED_FIELD ? 1.f : S->scalars[gc.node_of_pos[p]];
            if (p < kMaxNodes) s->gc.g.s[p] = s->gc.gw.s[p];
        }
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
        for (int p = 0; p < NF; ++p) {
            s->gc.gw.s[p] = S->scalars[gc.node_of_pos[p]];
            if (p < kMaxNodes) s->gc.g.s[p] = s->gc.gw.s[p];
        }
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
    if (gc.generic) {
        e = cudaMemcpyAsync(s->d_wide, &s->gc.gw, sizeof(GraphWide), cudaMemcpyHostToDevice, s->stream);
        if (e != cudaSuccess) { cuda_fail(s, e, "upload graph"); return bail(PF_ERR_CUDA); }
        e = cudaStreamSynchronize(s->stream);   // the source is host memory of the solver
        if (e != cudaSuccess) { cuda_fail(s, e, "upload graph"); return bail(PF_ERR_CUDA); }
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
            // binary16 lambda: 40-element (80-byte) boxes keep the 16-byte box-width rule
            ok = ok && encode4d(&s->tm_u[i], s->u_alloc[i], s->nx, s->ny, s->pitch, NL, nzl + 2, cfg->u_half ? 40 : 36,
                                ty + 1, cl, cfg->u_half ? 2 : 0);
        }
        for (int i = 0; i < 2; ++i) {
            // OSTAGE 2 stores one flow row per warp, OSTAGE 1 the whole tile
            ok = ok && encode4d(&s->tm_qo[i], s->q_alloc[i], s->nx, s->ny, s->pitch, (int64_t)3 * NF, nzl + 2, 32,
                                s->sinfo.ostage == 2 ? 1 : ty,
                                s->sinfo.ostage == 2 ? NF / s->sinfo.groups : (s->cluster ? NL / 2 : 3 * NF));
            ok = ok && encode4d(&s->tm_uo[i], s->u_alloc[i], s->nx, s->ny, s->pitch, NL, nzl + 2, 32, ty, cl,
                                cfg->u_half ? 2 : 0);
        }
        if (s->D16)  // bf16 rows: a 40-element (80-byte) box keeps the 16-byte box-width rule
            ok = ok && encode4d(&s->tm_D, s->D16, s->nx, s->ny, s->pitch, NL, nzl + 1, 40, ty + 1, cl, 1);
        else
            ok = ok && encode4d(&s->tm_D, s->D_alloc, s->nx, s->ny, s->pitch, NL, nzl + 1, 36, ty + 1, cl);
        if (s->s_ch) ok = ok && encode4d(&s->tm_S, s->S_alloc, s->nx, s->ny, s->pitch, s->s_ch, nzl, 32, ty, s->s_ch);
        else memset(&s->tm_S, 0, sizeof(s->tm_S));
        if (!ok) return bail(fail(PF_ERR_CUDA, "cuTensorMapEncodeTiled failed"));
        s->tx_bytes = (unsigned)(4 * (40 * (ty + 2) * 3 * (s->cluster ? NL / 2 : NF) + 32 * ty * s->s_ch) +
                                 (cfg->u_half ? 2 * 40 : 4 * 36) * (ty + 1) * cl +
                                 (s->D16 ? 2 * 40 : 4 * 36) * (ty + 1) * cl);
    }
    {   // plain projection where no square can under- or overflow (pf_math.cuh flow_step3; PF_SCALED_PROJ=1 off)
        bool fast = s->s_ch == 0 && cfg->shift == PF_SHIFT_MIN && cfg->cap == PF_CAP_L2 && gc.NF > 0;
        for (int p = 0; p < gc.NF && fast; ++p) fast = s->gc.g.s[p] >= 0x1p-60f && std::isfinite(s->gc.g.s[p]);
        if (getenv("PF_SCALED_PROJ") && strcmp(getenv("PF_SCALED_PROJ"), "1") == 0) fast = false;
        s->fastproj = fast ? 1 : 0;
    }
    choose_chunking(s);
    if (cfg->tblock == 2) {   // two iterations per HBM pass (pf_tb2.cuh)
        const bool whole = z0 == 0 && z1 == dims->nz;
        const bool ok_graph = gc.model == 0 && gc.NI == 0 && gc.NL >= 2 && gc.NL <= 4;
        const bool ok_s = S->kind == PF_S_SCALAR_PER_NODE || S->kind == PF_S_SHARED_FIELD || S->kind == PF_S_SCALED_FIELD;
        if (alm || !s->staged || !whole || !ok_graph || !ok_s || cfg->d_bf16 || cfg->u_half || cfg->ipc ||
            !tb2_kernel_lookup(gc.NL, cfg->cap, &s->tinfo))
            return bail(fail(PF_ERR_UNSUPPORTED, "config: tblock = 2 needs a Potts model with 2..4 labels on a whole "
                                                 "volume, scalar or shared capacities, fp32 storage"));
        const int ty = s->tinfo.tile_y, K = gc.NL;
        s->tb_smem = s->tinfo.smem_bytes;
        e = cudaFuncSetAttribute(s->tinfo.func, cudaFuncAttributeMaxDynamicSharedMemorySize, s->tb_smem);
        if (e != cudaSuccess) { cuda_fail(s, e, "cudaFuncSetAttribute (tb2)"); return bail(PF_ERR_CUDA); }
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, s->tinfo.func, s->tinfo.threads, s->tb_smem);
        bool ok = occ > 0;
        for (int i = 0; i < 2; ++i) {
            ok = ok && encode4d(&s->tb_q[i], s->q_alloc[i], s->nx, s->ny, s->pitch, 3 * K, nzl + 2, 36, ty + 4, 3 * K);
            ok = ok && encode4d(&s->tb_u[i], s->u_alloc[i], s->nx, s->ny, s->pitch, K, nzl + 2, 36, ty + 3, K);
            ok = ok && encode4d(&s->tb_uo[i], s->u_alloc[i], s->nx, s->ny, s->pitch, K, nzl + 2, 28, ty, K);
            ok = ok && encode4d(&s->tb_qo[i], s->q_alloc[i], s->nx, s->ny, s->pitch, 3 * K, nzl + 2, 28, ty, 3 * K);
        }
        ok = ok && encode4d(&s->tb_D, s->D_alloc, s->nx, s->ny, s->pitch, K, nzl + 1, 36, ty + 3, K);
        if (s->s_ch) ok = ok && encode4d(&s->tb_S, s->S_alloc, s->nx, s->ny, s->pitch, 1, nzl, 36, ty + 2, 1);
        else memset(&s->tb_S, 0, sizeof(s->tb_S));
        if (!ok) return bail(fail(PF_ERR_CUDA, "tblock: cuTensorMapEncodeTiled failed"));
        s->tb_tx = (unsigned)(4 * 36 * (3 * K * (ty + 4) + 2 * K * (ty + 3) + s->s_ch * (ty + 2)));
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->device);
        s->tb_tiles_x = (int)((s->nx + 27) / 28);
        s->tb_tiles = s->tb_tiles_x * (int)((s->ny + ty - 1) / ty);
        const int nch = best_chunks(s->tb_tiles, (int)nzl, (int64_t)sms * occ);
        s->tb_zchunk = (int)((nzl + nch - 1) / nch);
        s->tb_items = s->tb_tiles * (int)((nzl + s->tb_zchunk - 1) / s->tb_zchunk);
        s->tb_grid = (int)std::min<int64_t>((int64_t)sms * occ, s->tb_items);
        s->tb2 = true;
    } else if (cfg->tblock != 0) {
        return bail(fail(PF_ERR_INVALID, "config: tblock must be 0 or 2"));
    }
    e = cudaStreamSynchronize(s->stream);
    if (e != cudaSuccess) { cuda_fail(s, e, "create"); return bail(PF_ERR_CUDA); }
    *out = s;
    return PF_OK;
}

pf_status pf_reset(pf_solver *s) {
    pf_status st = check_usable(s);
    if (st != PF_OK) return st;
    DeviceGuard dg(s->device);
    // IPC-linked: a step of the device-side protocol -- the neighbours' last kernels (which write into this
    // slab's halo planes) must be done before the re-init, and their next kernels start after it
    const bool linked = s->ipc_exported && (s->link_below || s->link_above);
    if (linked && (st = ipc_wait_neighbours(s, s->ipc_seq)) != PF_OK) return st;
    if ((st = init_state(s)) != PF_OK) return st;
    if (linked) {
        s->ipc_seq += 1;
        if ((st = ipc_announce(s, s->ipc_seq)) != PF_OK) return st;
    }
    return PF_OK;
}

pf_status pf_set_state(pf_solver *s, const float *u, const float *q, int64_t iterations, int32_t u_is_log2) {
    pf_status st = check_usable(s);
    if (st != PF_OK) return st;
    if (s->alm) return fail(PF_ERR_UNSUPPORTED, "set_state: the explicit-flow ALM state also holds p, p_S");
    if (!u || !q) return fail(PF_ERR_INVALID, "set_state: u and q are required");
    if (iterations < 0) return fail(PF_ERR_INVALID, "set_state: iterations must be >= 0");
    if (u_is_log2 != 0 && u_is_log2 != 1) return fail(PF_ERR_INVALID, "set_state: u_is_log2 must be 0 or 1");
    DeviceGuard dg(s->device);
    const int NL = s->gc.NL, NV = s->gc.NV, NF = s->gc.NF, nd = s->ndim;
    const int64_t P = s->P, nzl = s->nzl;
    const int64_t V = s->nx * s->ny * nzl;
    // (a replayable graph captured the old state parity / iteration alignment)
    if (s->graph) {
        cudaStreamSynchronize(s->stream);
        cudaGraphExecDestroy(s->graph);
        s->graph = nullptr;
    }
    {   // lambda (or u) -> the internal storage, through a stream-ordered device copy for host inputs
        const float *src = u;
        float *scratch = nullptr;
        if (!is_device_ptr(u)) {
            CK(cudaMallocAsync((void **)&scratch, (size_t)V * NL * sizeof(float), s->stream), "u scratch");
            CK(cudaMemcpyAsync(scratch, u, (size_t)V * NL * sizeof(float), cudaMemcpyHostToDevice, s->stream), "upload u");
            src = scratch;
        }
        CK(launch_import_u(src, s->u[s->cur], NL, (int)s->nx, (int)s->ny, (int)s->pitch, nzl, ufmt(s), u_is_log2 ? 0 : 1,
                           s->stream),
           "import u");
        s->launches++;
        if (scratch) cudaFreeAsync(scratch, s->stream);
    }
    for (int p = 0; p < NF && p < NV; ++p) {   // nodes without a stored flow (Ishikawa end labels): not read
        const int v = s->gc.node_of_pos[p];
        for (int k = 0; k < nd; ++k)
            CK(copy_volume(true, s->q[s->cur] + ((int64_t)k * NF + p) * P, (int64_t)3 * NF,
                           const_cast<float *>(q) + ((int64_t)(v - 1) * nd + k) * V, s->nx, s->ny, s->pitch, nzl,
                           s->stream),
               "upload q");
    }
    CK(cudaMemsetAsync(s->d_err, 0xff, sizeof(unsigned long long), s->stream), "init err");
    if (!is_device_ptr(u) || !is_device_ptr(q)) CK(cudaStreamSynchronize(s->stream), "sync");   // host buffers
    s->iters = iterations;
    return PF_OK;
}

pf_status pf_set_step(pf_solver *s, float c, float tau) {
    pf_status st = check_usable(s);
    if (st != PF_OK) return st;
    if (!(c > 0.f) || !(tau > 0.f) || !std::isfinite(c) || !std::isfinite(tau))
        return fail(PF_ERR_INVALID, "set_step: c and tau must be finite and > 0");
    s->cfg.c = c;
    s->cfg.tau = tau;
    if (s->graph) {   // the captured launches carry the old constants
        DeviceGuard dg(s->device);
        cudaStreamSynchronize(s->stream);
        cudaGraphExecDestroy(s->graph);
        s->graph = nullptr;
    }
    return PF_OK;
}

pf_status pf_set_reserved_sms(pf_solver *s, int32_t sms) {
    pf_status st = check_usable(s);
    if (st != PF_OK) return st;
    if (sms < 0 || sms >= s->sms) return fail(PF_ERR_INVALID, "reserved SMs must be in [0, %d)", s->sms);
    s->reserved_sms = sms;
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

}  // extern "C"

namespace pfi {

// Launch items [ib, ie) of one iteration reading state `cur` (no swap).  ie == ib launches nothing.
int phase1_grid(const pf_solver *s) {
    if (!s->staged) return (int)(s->grid.x * s->grid.y * s->grid.z);
    const int per = s->cluster ? 2 : 1;
    int g = s->sgrid;
    if (s->reserved_sms > 0) g = std::min(g, std::max(per, (s->sms - s->reserved_sms) * std::max(1, s->ctas_per_sm)));
    return g / per * per;
}

pf_status launch_items(pf_solver *s, int ib, int ie, int check, int reserve_sms) {
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
        sa.strip = s->strip;
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
        sa.fastproj = s->fastproj;
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
        int sg = s->sgrid;
        if (reserve_sms > 0) sg = phase1_grid(s);   // leave SMs free for a concurrent exchange kernel
        const int grid = (int)std::min<int64_t>(sg / per, ie - ib) * per;
        void *args[] = {(void *)&sa};
        CK(cudaLaunchKernel(s->sinfo.func, dim3(grid), dim3(s->sinfo.threads), args, s->staged_smem, s->stream),
           s->cluster ? "launch pf_iter_cluster" : "launch pf_iter_staged");
        s->launch_parity ^= 1;
    } else if (s->gc.generic) {
        CK(launch_generic_iteration(s, check), "launch pf_generic_masses / pf_generic_flows");
        s->launches++;   // two kernels per iteration
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

pf_status launch_tb2(pf_solver *s, int check) {
    StagedArgs sa;
    memset(&sa, 0, sizeof(sa));
    sa.tm_q = s->tb_q[s->cur];
    sa.tm_u = s->tb_u[s->cur];
    sa.tm_D = s->tb_D;
    sa.tm_S = s->tb_S;
    sa.tm_uo = s->tb_uo[1 - s->cur];
    sa.tm_qo = s->tb_qo[1 - s->cur];
    sa.q_in = s->q[s->cur];
    sa.nx = (int)s->nx;
    sa.ny = (int)s->ny;
    sa.pitch = (int)s->pitch;
    sa.nzl = (int)s->nzl;
    sa.zg0 = 0;
    sa.nzg = (int)s->nz;
    sa.zchunk = s->tb_zchunk;
    sa.tiles_x = s->tb_tiles_x;
    sa.tiles = s->tb_tiles;
    sa.item_begin = 0;
    sa.items = s->tb_items;
    sa.s_ch = s->s_ch;
    sa.cap = s->cfg.cap;
    sa.shift = s->cfg.shift;
    sa.check = check;
    sa.tx_bytes = s->tb_tx;
    sa.inv_c = 1.0f / s->cfg.c;
    sa.ctau = s->cfg.c * s->cfg.tau;
    sa.resid_bits = s->d_resid;
    sa.err_voxel = s->d_err;
    sa.g = s->gc.g;
    sa.ticket = s->d_err + 1 + s->launch_parity;
    sa.ticket_next = s->d_err + 2 - s->launch_parity;
    void *args[] = {(void *)&sa};
    CK(cudaLaunchKernel(s->tinfo.func, dim3(s->tb_grid), dim3(s->tinfo.threads), args, s->tb_smem, s->stream),
       "launch pf_iter_tb2");
    s->launch_parity ^= 1;
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
    NvtxRange nv("pf check (residual read)");
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
        if (s->tb2 && n - t >= 2) {   // two iterations in one pass; the residual of the pair's last check iteration
            const int c1 = check_this_iteration(s);
            s->iters += 1;
            const int c2 = check_this_iteration(s);
            s->iters -= 1;
            if (c1 || c2) {
                CK(cudaMemsetAsync(s->d_resid, 0, sizeof(unsigned int), s->stream), "reset residual");
                *any_check = true;
            }
            if ((st = launch_tb2(s, c2 ? 2 : (c1 ? 1 : 0))) != PF_OK) return st;
            s->cur = 1 - s->cur;
            s->iters += 2;
            ++t;
            continue;
        }
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

// Iterations per graph: a multiple of check_every (the residual resets / checks sit at the same positions in
// every replay) whose launches return the ping-pong buffer and the ticket-counter parity to their start: an even
// number of launches -- 2 iterations, or 4 with two iterations per launch (tblock).
int graph_period(const pf_solver *s) {
    const int k = s->cfg.check_every;
    const int m = s->tb2 ? 4 : 2;
    if (k <= 0) return 16;
    int P = k;
    while (P % m) P += k;
    return P;
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
    s->graph_launches = s->launches - l0;   // kernels per replay (the generic path: two per iteration; tblock: 1/2)
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

}  // namespace pfi

extern "C" {

pf_status pf_iterate(pf_solver *s, int32_t n, float *residual) {
    pf_status st = check_usable(s);
    if (st != PF_OK) return st;
    if (n < 0) return fail(PF_ERR_INVALID, "n must be >= 0");
    if (s->link_below || s->link_above) return fail(PF_ERR_STATE, "linked slab: iterate with pf_iterate_linked / pf_ipc_step");
    if (s->phase_pending) return fail(PF_ERR_STATE, "pf_iterate: an iteration split by pf_iterate_phase is open");
    DeviceGuard dg(s->device);
    NvtxRange nv("pf_iterate");
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
        s->launches += s->graph_launches;
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
    NvtxRange nv(phase == 0 ? (check ? "pf boundary (check)" : "pf boundary") : (check ? "pf interior (check)" : "pf interior"));
    if (phase == 0) {
        if (check) CK(cudaMemsetAsync(s->d_resid, 0, sizeof(unsigned int), s->stream), "reset residual");
        // global-load kernel: no split, the whole iteration runs in phase 0
        if ((st = launch_items(s, 0, s->staged ? s->items_b : 1, check)) != PF_OK) return st;
        s->phase_pending = 1;
        return PF_OK;
    }
    if (s->staged && (st = launch_items(s, s->items_b, s->items, check, s->reserved_sms)) != PF_OK) return st;
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
    const int uf = ufmt(s);
    if (u && V > 0) {   // u = 2^lambda into a dense [l][z][y][x] volume (stream-ordered scratch for host outputs)
        const bool dev = is_device_ptr(u);
        float *dst = u;
        if (!dev) CK(cudaMallocAsync((void **)&dst, (size_t)V * NL * sizeof(float), s->stream), "u scratch");
        CK(launch_export_u(s->u[s->cur], dst, NL, (int)s->nx, (int)s->ny, (int)s->pitch, nzl, uf, 0, s->stream),
           "export u");
        s->launches++;
        if (!dev) {
            CK(cudaMemcpyAsync(u, dst, (size_t)V * NL * sizeof(float), cudaMemcpyDeviceToHost, s->stream),
               "download u");
            cudaFreeAsync(dst, s->stream);
        }
    }
    if (argmax) {
        const bool dev = is_device_ptr(argmax);
        uint8_t *dst = argmax;
        // stream-ordered scratch from the (retained) pool: cudaMalloc / cudaFree would synchronize the device
        if (!dev) CK(cudaMallocAsync((void **)&dst, (size_t)V, s->stream), "argmax scratch");
        CK(launch_argmax(s->u[s->cur], dst, NL, (int)s->nx, (int)s->ny, (int)s->pitch, nzl, uf, s->stream),
           "argmax kernel");
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
    CK(launch_node_labeling(s->u[s->cur], dst, w, NL, (int)s->nx, (int)s->ny, (int)s->pitch, s->nzl, ufmt(s),
                            s->stream),
       "node labeling kernel");
    s->launches++;
    if (!dev) {
        CK(cudaMemcpyAsync(u_node, dst, (size_t)V * sizeof(float), cudaMemcpyDeviceToHost, s->stream), "download");
        CK(cudaStreamSynchronize(s->stream), "sync");
        cudaFreeAsync(dst, s->stream);
    }
    return check_numeric(s);
}

pf_status pf_get_state(pf_solver *s, float *u_log2, float *q) {
    pf_status st = check_usable(s);
    if (st != PF_OK) return st;
    if (s->alm) return fail(PF_ERR_UNSUPPORTED, "get_state: the explicit-flow ALM state also holds p, p_S");
    DeviceGuard dg(s->device);
    const int NL = s->gc.NL;
    const int64_t P = s->P, nzl = s->nzl;
    const int64_t V = s->nx * s->ny * nzl;
    if (u_log2 && V > 0) {   // lambda as stored (fp32, or binary16 widened exactly)
        const bool dev = is_device_ptr(u_log2);
        float *dst = u_log2;
        if (!dev) CK(cudaMallocAsync((void **)&dst, (size_t)V * NL * sizeof(float), s->stream), "lambda scratch");
        CK(launch_export_u(s->u[s->cur], dst, NL, (int)s->nx, (int)s->ny, (int)s->pitch, nzl, ufmt(s), 1, s->stream),
           "export lambda");
        s->launches++;
        if (!dev) {
            CK(cudaMemcpyAsync(u_log2, dst, (size_t)V * NL * sizeof(float), cudaMemcpyDeviceToHost, s->stream),
               "download lambda");
            cudaFreeAsync(dst, s->stream);
        }
    }
    if (q) return pf_get_flows(s, q);
    CK(cudaStreamSynchronize(s->stream), "sync");
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
    a.ufmt = ufmt(s);
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
    a.gw = reinterpret_cast<const GraphWide *>(s->d_wide);   // generic graphs: weights and capacity scalars of every position
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
    const int64_t per_leaf = 2 * ubytes(s) + (s->D16 ? 2 : 4), per_flow = 8 * s->ndim;
    int64_t b = V * (per_leaf * s->gc.NL + per_flow * s->gc.NF);
    if (s->alm && s->gc.NI == 0)  // pass 1: q r/w, p r, u r (+ p_S r); pass 2: q r, D r, p w, u r/w (+ p_S r/w)
        b = V * ((int64_t)s->gc.NL * (8 * s->ndim + 4 + 4 + 4 * s->ndim + (s->D16 ? 2 : 4) + 4 + 8) + 12);
    else if (s->alm)  // DAG: per node pass 1 q r/w, p r, u r; pass 2 q r, p r/w, u r/w; D per label; p_S r, r/w
        b = V * ((int64_t)s->gc.NV * (8 * s->ndim + 4 + 4 + 4 * s->ndim + 8 + 8) +
                 (int64_t)s->gc.NL * (s->D16 ? 2 : 4) + 12);
    if (s->s_kind == PF_S_SHARED_FIELD || s->s_kind == PF_S_SCALED_FIELD) b += 4 * V;
    if (s->s_kind == PF_S_FIELD_PER_NODE) b += 4 * V * s->gc.NF;
    if (s->tb2) b /= 2;   // one pass moves the state once for two iterations
    info->algorithmic_bytes_per_iteration = b;
    info->device_bytes = s->device_bytes;
    info->kernel_launches = s->launches;
    info->model = s->gc.model;
    info->flow_nodes = s->gc.NF;
    info->cluster = s->cluster ? 1 : 0;
    info->phase1_ctas = phase1_grid(s);
    info->tblock = s->tb2 ? 2 : 1;
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
