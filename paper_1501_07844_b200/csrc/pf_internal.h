// pf_internal.h -- shared internals of the C-ABI implementation (pf_api.cu, pf_graph.cu, pf_slabs.cu):
// the solver object, error handling, and the launch helpers the multi-slab entry points reuse.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <cuda.h>
#include <nvtx3/nvToolsExt.h>

#include "pf.h"
#include "pf_alm.cuh"
#include "pf_aux.cuh"
#include "pf_cluster.cuh"
#include "pf_kernels.cuh"
#include "pf_staged.cuh"
#include "pf_tb2.cuh"

namespace pfi {

using namespace pf;

// last error message of this thread (pf_last_error) and the error constructor
extern thread_local std::string g_last_error;
pf_status fail(pf_status st, const char *fmt, ...);

// NVTX range for nsys timelines (boundary / interior / check / ipc step)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

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

bool is_device_ptr(const void *p);

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
    GraphConst g;    // dense weights of the compiled kernels (NI <= kMaxInternal, NV <= kMaxNodes)
    GraphWide gw;    // dense weights of every model-0 graph up to kWideNodes (the generic path, energies)
    bool generic = false;   // beyond the compiled kernel set: pf_generic.cu
    std::vector<std::vector<float>> W;  // W[pos][leaf slot] path weights
    std::vector<float> w_src;           // weight of the edge S -> position (0: none)
};

pf_status compile_graph(const pf_graph *gr, Compiled *out);

}  // namespace pfi

using namespace pf;

struct pf_solver {
    using Compiled = pfi::Compiled;
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
    float *M_alloc = nullptr;                         // generic path (pf_generic.cu): masses [z][v][y][pitch]
    float *d_wide = nullptr;                          // GraphWide on the device (energy kernel, generic graphs)
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
    // cross-process links (pf_ipc_*): state from cudaMalloc (IPC-exportable), a progress inbox the
    // neighbours announce their steps into, the neighbours' opened buffers and inbox words
    bool ipc = false;
    bool ipc_exported = false;
    uint32_t *ipc_inbox = nullptr;          // [0]: steps announced by the neighbour below, [1]: by the one above
    uint32_t *nb_inbox[2] = {nullptr, nullptr};   // the neighbours' inbox words this slab announces into
    uint32_t ipc_seq = 0;                   // protocol steps (pf_ipc_step / pf_reset) issued so far
    std::vector<void *> ipc_opened;
    // CUDA graph of `graph_iters` whole iterations (pf_iterate), replayed when the state matches the
    // capture: same ping-pong buffer, same counter parity, check iterations at the same positions
    cudaGraphExec_t graph = nullptr;
    int graph_iters = 0, graph_cur = 0, graph_parity = 0;
    bool graph_failed = false;
    int64_t graph_launches = 0;     // kernel launches one replay of the captured graph stands for
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
    int strip = 1;          // tile-order strip width in tiles (tile_origin)
    // boundary / interior split of the z-chunks (slabs with neighbours; pf_iterate_phase)
    int nb = 0, bplane[2] = {0, 0}, zlo = 0, zhi = 0, items_b = 0;
    int phase_pending = 0;  // 1 after pf_iterate_phase(0) until its phase 1
    int reserved_sms = 0;   // SMs a phase-1 launch leaves free (pf_set_reserved_sms)
    int fastproj = 0;       // plain projection is exact for this solver (flow_step3 SCALED = false)
    int sms = 148;
    unsigned int tx_bytes = 0;
    // two iterations per HBM pass (pf_config.tblock = 2, pf_tb2.cuh): its own tiles (28 wide), maps, chunking
    bool tb2 = false;
    StagedKernelInfo tinfo{};
    CUtensorMap tb_q[2], tb_u[2], tb_D, tb_S, tb_uo[2], tb_qo[2];
    int tb_smem = 0, tb_tiles_x = 0, tb_tiles = 0, tb_items = 0, tb_zchunk = 0, tb_grid = 0;
    unsigned int tb_tx = 0;
};

namespace pfi {

pf_status cuda_fail(pf_solver *s, cudaError_t e, const char *what);

#define CK(expr, what)                                     \
    do {                                                   \
        cudaError_t e__ = (expr);                          \
        if (e__ != cudaSuccess) return pfi::cuda_fail(s, e__, what); \
    } while (0)

inline int64_t ups(const pf_solver *s) { return (int64_t)s->gc.NL * s->P; }
// label state storage: 0 u fp32 (explicit-flow ALM), 1 lambda = log2 u fp32, 2 lambda binary16 (pf_config.u_half)
inline int ufmt(const pf_solver *s) { return s->alm ? 0 : (s->cfg.u_half ? 2 : 1); }
inline int64_t ubytes(const pf_solver *s) { return s->cfg.u_half ? 2 : 4; }
// q always carries 3 components internally (q^z == 0 for 2-D volumes), so the kernels need no ndim branch
inline int64_t qps(const pf_solver *s) { return (int64_t)3 * s->gc.NF * s->P; }

pf_status check_usable(const pf_solver *s);
pf_status check_numeric(pf_solver *s);
int check_this_iteration(pf_solver *s);
pf_status read_residual(pf_solver *s, bool any_check, float *residual);
pf_status launch_items(pf_solver *s, int ib, int ie, int check, int reserve_sms = 0);
pf_status launch_tb2(pf_solver *s, int check);   // iterations iters+1, iters+2 in one pass; check: 0, 1 or 2
int phase1_grid(const pf_solver *s);
// device-side ordering of IPC-linked slabs (pf_ipc_step, pf_reset): wait until both neighbours announced
// step `seq` in this slab's inbox / announce `seq` into theirs
pf_status ipc_wait_neighbours(pf_solver *s, uint32_t seq);
bool stream_mem_ops();
pf_status ipc_announce(pf_solver *s, uint32_t seq);
// dtype: 0 fp32, 1 bf16, 2 fp16 (binary16)
bool encode4d(CUtensorMap *m, const void *base, int64_t nx, int64_t ny, int64_t pitch, int64_t nch, int64_t nplanes,
              int bx, int by, int bc, int dtype = 0);

}  // namespace pfi

namespace pf {
// generic path (pf_generic.cu): graphs beyond the compiled kernel set, two kernels per iteration
cudaError_t launch_generic_iteration(const pf_solver *s, int check);
const void *generic_kernel_func();
}  // namespace pf
