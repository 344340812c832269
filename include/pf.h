/*
 * pf.h -- C-ABI of the B200 pseudo-flow continuous max-flow solver (arXiv 1501.07844).
 *
 * The library (paper_1501_07844_b200/libpf.so) runs the per-iteration hot path of
 * the paper's Algorithm 1 (Potts), Algorithm 2 (HMF / DAGMF,
 * P:279-305) and Algorithm 3 (Ishikawa) on one sm_100a GPU per solver,
 * entirely in its own CUDA kernels; z-slab solvers cooperate across devices and
 * processes (pf_halo_regions, pf_exchange_local, pf_link_slabs, pf_ipc_*).  No torch types cross this boundary; PyTorch (above it) only provides
 * device selection, streams and process groups.
 *
 * Problem statement (BASELINE.json north_star):
 *   create(volume dims, label graph, data terms D_L, smoothness S_L), iterate(n),
 *   get_labeling.
 *
 * Conventions
 *   - Every call returns pf_status; PF_OK == 0.  On error a message is available
 *     from pf_last_error() (thread-local, valid until the next call on the thread).
 *     After PF_ERR_CUDA or PF_ERR_NUMERIC the solver is poisoned: every later call
 *     except pf_destroy returns PF_ERR_STATE.
 *   - Boundary layout of every volume: x fastest, then y, then z (V = nx*ny*nz_local
 *     values).  End labels (leaves) are numbered in increasing node-id order; that
 *     number is the label id written by pf_get_labeling.
 *   - Pointers may be host or device memory (detected per call with
 *     cudaPointerGetAttributes).  Inputs are copied during the call and the caller
 *     keeps ownership; outputs go into caller-allocated buffers.
 *   - One solver per device; a solver is not thread-safe.  Work is issued on the
 *     solver's stream (default: a stream created by pf_create; see pf_set_stream);
 *     calls that return data to the host synchronize that stream.
 *
 * Spatial discretization (readings R4, R5):
 *   nabla = forward differences, 0 at the last index of each axis;
 *   div   = -nabla^T (backward differences, q^k(-1) = 0);
 *   |q(x)| <= S(x) is the Euclidean ball (PF_CAP_L2, isotropic TV) or the box
 *   (PF_CAP_LINF, anisotropic l1 TV).
 */
#ifndef PF_H_
#define PF_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pf_solver pf_solver; /* opaque; owns all of its device memory */

typedef enum {
    PF_OK = 0,
    PF_ERR_INVALID = 1, /* bad dims, config, pointers, slab range */
    PF_ERR_GRAPH = 2,   /* label graph violates the DAGMF assumptions (all violations listed) */
    PF_ERR_OOM = 3,     /* device allocation failed */
    PF_ERR_CUDA = 4,    /* CUDA runtime error (message carries cudaGetErrorString) */
    PF_ERR_UNSUPPORTED = 5, /* graph beyond 31 non-source nodes / 16 end labels, or an unsupported combination */
    PF_ERR_NUMERIC = 6, /* a(x) <= 0 or not finite detected at a check (message names the voxel) */
    PF_ERR_STATE = 7    /* solver poisoned by an earlier error, or calls out of order (split iterations,
                           linked slabs, IPC protocol) */
} pf_status;

typedef enum { PF_CAP_L2 = 0, PF_CAP_LINF = 1 } pf_capacity;

/* Exponent shift of the label update (reading R1).  PF_SHIFT_MIN
 * subtracts m(x) = min over end labels of d_L(x) before exp (log-sum-exp form);
 * PF_SHIFT_NONE is the literal listing P:147 / P:290. */
typedef enum { PF_SHIFT_MIN = 0, PF_SHIFT_NONE = 1 } pf_shift;

typedef struct {
    int32_t ndim;           /* 2 or 3 */
    int64_t nx, ny, nz;     /* GLOBAL extents, each >= 1; nz == 1 when ndim == 2 */
} pf_dims;

/* Label graph.  Node 0 is the source S.  Edge e is
 * parent[e] -> child[e] with weight w_(parent,child) = weight[e] > 0.  End labels
 * L = {L : L.C empty}.  Requirements (PF_ERR_GRAPH otherwise):
 * acyclic, S has no parents, every node reachable from S, >= 2 end labels,
 * weights > 0, and W_(S,L) = 1 for every end label (reading R9: needed for
 * sum_L u_L = 1 <=> u_S = 1).  A Potts model is the star S -> L_k. */
typedef struct {
    int32_t num_nodes;
    int32_t num_edges;
    const int32_t *parent;
    const int32_t *child;
    const float *weight;
} pf_graph;

typedef enum {
    PF_S_SCALAR_PER_NODE = 0, /* scalars[v] for v = 1..num_nodes-1 (scalars[0] ignored) */
    PF_S_SHARED_FIELD = 1,    /* fields[0]: one local volume shared by every node (Eq. 1 writes S(x)) */
    PF_S_FIELD_PER_NODE = 2,  /* fields[v-1]: one local volume per non-source node v (S_L(x)) */
    PF_S_SCALED_FIELD = 3     /* S_v(x) = scalars[v] * fields[0](x): one shared field, per-node factors */
} pf_s_kind;

typedef struct {
    pf_s_kind kind;
    const float *scalars;
    const float *const *fields;
} pf_smoothness;

typedef struct {
    float c;             /* proximal weight c > 0 (Eq. 6) */
    float tau;           /* flow step tau > 0 (Eq. 8) */
    int32_t cap;         /* pf_capacity */
    int32_t shift;       /* pf_shift */
    int32_t check_every; /* residual max|u_new - u_old| every k iterations; 0 = never */
    int32_t d_bf16;      /* 1: store D_L as bf16 (round-to-nearest-even at create; BASELINE.json
                          * north_star "optionally bf16-stored D_L"): the solver then
                          * solves the problem with data terms bf16(D_L) exactly, 2 B fewer per
                          * voxel-label-iteration.  0: fp32. */
    int32_t ipc;         /* 1: allocate the state so that another process can map it (pf_ipc_export);
                          * 0: stream-ordered pool allocations. */
    int32_t method;      /* PF_METHOD_PSEUDO_FLOW (default): Alg. 1 / 2 / 3.  PF_METHOD_EXPLICIT_ALM: the
                          * explicit-flow ("full-flow") augmented-Lagrangian solver that stores
                          * the source / sink flows -- Eq. 3 for Potts, Eq. 11 for
                          * HMF / DAG graphs -- the comparison arm of SURVEY 8(f2): c = the ALM penalty, tau
                          * = its flow step; whole volumes, scalar / shared / per-node capacities, <= 16
                          * non-source nodes, no Ishikawa model (else PF_ERR_UNSUPPORTED); no split or
                          * linked iterations. */
    int32_t u_half;      /* 1: store the labeling state lambda = log2 u as IEEE binary16 instead of fp32
                          * (reduced-precision storage): 4 B fewer per voxel-label-iteration
                          * (lambda read + written: 36 -> 32 in 3-D).  Every arithmetic step stays fp32; each stored lambda is
                          * rounded to nearest binary16, a relative error <= 2^-11 |lambda|, i.e. an absolute
                          * error in u <= 2^-11 u |ln u| <= 2^-11 / e = 1.8e-4 per store (R25 for the
                          * re-derived parity bar).  Needs the TMA-staged kernels (PF_ERR_UNSUPPORTED for the
                          * global-load fallback and the explicit-flow ALM).  0: fp32. */
    int32_t tblock;      /* 2: temporal blocking -- TWO iterations per HBM pass: pf_iterate runs
                          * pairs of iterations in one fused launch that keeps iteration t's flows, labels and
                          * masses on chip for iteration t + 1 (an odd remainder runs as one ordinary iteration);
                          * bitwise the same results as tblock = 0.  Supported for Potts models with 2..4 labels
                          * on whole volumes with scalar or shared-field capacities and fp32 storage
                          * (PF_ERR_UNSUPPORTED otherwise: the on-chip state of larger graphs does not fit the
                          * 227 KB of shared memory per CTA).  0 (default): one iteration
                          * per pass. */
} pf_config;

enum { PF_METHOD_PSEUDO_FLOW = 0, PF_METHOD_EXPLICIT_ALM = 1 };

/* z-slab of a volume split along z across ranks / devices.
 * The solver owns global planes [z_begin, z_end).  Inputs D_L cover
 * [z_begin, min(z_end + 1, nz)): the owned slab plus the static halo plane above
 * it (absent at the top of the volume).  Smoothness fields cover the owned slab. */
typedef struct {
    int64_t z_begin, z_end;
} pf_slab;

/* Ishikawa model (Alg. 3).  A graph that is the Ishikawa chain -- level nodes N_1..N_N with
 * S -> N_1 -> ... -> N_N, end labels L_0..L_N (increasing node ids) with S -> L_0 and N_i -> L_i, all
 * weights 1 -- whose end labels have identically zero capacity (scalar 0, or factor 0 of a
 * PF_S_SCALED_FIELD) is solved by the dedicated Ishikawa kernels: flows are stored for the N level
 * nodes only (prefix excesses, suffix masses), N <= 15.  Any other graph runs Algorithm 2.
 *
 * Graph size: up to 31 non-source nodes and 16 end labels (else PF_ERR_UNSUPPORTED).  Graphs
 * with <= 4 internal and <= 16 non-source nodes (Potts up to 16 labels, the configs' HMF tree and DAG) run on
 * the fused one-pass kernels; larger ones on the generic two-pass kernels (pf_generic.cu: same arithmetic,
 * masses through an HBM scratch buffer), which take whole volumes with the fp32 label state only
 * (PF_ERR_UNSUPPORTED for a slab, ipc, u_half or tblock). */

/* Create a solver for the (slab of the) volume and initialise the state:
 * u_L = 1/|L|, q = 0 (reading R8).
 *   D    : array of |L| pointers, one volume per end label in node-id order.
 *   slab : NULL for the whole volume. */
pf_status pf_create(const pf_dims *dims, const pf_graph *graph, const float *const *D, const pf_smoothness *S,
                    const pf_config *cfg, const pf_slab *slab, pf_solver **out);

/* Re-initialise u and q (row a0) keeping D and S resident.  IPC-linked slabs (pf_ipc_*): every rank
 * resets, then a host barrier, before the next pf_ipc_step. */
pf_status pf_reset(pf_solver *s);

/* Run n iterations of the while-loop body of Alg. 1 / Alg. 2, one fused kernel
 * launch per iteration.  If residual != NULL it receives max over owned voxels
 * and end labels of |u_new - u_old| at the last iteration of this call that was a
 * check iteration (global count % check_every == 0), or -1 if none was.  A
 * residual != NULL synchronizes the stream.  Multi-slab: the halo planes must be
 * exchanged between calls (pf_halo_regions / pf_exchange_local); n must then be 1. */
pf_status pf_iterate(pf_solver *s, int32_t n, float *residual);

/* "while not converged" (Alg. 1, Alg. 2; reading R7): iterate until the residual
 * max|u_new - u_old| of a check iteration (every check_every-th, fused into the iteration kernel)
 * is <= tol, or max_iters iterations have run.  Only the check iterations synchronize the
 * stream (one 4-byte read).  iters_done (may be NULL) receives the iterations run by this call,
 * residual (may be NULL) the last residual read (-1 if none).  Errors: PF_ERR_INVALID
 * (max_iters < 0, tol < 0 or NaN, check_every == 0), PF_ERR_NUMERIC as pf_iterate. */
pf_status pf_run(pf_solver *s, int32_t max_iters, float tol, int32_t *iters_done, float *residual);

/* One iteration split in two launches so that a slab's halo exchange overlaps its interior
 * compute (BASELINE.json north_star "halo exchange ... overlapped with
 * interior compute").  phase 0 computes the new state on the boundary planes only -- plane 0 if
 * there is a neighbour below, plane nz_local-1 if there is one above -- so the send regions of
 * the new state are final once phase 0 has completed on the stream; phase 1 computes every other
 * plane and completes the iteration (state swap).  The usual pattern: phase 0, record an event,
 * phase 1, pf_halo_regions (now describing the new state), exchange on another stream after the
 * event, and make the solver's stream wait for the exchange before the next phase 0.  Results
 * are bitwise those of pf_iterate(s, 1, residual).  residual: as pf_iterate, phase 1 only.
 * Errors: PF_ERR_INVALID (phase not 0/1), PF_ERR_STATE (phases out of order; pf_iterate while a
 * split iteration is open). */
pf_status pf_iterate_phase(pf_solver *s, int32_t phase, float *residual);

/* Current labeling of the owned slab: u (may be NULL) as [|L|][V_local] and the
 * thresholded labeling argmax (may be NULL) as uint8 [V_local], ties to the lowest
 * label id ("thresholded"), taken on the exported u values.  The pseudo-flow
 * state is log2 u (reading R18); u is exported as 2^lambda in fp32 (labels below
 * 2^-126 read as 0).  Host or device buffers. */
pf_status pf_get_labeling(pf_solver *s, float *u, uint8_t *argmax);

/* Leave `sms` SMs free during the interior launch of a split iteration (pf_iterate_phase(1)), so that a
 * halo-exchange kernel posted concurrently on another stream (NCCL P2P) finds SMs to run on: the
 * persistent grid otherwise occupies every SM with one ~216 KB CTA until the interior is done, and the
 * exchange could not overlap it.  The work-item queue lets any grid size finish the same items; results
 * are bitwise unchanged.  0 (default) = all SMs.  Errors: PF_ERR_INVALID (sms < 0 or >= the SM count). */
pf_status pf_set_reserved_sms(pf_solver *s, int32_t sms);

/* Labeling of any node v of the graph (row a9, "intermediate labels on demand"): u_v(x) =
 * sum_B W_(v,B) u_B(x) over the end labels (path weights P:199-209), u_S = 1.  node: graph node
 * id (0 = S).  u_node: [V_local] fp32, host or device.  Errors: PF_ERR_INVALID (node out of range, NULL). */
pf_status pf_get_node_labeling(pf_solver *s, int32_t node, float *u_node);

/* Spatial flows of the owned slab as [num_nodes-1][ndim][V_local], node-id order. */
pf_status pf_get_flows(pf_solver *s, float *q);

/* Energies over the owned slab, accumulated in fp64: primal E(u) (Eq. 1 P:53-59 /
 * Eq. 9, intermediate labels u_v = sum_B W_(v,B) u_B) and pseudo-flow dual
 * F(q) = sum_x min_L d_L(x) (Eq. 4 P:82-85 / Eq. 13).  Multi-slab: the
 * halos must be current; the caller sums over ranks. */
pf_status pf_get_energy(pf_solver *s, double *primal, double *dual);

/* The exact resumable state of the owned slab (checkpoint; SURVEY "Checkpoint/resume", test P11).  The
 * pseudo-flow solver stores the labeling as lambda_L = log2 u_L in fp32 (reading R18: a stored label cannot
 * underflow; pf_get_labeling exports u = 2^lambda), so a bitwise resume needs lambda itself:
 * u_log2: [|L|][z][y][x] of lambda (may be NULL); q: [num_nodes-1][ndim][z][y][x] as pf_get_flows (may be
 * NULL); host or device.  Errors: PF_ERR_UNSUPPORTED (explicit-flow ALM). */
pf_status pf_get_state(pf_solver *s, float *u_log2, float *q);

/* Restore a state -- checkpoint / resume (test P11: 150 + resume + 150 iterations == 300, bitwise, from
 * pf_get_state), or start from a given labeling.  u: [|L|][z][y][x] of the owned slab, end-label order:
 * lambda = log2 u as pf_get_state returns it (u_is_log2 = 1), or the labeling u itself (u_is_log2 = 0,
 * converted with a correctly rounded log2; u = 0 is a dead label, lambda = -inf).  q: [num_nodes-1][ndim]
 * [z][y][x], node-id order (as pf_get_flows; the zero flows of Ishikawa end labels are not read);
 * host or device pointers, read before the call returns (host) or in stream order (device); the caller
 * keeps ownership.  `iterations` = pf_iterations at save time: it fixes which later iterations are
 * residual-check iterations.  c and tau are not part of the state (pf_set_step).  Slab solvers: only
 * the owned planes are written -- refresh the halo planes with the exchange before iterating.
 * Errors: PF_ERR_INVALID (NULL u / q, negative iterations), PF_ERR_UNSUPPORTED (explicit-flow ALM,
 * whose state also holds p and p_S). */
pf_status pf_set_state(pf_solver *s, const float *u, const float *q, int64_t iterations, int32_t u_is_log2);

/* Change the step constants c (entropic proximal weight, Eq. 7 / P:119) and tau (flow step)
 * between calls, e.g. for a c-annealing schedule; the state is kept.  Errors:
 * PF_ERR_INVALID (non-positive or non-finite). */
pf_status pf_set_step(pf_solver *s, float c, float tau);

/* Iterations run since create / reset. */
pf_status pf_iterations(const pf_solver *s, int64_t *done);

/* Issue all work on `stream` (a cudaStream_t, may be NULL for the legacy default stream). */
pf_status pf_set_stream(pf_solver *s, void *stream);

/* Halo planes of the CURRENT state.  After an iteration,
 * the solver's neighbour below (rank-1) needs this solver's first-plane u and q,
 * the neighbour above (rank+1) needs this solver's last-plane q^z.  Each region is
 * a contiguous device range: send regions are read, recv regions are written by
 * the exchange.  Entries of a missing neighbour are NULL / 0. */
typedef struct {
    void *send_down_u, *recv_up_u;   /* |L| planes: own plane 0 -> below; halo plane above <- above */
    void *send_down_q, *recv_up_q;   /* ndim*(num_nodes-1) planes */
    void *send_up_qz, *recv_down_qz; /* (num_nodes-1) planes: own last plane q^z -> above; halo below <- below */
    int64_t bytes_u, bytes_q, bytes_qz;
} pf_halo;

pf_status pf_halo_regions(pf_solver *s, pf_halo *h);

/* Single-process exchange between consecutive slabs solvers[0..n-1] (ascending z),
 * possibly on different devices (peer copies).  Issued on each receiver's stream
 * after the senders' pending work. */
pf_status pf_exchange_local(pf_solver *const *solvers, int32_t n);

/* Fused halo exchange for consecutive z-slab solvers[0..n-1] (ascending z) driven from one process,
 * on one or several devices with peer access: after linking, every iteration
 * kernel also TMA-stores its boundary planes of the new state straight into the neighbours' halo
 * planes (plane 0 -> the slab below, q^z of the last plane -> the slab above; peer memory over
 * NVLink), so no exchange step remains.  Requires the TMA-staged kernel variants that store whole
 * tiles (PF_ERR_UNSUPPORTED otherwise: use pf_exchange_local) and slabs at the same iteration.  Linked
 * solvers must be iterated together with pf_iterate_linked (pf_iterate / pf_iterate_phase return
 * PF_ERR_STATE) and destroyed together. */
pf_status pf_link_slabs(pf_solver *const *solvers, int32_t n);

/* `iters` iterations of every linked slab; iteration t+1 of a slab is ordered (events, no host sync)
 * after iteration t of both neighbours.  residual: as pf_iterate, max over the slabs. */
pf_status pf_iterate_linked(pf_solver *const *solvers, int32_t n, int32_t iters, float *residual);

/* Fused halo exchange across PROCESSES (one process per GPU, torchrun): the same in-kernel peer
 * stores as pf_link_slabs, with the neighbours' state buffers shared by CUDA IPC (NVLink peer memory),
 * ordered ON THE DEVICE by progress words (no host synchronisation per iteration).
 *   pf_ipc_export: the slab's buffers and its progress inbox as a plain blob for the neighbours.
 *     Needs pf_config.ipc = 1 and a tile-storing kernel variant.
 *   pf_ipc_link:   open the neighbours' blobs (NULL where there is none).
 *   pf_ipc_step:   one iteration: the stream waits (cuStreamWaitValue32, GEQ) until both neighbours
 *     have announced the previous step in this slab's inbox, runs the linked kernel (which also stores
 *     the boundary planes into the neighbours' halo planes), then writes this slab's step count into
 *     the neighbours' inboxes (cuStreamWriteValue32, after a memory barrier).  Iteration t+1 of a slab
 *     therefore starts only after iteration t of both neighbours: RAW on the halo planes it reads, WAR on
 *     the neighbour halo planes it writes.  pf_reset is a step of the same protocol (it re-initialises
 *     the halo planes the neighbours write into).
 * Protocol: export, exchange the blobs, link, one host barrier; then every rank issues the same sequence
 * of pf_ipc_step / pf_reset calls -- no host barrier per iteration (the ranks' streams run ahead on
 * their own).  residual: as pf_iterate.  Errors: PF_ERR_STATE (no ipc config / not exported),
 * PF_ERR_INVALID (blobs that are not this slab's neighbours at the same iteration), PF_ERR_UNSUPPORTED
 * (kernel variant, or stream memory operations unavailable). */
typedef struct {
    uint8_t u[2][64], q[2][64], event[64];   /* cudaIpcMemHandle_t x 4, (unused) */
    int64_t nx, ny, nzl, z0, pitch;
    int32_t NF, NL, tile_y, cluster, cur;
    uint8_t inbox[64];                       /* cudaIpcMemHandle_t of the progress inbox */
    uint32_t seq;                            /* protocol steps taken so far */
    int32_t u_half;                          /* pf_config.u_half of the slab */
} pf_ipc_slab;

pf_status pf_ipc_export(pf_solver *s, pf_ipc_slab *out);
pf_status pf_ipc_link(pf_solver *s, const pf_ipc_slab *below, const pf_ipc_slab *above);
pf_status pf_ipc_step(pf_solver *s, float *residual);

/* Static description of the kernel configuration (for reports). */
typedef struct {
    int32_t tile_x, tile_y, z_chunk, threads_per_cta, ctas, regs_per_thread, smem_bytes, ctas_per_sm;
    int64_t algorithmic_bytes_per_iteration;
    int64_t device_bytes;                    /* resident footprint of this solver */
    int64_t kernel_launches;                 /* this solver's own kernels launched so far */
    int32_t staged;                          /* 1: TMA-staged persistent kernel, 0: global-load kernel */
    int32_t work_items;                      /* (tile, z-chunk) items per iteration */
    int32_t model;                           /* 0: Alg. 1/2 (star / tree / DAG), 1: Alg. 3 (Ishikawa chain) */
    int32_t flow_nodes;                      /* nodes whose spatial flow is stored */
    int32_t cluster;                         /* 1: labels split over a 2-CTA cluster (pf_iter_cluster) */
    int32_t phase1_ctas;                     /* grid of a pf_iterate_phase(1) launch (see pf_set_reserved_sms) */
    int32_t tblock;                          /* iterations per HBM pass of pf_iterate (1 or 2, pf_config.tblock) */
} pf_kernel_info;

pf_status pf_get_kernel_info(const pf_solver *s, pf_kernel_info *info);

void pf_destroy(pf_solver *s);

const char *pf_last_error(void);

/* Library version string. */
const char *pf_version(void);

#ifdef __cplusplus
}
#endif

#endif /* PF_H_ */
