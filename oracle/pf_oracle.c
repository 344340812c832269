/*
 * pf_oracle.c -- CPU ORACLE for the pseudo-flow iteration of arXiv 1501.07844.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  The
 * product path (paper_1501_07844_b200/) never includes, links or calls it, and
 * it shares no header, helper or constant with the CUDA code.
 *
 * Plain, slow, obviously-correct: fp64, one whole-field pass per line of the
 * paper's listings, in the listings' order and notation.  Single-threaded by
 * default; oracle_set_threads(n) splits every whole-field pass over n OpenMP
 * threads by voxel range.  Every pass is a per-voxel pure function (it writes
 * only voxel i of its output, from inputs no pass of the same loop writes), so
 * the result is bit-identical for any thread count; the
 * first-failing-voxel scans stay serial.
 *   oracle_potts    -- Algorithm 1
 *   oracle_dag      -- Algorithm 2, d_L recursion P:190-197
 *   oracle_ishikawa -- Algorithm 3
 *
 * Readings of what the paper leaves open:
 *   R1  exponent shift: shift==0 (SHIFT_MIN) subtracts m(x) = min over end
 *       labels of the exponent argument before exp; shift==1 (SHIFT_NONE) is the
 *       literal listing.
 *   R4  nabla = forward difference, 0 at the last index of each axis;
 *       div = its negative adjoint: sum_k q^k(x) - q^k(x-e_k), q^k(-1) = 0.
 *   R5  |q| <= S: cap==0 Euclidean ball, cap==1 box (|q^k| <= S, dual of l1-TV).
 *   R14 Proj: if |q| > S then q*S/|q| else q (S = 0, q = 0 gives 0).
 *   R8  q starts at 0; u starts at 1/|L| -- set by the caller.
 *   R18 no floor: the listings never set a label to 0, so the oracle does
 *       not either (u_floor = 0, the default of the Python wrapper).  u_floor > 0 is an opt-in
 *       DIAGNOSTIC only (normalised values below it set to 0); no parity test uses it.
 *
 * Layouts (the C-ABI boundary layout): every field is one volume of V = nx*ny*nz
 * values, x fastest.  u: [NL][V] (end labels in node-id order), q: [node][k][V]
 * for non-source nodes in node-id order, k = 0..ndim-1 (x, y, z).
 *
 * Return: 0 on success, -1 - voxel on numerical collapse (a(x) <= 0 or not
 * finite), -1000000000000 on bad arguments.
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define BAD_ARGS (-1000000000000LL)

static int g_threads = 1;

/* Threads for the whole-field passes (1 = the plain single-threaded oracle); results do not depend on it. */
void oracle_set_threads(int n) { g_threads = n < 1 ? 1 : n; }

#define PFOR _Pragma("omp parallel for schedule(static) num_threads(g_threads)")

typedef struct {
    int ndim;
    int64_t nx, ny, nz;
} odims;

/* -1 - (first voxel with a(x) <= 0 or not finite), or 0: a serial scan, so the reported
 * voxel does not depend on the thread count */
static int64_t first_bad(const double *a, int64_t n) {
    for (int64_t i = 0; i < n; ++i)
        if (!(a[i] > 0.0) || !isfinite(a[i])) return -1 - i;
    return 0;
}

static int64_t vol(const odims *d) { return d->nx * d->ny * d->nz; }

static int64_t axis_len(const odims *d, int k) { return k == 0 ? d->nx : (k == 1 ? d->ny : d->nz); }
static int64_t axis_stride(const odims *d, int k) { return k == 0 ? 1 : (k == 1 ? d->nx : d->nx * d->ny); }
static int64_t axis_coord(const odims *d, int64_t i, int k) {
    if (k == 0) return i % d->nx;
    if (k == 1) return (i / d->nx) % d->ny;
    return i / (d->nx * d->ny);
}

/* (nabla f)^k(x) = f(x+e_k) - f(x), 0 at the last index along k (reading R4). */
static void grad_axis(const odims *d, const double *f, int k, double *g) {
    const int64_t n = vol(d), s = axis_stride(d, k), len = axis_len(d, k);
    PFOR
    for (int64_t i = 0; i < n; ++i)
        g[i] = (axis_coord(d, i, k) < len - 1) ? f[i + s] - f[i] : 0.0;
}

/* div q (x) = sum_k q^k(x) - q^k(x-e_k), with q^k(-1) = 0 (reading R4). */
static void divergence(const odims *d, const double *q /* [ndim][V] */, double *out) {
    const int64_t n = vol(d);
    PFOR
    for (int64_t i = 0; i < n; ++i) out[i] = 0.0;
    for (int k = 0; k < d->ndim; ++k) {
        const double *qk = q + (int64_t)k * n;
        const int64_t s = axis_stride(d, k);
        PFOR
        for (int64_t i = 0; i < n; ++i)
            out[i] += qk[i] - (axis_coord(d, i, k) > 0 ? qk[i - s] : 0.0);
    }
}

/* Proj_{|q(x)| <= S(x)} (readings R5, R14). */
static void project(const odims *d, double *q /* [ndim][V] */, const double *S, int cap) {
    const int64_t n = vol(d);
    PFOR
    for (int64_t i = 0; i < n; ++i) {
        if (cap == 0) {
            double nrm2 = 0.0;
            for (int k = 0; k < d->ndim; ++k) nrm2 += q[(int64_t)k * n + i] * q[(int64_t)k * n + i];
            double nrm = sqrt(nrm2);
            if (nrm > S[i]) {
                double f = S[i] / nrm;
                for (int k = 0; k < d->ndim; ++k) q[(int64_t)k * n + i] *= f;
            }
        } else {
            for (int k = 0; k < d->ndim; ++k) {
                double *v = &q[(int64_t)k * n + i];
                if (*v > S[i]) *v = S[i];
                if (*v < -S[i]) *v = -S[i];
            }
        }
    }
}

/* q <- Proj(q - c*tau*nabla f)  (the flow step of P:148 / P:298). */
static void flow_step(const odims *d, double *q, const double *f, const double *S, double ctau, int cap,
                      double *tmp) {
    const int64_t n = vol(d);
    for (int k = 0; k < d->ndim; ++k) {
        grad_axis(d, f, k, tmp);
        double *qk = q + (int64_t)k * n;
        PFOR
        for (int64_t i = 0; i < n; ++i) qk[i] = qk[i] - ctau * tmp[i];
    }
    project(d, q, S, cap);
}

static int check_dims(const odims *d) {
    if (d->ndim != 2 && d->ndim != 3) return 0;
    if (d->nx < 1 || d->ny < 1 || d->nz < 1) return 0;
    if (d->ndim == 2 && d->nz != 1) return 0;
    return 1;
}

/*
 * Algorithm 1, `niter` passes of the while-loop body.
 *   line 147: u_L <- u_L exp(-(D_L + div q_L)/c)        [R1: minus m(x)]
 *   line 148: q_L <- Proj(q_L - c tau nabla u_L)        [u_L unnormalized here]
 *   line 149: a   <- sum_L u_L
 *   line 150: u_L <- u_L / a
 * D: [K][V]; S: [K][V] (capacity of each label's flow); u: [K][V]; q: [K][ndim][V].
 */
int64_t oracle_potts(int ndim, int64_t nx, int64_t ny, int64_t nz, int K, const double *D, const double *S,
                     double *u, double *q, double c, double tau, int shift, int cap, int niter, double u_floor) {
    odims d = {ndim, nx, ny, nz};
    if (!check_dims(&d) || K < 2 || !(c > 0) || !(tau > 0)) return BAD_ARGS;
    const int64_t n = vol(&d);
    double *arg = (double *)malloc(sizeof(double) * n * K);   /* D_L + div q_L */
    double *m = (double *)malloc(sizeof(double) * n);
    double *a = (double *)malloc(sizeof(double) * n);
    double *tmp = (double *)malloc(sizeof(double) * n);
    int64_t status = 0;
    for (int it = 0; it < niter && status == 0; ++it) {
        /* line 147 */
        for (int L = 0; L < K; ++L) {
            divergence(&d, q + (int64_t)L * ndim * n, arg + (int64_t)L * n);
            PFOR
            for (int64_t i = 0; i < n; ++i) arg[(int64_t)L * n + i] = D[(int64_t)L * n + i] + arg[(int64_t)L * n + i];
        }
        PFOR
        for (int64_t i = 0; i < n; ++i) {
            double mm = arg[i];
            for (int L = 1; L < K; ++L) mm = fmin(mm, arg[(int64_t)L * n + i]);
            m[i] = (shift == 0) ? mm : 0.0;
        }
        for (int L = 0; L < K; ++L)
            PFOR
            for (int64_t i = 0; i < n; ++i)
                u[(int64_t)L * n + i] = u[(int64_t)L * n + i] * exp(-(arg[(int64_t)L * n + i] - m[i]) / c);
        /* line 148 */
        for (int L = 0; L < K; ++L)
            flow_step(&d, q + (int64_t)L * ndim * n, u + (int64_t)L * n, S + (int64_t)L * n, c * tau, cap, tmp);
        /* line 149 */
        PFOR
        for (int64_t i = 0; i < n; ++i) {
            a[i] = 0.0;
            for (int L = 0; L < K; ++L) a[i] += u[(int64_t)L * n + i];
        }
        status = first_bad(a, n);
        /* line 150 */
        if (status == 0)
            for (int L = 0; L < K; ++L)
                PFOR
                for (int64_t i = 0; i < n; ++i) {
                    u[(int64_t)L * n + i] = u[(int64_t)L * n + i] / a[i];
                    if (u[(int64_t)L * n + i] < u_floor) u[(int64_t)L * n + i] = 0.0; /* R18 */
                }
    }
    free(arg); free(m); free(a); free(tmp);
    return status;
}

/* ---------------------------------------------------------------------------
 * Label graph helpers for Algorithm 2: children / parents lists, end labels
 * L = {L : L.C = empty} and the top-down order O by Kahn's
 * algorithm with lowest-node-id tie-break.
 * ------------------------------------------------------------------------- */
typedef struct {
    int nn, ne;
    const int *par, *chi;
    const double *w;
    int order[256];     /* O: starts with S */
    int is_leaf[256];
    int leaf_slot[256];
    int nleaf;
} ograph;

static int graph_setup(ograph *g, int nn, int ne, const int *par, const int *chi, const double *w) {
    if (nn < 2 || nn > 256 || ne < 1) return 0;
    g->nn = nn; g->ne = ne; g->par = par; g->chi = chi; g->w = w;
    int indeg[256] = {0}, placed[256] = {0}, nchild[256] = {0};
    for (int e = 0; e < ne; ++e) {
        if (par[e] < 0 || par[e] >= nn || chi[e] < 0 || chi[e] >= nn) return 0;
        indeg[chi[e]]++;
        nchild[par[e]]++;
    }
    if (indeg[0] != 0) return 0;
    for (int k = 0; k < nn; ++k) {
        int pick = -1;
        for (int v = 0; v < nn; ++v)
            if (!placed[v] && indeg[v] == 0) { pick = v; break; }
        if (pick < 0) return 0; /* cycle */
        placed[pick] = 1;
        g->order[k] = pick;
        for (int e = 0; e < ne; ++e)
            if (par[e] == pick) indeg[chi[e]]--;
    }
    if (g->order[0] != 0) return 0;
    g->nleaf = 0;
    for (int v = 0; v < nn; ++v) {
        g->is_leaf[v] = (v != 0 && nchild[v] == 0);
        g->leaf_slot[v] = g->is_leaf[v] ? g->nleaf++ : -1;
    }
    return 1;
}

/*
 * Algorithm 2, `niter` passes of the while-loop body.
 * D: [NL][V] (end labels in node-id order); S: [nn][V] (row 0 unused);
 * u: [NL][V]; q: [nn-1][ndim][V] for nodes 1..nn-1.
 */
int64_t oracle_dag(int ndim, int64_t nx, int64_t ny, int64_t nz, int nn, int ne, const int *par, const int *chi,
                   const double *w, const double *D, const double *S, double *u, double *q, double c, double tau,
                   int shift, int cap, int niter, double u_floor) {
    odims d = {ndim, nx, ny, nz};
    ograph g;
    if (!check_dims(&d) || !graph_setup(&g, nn, ne, par, chi, w) || g.nleaf < 2 || !(c > 0) || !(tau > 0))
        return BAD_ARGS;
    const int64_t n = vol(&d);
    double *dd = (double *)calloc((size_t)n * nn, sizeof(double)); /* d_L, row per node */
    double *m = (double *)malloc(sizeof(double) * n);
    double *a = (double *)malloc(sizeof(double) * n);
    double *tmp = (double *)malloc(sizeof(double) * n);
#define DROW(v) (dd + (int64_t)(v) * n)
#define QOF(v) (q + (int64_t)((v) - 1) * ndim * n)
#define UOF(v) (u + (int64_t)g.leaf_slot[v] * n)
#define DOF(v) (D + (int64_t)g.leaf_slot[v] * n)
#define SOF(v) (S + (int64_t)(v) * n)
    int64_t status = 0;
    for (int it = 0; it < niter && status == 0; ++it) {
        /* P:282  forall L: d_L <- div q_L   (d_S = 0, S has no flow) */
        PFOR
        for (int64_t i = 0; i < n; ++i) DROW(0)[i] = 0.0;
        for (int v = 1; v < nn; ++v) divergence(&d, QOF(v), DROW(v));
        /* P:283  forall L in end labels: d_L <- d_L + D_L */
        for (int v = 1; v < nn; ++v)
            if (g.is_leaf[v])
                PFOR
                for (int64_t i = 0; i < n; ++i) DROW(v)[i] = DROW(v)[i] + DOF(v)[i];
        /* P:284-288  for L in O\{S}: for L' in L.C: d_L' <- d_L' + w_(L,L') d_L */
        for (int k = 1; k < nn; ++k) {
            int L = g.order[k];
            for (int e = 0; e < ne; ++e)
                if (par[e] == L)
                    PFOR
                    for (int64_t i = 0; i < n; ++i) DROW(chi[e])[i] = DROW(chi[e])[i] + w[e] * DROW(L)[i];
        }
        /* P:290  forall L in end labels: u_L <- u_L exp(-d_L / c)   [R1: minus m(x)] */
        PFOR
        for (int64_t i = 0; i < n; ++i) {
            double mm = INFINITY;
            for (int v = 1; v < nn; ++v)
                if (g.is_leaf[v]) mm = fmin(mm, DROW(v)[i]);
            m[i] = (shift == 0) ? mm : 0.0;
        }
        for (int v = 1; v < nn; ++v)
            if (g.is_leaf[v])
                PFOR
                for (int64_t i = 0; i < n; ++i) UOF(v)[i] = UOF(v)[i] * exp(-(DROW(v)[i] - m[i]) / c);
        /* P:291  forall L in end labels: d_L <- u_L */
        for (int v = 1; v < nn; ++v)
            if (g.is_leaf[v]) memcpy(DROW(v), UOF(v), sizeof(double) * n);
        /* P:292  a <- sum over end labels of u_L */
        PFOR
        for (int64_t i = 0; i < n; ++i) {
            a[i] = 0.0;
            for (int v = 1; v < nn; ++v)
                if (g.is_leaf[v]) a[i] += UOF(v)[i];
        }
        status = first_bad(a, n);
        if (status != 0) break;
        /* P:293  u_L <- u_L / a */
        for (int v = 1; v < nn; ++v)
            if (g.is_leaf[v])
                PFOR
                for (int64_t i = 0; i < n; ++i) {
                    UOF(v)[i] = UOF(v)[i] / a[i];
                    if (UOF(v)[i] < u_floor) UOF(v)[i] = 0.0; /* R18 */
                }
        /* P:295  forall L not in end labels: d_L <- 0 */
        for (int v = 0; v < nn; ++v)
            if (!g.is_leaf[v])
                PFOR
                for (int64_t i = 0; i < n; ++i) DROW(v)[i] = 0.0;
        /* P:296-302  for L in O^-1\{S}: q_L <- Proj(q_L - c tau nabla d_L);
                      for L' in L.P\{S}: d_L' <- d_L' + w_(L',L) d_L */
        for (int k = nn - 1; k >= 1; --k) {
            int L = g.order[k];
            flow_step(&d, QOF(L), DROW(L), SOF(L), c * tau, cap, tmp);
            for (int e = 0; e < ne; ++e)
                if (chi[e] == L && par[e] != 0)
                    PFOR
                    for (int64_t i = 0; i < n; ++i) DROW(par[e])[i] = DROW(par[e])[i] + w[e] * DROW(L)[i];
        }
    }
#undef DROW
#undef QOF
#undef UOF
#undef DOF
#undef SOF
    free(dd); free(m); free(a); free(tmp);
    return status;
}

/* Topological order O (Kahn, lowest-id tie-break) -- exported for the pins. */
int oracle_topo_order(int nn, int ne, const int *par, const int *chi, const double *w, int *order_out) {
    ograph g;
    if (!graph_setup(&g, nn, ne, par, chi, w)) return 0;
    for (int k = 0; k < nn; ++k) order_out[k] = g.order[k];
    return 1;
}

/* Exported operator entry points (for the operator pins in tests/test_oracle_pins.py). */
int oracle_grad(int ndim, int64_t nx, int64_t ny, int64_t nz, const double *f, int k, double *g) {
    odims d = {ndim, nx, ny, nz};
    if (!check_dims(&d) || k < 0 || k >= ndim) return 0;
    grad_axis(&d, f, k, g);
    return 1;
}

int oracle_div(int ndim, int64_t nx, int64_t ny, int64_t nz, const double *q, double *out) {
    odims d = {ndim, nx, ny, nz};
    if (!check_dims(&d)) return 0;
    divergence(&d, q, out);
    return 1;
}

int oracle_project(int ndim, int64_t nx, int64_t ny, int64_t nz, double *q, const double *S, int cap) {
    odims d = {ndim, nx, ny, nz};
    if (!check_dims(&d)) return 0;
    project(&d, q, S, cap);
    return 1;
}

/*
 * Algorithm 3: continuous Ishikawa model with N levels and N+1 labels L_0..L_N,
 * `niter` passes of the while-loop body, in the listing's order:
 *   P:318  d_0 <- 0
 *   P:319  for i = 1..N: d_i <- d_{i-1} + div q_i                 (prefix of the level flows)
 *   P:322  forall i: d_i <- d_i + D_i
 *   P:324  forall i: u_i <- u_i exp(-d_i/c)                        [R1: minus m(x) = min_i d_i]
 *   P:325  forall i: d_i <- u_i                                    (unnormalised masses)
 *   P:326  a <- sum_i u_i
 *   P:327  forall i: u_i <- u_i / a                                [R18 floor]
 *   P:329  for i = N-1 .. 1: d_i <- d_i + d_{i+1}                  (reading of the stray prime on
 *                                                                   d_{L_{i+1}}': the value just
 *                                                                   accumulated, i.e. a suffix sum)
 *   P:332  for i = 1..N: q_i <- Proj(q_i - c tau nabla d_i)
 * D: [N+1][V]; S: [N][V] (capacity of level flow q_i, i = 1..N); u: [N+1][V]; q: [N][ndim][V].
 */
int64_t oracle_ishikawa(int ndim, int64_t nx, int64_t ny, int64_t nz, int N, const double *D, const double *S,
                        double *u, double *q, double c, double tau, int shift, int cap, int niter, double u_floor) {
    odims d = {ndim, nx, ny, nz};
    if (!check_dims(&d) || N < 1 || !(c > 0) || !(tau > 0)) return BAD_ARGS;
    const int64_t n = vol(&d);
    const int NL = N + 1;
    double *dd = (double *)malloc(sizeof(double) * n * NL);
    double *m = (double *)malloc(sizeof(double) * n);
    double *a = (double *)malloc(sizeof(double) * n);
    double *tmp = (double *)malloc(sizeof(double) * n);
#define DI(i) (dd + (int64_t)(i) * n)
#define UI(i) (u + (int64_t)(i) * n)
#define QI(i) (q + (int64_t)((i) - 1) * ndim * n)
    int64_t status = 0;
    for (int it = 0; it < niter && status == 0; ++it) {
        PFOR
        for (int64_t x = 0; x < n; ++x) DI(0)[x] = 0.0;
        for (int i = 1; i <= N; ++i) {
            divergence(&d, QI(i), tmp);
            PFOR
            for (int64_t x = 0; x < n; ++x) DI(i)[x] = DI(i - 1)[x] + tmp[x];
        }
        for (int i = 0; i <= N; ++i)
            PFOR
            for (int64_t x = 0; x < n; ++x) DI(i)[x] = DI(i)[x] + D[(int64_t)i * n + x];
        PFOR
        for (int64_t x = 0; x < n; ++x) {
            double mm = DI(0)[x];
            for (int i = 1; i <= N; ++i) mm = fmin(mm, DI(i)[x]);
            m[x] = (shift == 0) ? mm : 0.0;
        }
        for (int i = 0; i <= N; ++i)
            PFOR
            for (int64_t x = 0; x < n; ++x) UI(i)[x] = UI(i)[x] * exp(-(DI(i)[x] - m[x]) / c);
        for (int i = 0; i <= N; ++i) memcpy(DI(i), UI(i), sizeof(double) * n);
        PFOR
        for (int64_t x = 0; x < n; ++x) {
            a[x] = 0.0;
            for (int i = 0; i <= N; ++i) a[x] += UI(i)[x];
        }
        status = first_bad(a, n);
        if (status != 0) break;
        for (int i = 0; i <= N; ++i)
            PFOR
            for (int64_t x = 0; x < n; ++x) {
                UI(i)[x] = UI(i)[x] / a[x];
                if (UI(i)[x] < u_floor) UI(i)[x] = 0.0;
            }
        for (int i = N - 1; i >= 1; --i)
            PFOR
            for (int64_t x = 0; x < n; ++x) DI(i)[x] = DI(i)[x] + DI(i + 1)[x];
        for (int i = 1; i <= N; ++i)
            flow_step(&d, QI(i), DI(i), S + (int64_t)(i - 1) * n, c * tau, cap, tmp);
    }
#undef DI
#undef UI
#undef QI
    free(dd); free(m); free(a); free(tmp);
    return status;
}
