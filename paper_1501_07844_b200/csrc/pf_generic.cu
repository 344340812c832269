// pf_generic.cu -- the pseudo-flow iteration (Alg. 2) for ANY label DAG up to kWideNodes = 31
// non-source nodes and 16 end labels: the graphs the compiled kernel set (pf_iter_inst.py: <= 4 internal,
// <= 16 non-source nodes) does not cover (SURVEY 8.6 limits).  Same per-voxel arithmetic as the fused kernels
// (pf_math.cuh: the same divergence, excess order, label update with the same summation grouping, bottom-up
// masses, flow step and projection), with the graph as dense runtime weights (GraphWide, kernel parameters:
// constant-bank operands) and two HBM passes per iteration instead of one fused pass:
//   pass A (pf_generic_masses): div q_v, d_L += D_L, top-down pushes, label update (u' written), bottom-up
//           masses M_v -> scratch buffer M [z][v][y][pitch];
//   pass B (pf_generic_flows):  q'_v = Proj(q_v - c tau nabla M_v) from M at x, x+e_x, x+e_y, x+e_z.
// One thread per voxel; whole volumes (no z-slab decomposition).  Throughput is not the point here (the configs
// all run on the fused kernels); generality is.
#include <array>
#include <utility>

#include "pf_internal.h"

namespace pf {

struct GenericArgs {
    const float *u_in;   // log2 u, plane 0
    float *u_out;
    const float *q_in;   // plane 0
    float *q_out;
    const void *D;       // fp32 or bf16
    int d_bf16;
    const float *S;      // null, shared field [z][y][pitch], or per-node fields [z][v][y][pitch]
    float *M;            // masses scratch [z][v][y][pitch]
    int nx, ny, nzl, pitch, nzg;
    int NI, NL, NV;
    int s_kind;          // 0 scalar per node, 1 shared field (x s[v]), 2 field per node
    int cap, shift, check;
    float inv_c, ctau;
    unsigned int *resid_bits;
    unsigned long long *err_voxel;
    GraphWide g;
};

constexpr int kGL = 16;   // end labels

// label_update (pf_math.cuh) with a runtime label count: the same operations and summation grouping for every NL
// (halves of (quarter + quarter) for NL >= kHalfSplitNL, else four quarters), so a graph shape that both paths
// support rounds identically.
__device__ __forceinline__ float label_update_rt(const float *dl, const float *lold, float *ut, float *lnew, int NL,
                                                 int shift, float k2) {
    float r[kGL], e[kGL];
    if (NL >= kHalfSplitNL) {   // halves [0, H) and [H, NL), each (first N/2) + (rest) -- label_half
        const int H = NL / 2, N1 = NL - H;
        float m0 = 0.f, m1 = 0.f;
        if (shift == 0) {   // min over the half (fminf is exact: the order does not matter)
            m0 = FLT_MAX;
            m1 = FLT_MAX;
#pragma unroll
            for (int l = 0; l < kGL; ++l) {
                if (l < H) m0 = fminf(m0, dl[l]);
                else if (l < NL) m1 = fminf(m1, dl[l]);
            }
        }
        float T0 = -FLT_MAX, T1 = -FLT_MAX;
#pragma unroll
        for (int l = 0; l < kGL; ++l)
            if (l < NL) {
                r[l] = fmaf((l < H ? m0 : m1) - dl[l], k2, lold[l]);
                if (l < H) T0 = fmaxf(T0, r[l]);
                else T1 = fmaxf(T1, r[l]);
            }
        float sa0 = 0.f, sb0 = 0.f, sa1 = 0.f, sb1 = 0.f;
#pragma unroll
        for (int l = 0; l < kGL; ++l)
            if (l < NL) {
                r[l] = r[l] - (l < H ? T0 : T1);
                e[l] = ex2_approx(r[l]);
                if (l < H) {
                    if (l < H / 2) sa0 += e[l];
                    else sb0 += e[l];
                } else {
                    if (l - H < N1 / 2) sa1 += e[l];
                    else sb1 += e[l];
                }
            }
        const float sh0 = sa0 + sb0, sh1 = sa1 + sb1;
        float c0, g0, c1, g1;
        const float s = label_halves_combine(m0, T0, sh0, m1, T1, sh1, 0, shift, k2, c0, g0);
        label_halves_combine(m0, T0, sh0, m1, T1, sh1, 1, shift, k2, c1, g1);
#pragma unroll
        for (int l = 0; l < kGL; ++l)
            if (l < NL) {
                lnew[l] = r[l] + (l < H ? c0 : c1);
                ut[l] = e[l] * (l < H ? g0 : g1);
            }
        return s;
    }
    const int H = NL / 2, Q1 = H / 2, Q3 = H + (NL - H) / 2;
    float m = 0.f;
    if (shift == 0) {
        m = dl[0];
#pragma unroll
        for (int l = 1; l < kGL; ++l)
            if (l < NL) m = fminf(m, dl[l]);
    }
    float T = -FLT_MAX;
#pragma unroll
    for (int l = 0; l < kGL; ++l)
        if (l < NL) {
            r[l] = fmaf(m - dl[l], k2, lold[l]);
            T = fmaxf(T, r[l]);
        }
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
    for (int l = 0; l < kGL; ++l)
        if (l < NL) {
            r[l] = r[l] - T;
            e[l] = ex2_approx(r[l]);
            if (l < Q1) s0 += e[l];
            else if (l < H) s1 += e[l];
            else if (l < Q3) s2 += e[l];
            else s3 += e[l];
        }
    const float s = (s0 + s1) + (s2 + s3);
    const float ls = lg2_approx(s), g = ex2_approx(T);
#pragma unroll
    for (int l = 0; l < kGL; ++l)
        if (l < NL) {
            lnew[l] = r[l] - ls;
            ut[l] = e[l] * g;
        }
    return s;
}

// pass A: rows a1-a4 (+ a8 residual) of one voxel.  NI (internal positions) is a template parameter so every
// array index is a compile-time constant (registers, no local memory); the end-label count is a runtime bound.
template <int NI>
__global__ void __launch_bounds__(256) pf_generic_masses(const GenericArgs a) {
    const int x = blockIdx.x * 32 + threadIdx.x, y = blockIdx.y * 8 + threadIdx.y, z = blockIdx.z;
    float resid = 0.f;
    if (x < a.nx && y < a.ny) {
        const int NL = a.NL, NV = NI + a.NL;
        const int64_t P = (int64_t)a.pitch * a.ny, pix = (int64_t)y * a.pitch + x;
        const int64_t qps = (int64_t)3 * NV * P, ups = (int64_t)NL * P;
        const float *qb = a.q_in + z * qps + pix;
        float d[kWideNodes];   // div q_v, then the excesses d_v
#pragma unroll
        for (int v = 0; v < kWideNodes; ++v)
            if (v < NV) {
                const float qx = qb[v * P], qxm = x > 0 ? qb[v * P - 1] : 0.f;
                const float qy = qb[(NV + v) * P], qym = y > 0 ? qb[(NV + v) * P - a.pitch] : 0.f;
                const float qz = qb[(2 * NV + v) * P], qzm = z > 0 ? qb[(2 * NV + v) * P - qps] : 0.f;
                d[v] = ((qx - qxm) + (qy - qym)) + (qz - qzm);
            }
        float lold[kGL], dl[kGL];
#pragma unroll
        for (int l = 0; l < kGL; ++l)
            if (l < NL) lold[l] = a.u_in[z * ups + l * P + pix];
        // d_L <- d_L + D_L, then the top-down pushes along O \ {S}, positions in topological order
#pragma unroll
        for (int v = 0; v < kWideNodes; ++v)
            if (v >= NI && v < NV) d[v] = load_D(a.D, z * ups + (v - NI) * P + pix, a.d_bf16) + d[v];
#pragma unroll
        for (int i = 0; i < kWideNodes; ++i)
            if (i < NI)
#pragma unroll
                for (int j = i + 1; j < kWideNodes; ++j)
                    if (j < NV) d[j] = fmaf(a.g.w[i][j], d[i], d[j]);
#pragma unroll
        for (int l = 0; l < kGL; ++l)
            if (l < NL && NI + l < kWideNodes) dl[l] = d[NI + l];
        // label update (Eq. 15; readings R1, R18) on the log2 state
        float ut[kGL], un[kGL];
        const float k2 = kLog2e * a.inv_c;
        const float sum = label_update_rt(dl, lold, ut, un, NL, a.shift, k2);
        if (label_sum_bad(sum)) atomicMin(a.err_voxel, ((unsigned long long)z * a.ny + y) * a.nx + x);
#pragma unroll
        for (int l = 0; l < kGL; ++l)
            if (l < NL) {
                st_stream(a.u_out + z * ups + l * P + pix, un[l]);
                if (a.check) resid = fmaxf(resid, fabsf(u_of_log2(un[l]) - u_of_log2(lold[l])));
            }
        // masses: M_L = u~_L, bottom-up pushes along O^-1; d is reused for M
#pragma unroll
        for (int l = 0; l < kGL; ++l)
            if (l < NL && NI + l < kWideNodes) d[NI + l] = ut[l];
#pragma unroll
        for (int i = kWideNodes - 1; i >= 0; --i)
            if (i < NI) {
                float acc = 0.f;
#pragma unroll
                for (int j = i + 1; j < kWideNodes; ++j)
                    if (j < NV) acc = fmaf(a.g.w[i][j], d[j], acc);
                d[i] = acc;
            }
        float *Mz = a.M + (int64_t)z * NV * P + pix;
#pragma unroll
        for (int v = 0; v < kWideNodes; ++v)
            if (v < NV) Mz[v * P] = d[v];
    }
    if (a.check) {
        const int lane = (threadIdx.y * 32 + threadIdx.x) & 31;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) resid = fmaxf(resid, __shfl_xor_sync(0xffffffffu, resid, o));
        if (lane == 0 && resid > 0.f) atomicMax(a.resid_bits, __float_as_uint(resid));
    }
}

// pass B: rows a5-a7 of one voxel -- the flow step and projection of every node (Eq. 16; R5, R14)
__global__ void __launch_bounds__(256) pf_generic_flows(const GenericArgs a) {
    const int x = blockIdx.x * 32 + threadIdx.x, y = blockIdx.y * 8 + threadIdx.y, z = blockIdx.z;
    if (x >= a.nx || y >= a.ny) return;
    const int NV = a.NV;
    const int64_t P = (int64_t)a.pitch * a.ny, pix = (int64_t)y * a.pitch + x;
    const int64_t qps = (int64_t)3 * NV * P, mps = (int64_t)NV * P;
    const float cx = x < a.nx - 1 ? a.ctau : 0.f, cy = y < a.ny - 1 ? a.ctau : 0.f;
    const bool has_z = z < a.nzl - 1;
    const float cz = has_z ? a.ctau : 0.f;
    const float *Mz = a.M + z * mps + pix;
    const float *qb = a.q_in + z * qps + pix;
    float *qo = a.q_out + z * qps + pix;
    const float sb = a.s_kind == 1 ? a.S[z * P + pix] : 1.f;
#pragma unroll 1
    for (int v = 0; v < NV; ++v) {
        const float mc = Mz[v * P];
        const float gx = (x < a.nx - 1 ? Mz[v * P + 1] : 0.f) - mc;
        const float gy = (y < a.ny - 1 ? Mz[v * P + a.pitch] : 0.f) - mc;
        const float gz = (has_z ? Mz[v * P + mps] : 0.f) - mc;
        float hx = qb[v * P], hy = qb[(NV + v) * P], hz = qb[(2 * NV + v) * P];
        const float sv = a.s_kind == 2 ? a.S[(z * NV + v) * P + pix] : sb * a.g.s[v];
        if (a.cap == 0) flow_step3<0>(cx, cy, cz, gx, gy, gz, sv, hx, hy, hz);
        else flow_step3<1>(cx, cy, cz, gx, gy, gz, sv, hx, hy, hz);
        st_stream(qo + v * P, hx);
        st_stream(qo + (NV + v) * P, hy);
        st_stream(qo + (2 * NV + v) * P, hz);
    }
}

template <int NI>
void launch_masses(const GenericArgs &a, dim3 grid, dim3 block, cudaStream_t st) {
    pf_generic_masses<NI><<<grid, block, 0, st>>>(a);
}
using MassesLaunch = void (*)(const GenericArgs &, dim3, dim3, cudaStream_t);
template <int... I>
constexpr auto masses_table(std::integer_sequence<int, I...>) {
    return std::array<MassesLaunch, sizeof...(I)>{&launch_masses<I>...};
}
const auto generic_masses_table = masses_table(std::make_integer_sequence<int, kWideNodes>{});

cudaError_t launch_generic_iteration(const pf_solver *s, int check) {
    GenericArgs a;
    memset(&a, 0, sizeof(a));
    a.u_in = s->u[s->cur];
    a.u_out = s->u[1 - s->cur];
    a.q_in = s->q[s->cur];
    a.q_out = s->q[1 - s->cur];
    a.D = s->Dptr();
    a.d_bf16 = s->D16 ? 1 : 0;
    a.S = s->S_alloc;
    a.M = s->M_alloc;
    a.nx = (int)s->nx;
    a.ny = (int)s->ny;
    a.nzl = (int)s->nzl;
    a.pitch = (int)s->pitch;
    a.nzg = (int)s->nz;
    a.NI = s->gc.NI;
    a.NL = s->gc.NL;
    a.NV = s->gc.NV;
    a.s_kind = s->s_kind == PF_S_SCALED_FIELD ? 1 : s->s_kind;
    a.cap = s->cfg.cap;
    a.shift = s->cfg.shift;
    a.check = check;
    a.inv_c = 1.0f / s->cfg.c;
    a.ctau = s->cfg.c * s->cfg.tau;
    a.resid_bits = s->d_resid;
    a.err_voxel = s->d_err;
    a.g = s->gc.gw;
    const dim3 grid((unsigned)((s->nx + 31) / 32), (unsigned)((s->ny + 7) / 8), (unsigned)s->nzl), block(32, 8);
    generic_masses_table[a.NI](a, grid, block, s->stream);
    pf_generic_flows<<<grid, block, 0, s->stream>>>(a);
    return cudaGetLastError();
}

const void *generic_kernel_func() { return (const void *)&pf_generic_masses<kMaxInternal + 1>; }

}  // namespace pf
