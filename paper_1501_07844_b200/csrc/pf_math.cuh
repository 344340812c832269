// pf_math.cuh -- the per-voxel arithmetic of one pseudo-flow iteration, shared by both data-movement
// variants of the fused kernel (pf_kernels.cuh global-load, pf_staged.cuh TMA-staged) so that the two
// are bitwise identical.  Paper references: PAPER.md P:144-153 (Alg. 1), P:279-305 (Alg. 2).
#pragma once
#include <cfloat>
#include <cstdint>
#include <cstring>

#include <cuda_fp16.h>

namespace pf {

constexpr float kLog2e = 1.4426950408889634f;

// 2^x on the SFU (MUFU.EX2, max rel. error ~2^-22).  Results below 2^-126 flush to 0.  It is only applied
// to TRANSIENT values -- the per-label factors e_L <= 1 whose sum s >= 1 absorbs anything below 2^-126, the
// masses u~ and the exported labeling u = 2^lambda -- never to the stored state, which is lambda = log2 u
// (reading R18): no stored label can underflow and die.
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// log2(x) on the SFU (MUFU.LG2); only called on the label-update sum s in [1, 2K] (max abs. error ~2^-22).
__device__ __forceinline__ float lg2_approx(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// The labeling u_L of a stored log2 value (exports, argmax, residual, energies).
__device__ __forceinline__ float u_of_log2(float lam) { return ex2_approx(lam); }

// 1/sqrt(x) on the SFU (MUFU.RSQ).  Only called on x in [1, 3] (the rescaled squared norm below), where
// rsqrtf() would return the same value after a denormal-input guard that can never trigger.
__device__ __forceinline__ float rsqrt_approx(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// bf16 storage of D (pf_config.d_bf16): round-to-nearest-even on upload, exact widening on load.
// (D is finite and >= 0 by validation, so no NaN handling is needed.)
__host__ __device__ __forceinline__ uint16_t f32_to_bf16_rn(float f) {
    uint32_t b;
    memcpy(&b, &f, 4);
    b += 0x7fffu + ((b >> 16) & 1u);
    return (uint16_t)(b >> 16);
}
__device__ __forceinline__ float bf16_to_f32(uint16_t h) { return __uint_as_float((uint32_t)h << 16); }
__device__ __forceinline__ float load_D(const void *D, int64_t i, int bf16) {
    return bf16 ? bf16_to_f32(__ldg(reinterpret_cast<const unsigned short *>(D) + i))
                : __ldg(reinterpret_cast<const float *>(D) + i);
}

// Streaming (evict-first) store: the new state is not re-read in this launch, keep it out of L2's way.
__device__ __forceinline__ void st_stream_h(__half *p, __half v) {
    asm volatile("st.global.cs.b16 [%0], %1;" ::"l"(p), "h"(__half_as_ushort(v)) : "memory");
}

// Stored label state (pf_config.u_half): lambda = log2 u rounded to nearest binary16 once per store; the
// arithmetic stays fp32.  round_state gives the value the next iteration will read back.
__device__ __forceinline__ float round_state_half(float lam) { return __half2float(__float2half_rn(lam)); }

__device__ __forceinline__ void st_stream(float *p, float v) {
    asm volatile("st.global.cs.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

// Label update of one voxel (P:147-150 / P:290-293, Eq. 7 / Eq. 15; reading R1) on the log2 state
// lambda_L = log2 u_L (reading R18):
//   m = min_L d_L (SHIFT_MIN) or 0;   u~_L = u_L exp(-(d_L - m)/c);   a = sum u~;   u'_L = u~_L / a
// evaluated as
//   t_L = lambda_L + (m - d_L) log2(e)/c  (= log2 u~_L),   T = max_L t_L,   r_L = t_L - T,   e_L = 2^r_L in (0, 1],
//   s = sum_L e_L in [1, K],   lambda'_L = r_L - log2 s  (= log2 u'_L),   u~_L = e_L 2^T  (the masses M_L)
// -- the same quantities (a = s 2^T), but the stored state is a logarithm, so no label underflows and dies in
// fp32 (which made fp32 trajectories leave the exact iteration where a label decays below 2^-149 and later
// revives; R18) and a is never formed as a number that could under- or overflow.
// d[NI..NI+NL) holds the end-label excesses on entry; ut receives u~ (the unnormalised masses), lnew lambda'.
// Returns s (>= 1; NaN / not finite flags a numerical collapse).
//
// Summation order: s = (q0 + q1) + (q2 + q3), q_i the sequential sum of the i-th quarter of the labels
// (quarters = halves of halves).  With many labels (NL >= kHalfSplitNL) the two halves h are reduced
// separately -- their own shift m_h, maximum T_h and sum s_h = quarter + quarter -- and combined from the
// three numbers (m_h, T_h, s_h) of each half (label_halves_combine), which is the arithmetic of the
// label-split kernels (two warps or two CTAs per voxel row exchange exactly those three numbers, once), so
// every variant rounds identically.
constexpr int kHalfSplitNL = 10;

__device__ __forceinline__ float halves_sum(float a0, float f0, float a1, float f1) { return fmaf(a1, f1, a0 * f0); }

// One half of the labels (N of them, starting at d / lold): shift m_h, r_L = t_L - T_h, e_L = 2^r_L,
// s_h = (first N/2) + (rest).  Also the whole-label-set step when called with all labels (then m_h = m).
template <int N>
__device__ __forceinline__ void label_half(const float *d, const float *lold, float *r, float *e, int shift, float k2,
                                           float &mh, float &Th, float &sh) {
    mh = 0.f;
    if (shift == 0) {
        mh = d[0];
#pragma unroll
        for (int l = 1; l < N; ++l) mh = fminf(mh, d[l]);
    }
#pragma unroll
    for (int l = 0; l < N; ++l) r[l] = fmaf(mh - d[l], k2, lold[l]);   // t_L
    // (floor -FLT_MAX: a half whose labels are all exactly dead, lambda = -inf, gives e = 0, s_h = 0 and
    // lambda' = -inf instead of -inf - (-inf) = NaN)
    Th = -FLT_MAX;
#pragma unroll
    for (int l = 0; l < N; ++l) Th = fmaxf(Th, r[l]);
    float sa = 0.f, sb = 0.f;
#pragma unroll
    for (int l = 0; l < N; ++l) {
        r[l] = r[l] - Th;
        e[l] = ex2_approx(r[l]);
        if (l < N / 2) sa += e[l];
        else sb += e[l];
    }
    sh = sa + sb;
}

// Combine the two halves' (m_h, T_h, s_h): with the common shift m = min(m_0, m_1) the half maxima are
// G_h = T_h + (m - m_h) log2(e)/c, T = max G_h, s = s_0 2^(G_0 - T) + s_1 2^(G_1 - T).  For half `h` returns
// lambda offset c_h = (G_h - T) - log2 s (lambda'_L = r_L + c_h) and mass scale g_h = 2^G_h (u~_L = e_L g_h);
// the return value is s.
__device__ __forceinline__ float label_halves_combine(float m0, float T0, float s0, float m1, float T1, float s1, int h,
                                                      int shift, float k2, float &ch, float &gh) {
    const float m = shift == 0 ? fminf(m0, m1) : 0.f;
    const float G0 = fmaf(m - m0, k2, T0), G1 = fmaf(m - m1, k2, T1);
    const float T = fmaxf(G0, G1);
    const float s = halves_sum(s0, ex2_approx(G0 - T), s1, ex2_approx(G1 - T));
    const float G = h == 0 ? G0 : G1;
    ch = (G - T) - lg2_approx(s);
    gh = ex2_approx(G);
    return s;
}

template <int NI, int NL>
__device__ __forceinline__ float label_update(const float (&d)[NI + NL], const float (&lold)[NL], float (&ut)[NL],
                                              float (&lnew)[NL], int shift, float k2 /* log2(e)/c */) {
    float r[NL], e[NL];
    if constexpr (NL >= kHalfSplitNL) {
        constexpr int H = NL / 2;
        float m0, T0, s0, m1, T1, s1;
        label_half<H>(d + NI, lold, r, e, shift, k2, m0, T0, s0);
        label_half<NL - H>(d + NI + H, lold + H, r + H, e + H, shift, k2, m1, T1, s1);
        float c0, g0, c1, g1;
        const float s = label_halves_combine(m0, T0, s0, m1, T1, s1, 0, shift, k2, c0, g0);
        label_halves_combine(m0, T0, s0, m1, T1, s1, 1, shift, k2, c1, g1);
#pragma unroll
        for (int l = 0; l < NL; ++l) {
            lnew[l] = r[l] + (l < H ? c0 : c1);
            ut[l] = e[l] * (l < H ? g0 : g1);
        }
        return s;
    } else {
        constexpr int H = NL / 2, Q1 = H / 2, Q3 = H + (NL - H) / 2;
        float m = 0.f;
        if (shift == 0) {
            m = d[NI];
#pragma unroll
            for (int l = 1; l < NL; ++l) m = fminf(m, d[NI + l]);
        }
#pragma unroll
        for (int l = 0; l < NL; ++l) r[l] = fmaf(m - d[NI + l], k2, lold[l]);   // t_L
        float T = -FLT_MAX;   // (as label_half: every label dead gives s = 0, flagged as a collapse)
#pragma unroll
        for (int l = 0; l < NL; ++l) T = fmaxf(T, r[l]);
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
        for (int l = 0; l < NL; ++l) {
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
        for (int l = 0; l < NL; ++l) {
            lnew[l] = r[l] - ls;
            ut[l] = e[l] * g;
        }
        return s;
    }
}

// max |u' - u| over the labels of one voxel (residual, row a8) from the old and new log2 states
template <int N>
__device__ __forceinline__ float resid_log2(const float *lnew, const float *lold, float acc) {
#pragma unroll
    for (int l = 0; l < N; ++l) acc = fmaxf(acc, fabsf(u_of_log2(lnew[l]) - u_of_log2(lold[l])));
    return acc;
}

// numerical collapse of the label update (a(x) <= 0 or not finite): s (>= 1 when sane) is 0,
// infinite or NaN -- e.g. every label of the voxel at lambda = -inf, or a non-finite excess
__device__ __forceinline__ bool label_sum_bad(float s) { return !(s > 0.f) || !(s <= FLT_MAX); }

// Edge mask of a compiled graph (pf_graph.cu): bit i * kMaxNodes + j set iff w[i][j] != 0 (internal position i ->
// position j).  Kernels specialised for a mask emit only the graph's edges (the flat per-level schedule of row
// a10); ~0 = dense rows, any graph.  Skipped terms are fmaf(0, x, y) = y up to the sign of a zero.
constexpr uint64_t kDenseMask = ~0ull;
__host__ __device__ constexpr bool edge_on(uint64_t mask, int i, int j) { return (mask >> (i * 16 + j)) & 1ull; }

// Top-down excess pushes along O \ {S}: d_j += w_ij d_i for internal i (positions < NI).
template <int NI, int NV, uint64_t MASK = kDenseMask>
__device__ __forceinline__ void push_down(float (&d)[NV], const float (&w)[kMaxInternal][kMaxNodes]) {
#pragma unroll
    for (int i = 0; i < NI; ++i)
#pragma unroll
        for (int j = i + 1; j < NV; ++j)
            if (MASK == kDenseMask || edge_on(MASK, i, j)) d[j] = fmaf(w[i][j], d[i], d[j]);
}

// Bottom-up masses along O^-1 \ {S}: M_i = sum_j w_ij M_j for internal i.
template <int NI, int NV, uint64_t MASK = kDenseMask>
__device__ __forceinline__ void push_up(float (&M)[NV], const float (&w)[kMaxInternal][kMaxNodes]) {
#pragma unroll
    for (int i = NI - 1; i >= 0; --i) {
        float acc = 0.f;
#pragma unroll
        for (int j = i + 1; j < NV; ++j)
            if (MASK == kDenseMask || edge_on(MASK, i, j)) acc = fmaf(w[i][j], M[j], acc);
        M[i] = acc;
    }
}

// Label models.  MODEL 0: general DAG (Potts = star, HMF = tree), every non-source node carries a flow,
// positions 0..NI-1 internal (topological order), NI..NI+NL-1 end labels.  MODEL 1: Ishikawa chain
// (Alg. 3): NI = N level nodes carry the flows q_1..q_N, the NL = N+1 ordered labels carry none.
template <int MODEL, int NI, int NL>
struct Model {
    static constexpr int NV = NI + NL;
    static constexpr int NF = MODEL == 1 ? NI : NV;   // nodes with a spatial flow
};

// End-label excesses from the flow divergences dq and data terms Dv into dlab[NI + l].
//   MODEL 0: d_v = div q_v; d_L += D_L; top-down pushes
//   MODEL 1: d_0 = D_0; d_i = (d_{i-1} + div q_i) + D_i (prefix)
template <int MODEL, int NI, int NL, uint64_t MASK = kDenseMask>
__device__ __forceinline__ void label_excess(const float (&dq)[Model<MODEL, NI, NL>::NF], const float (&Dv)[NL],
                                             float (&dlab)[NI + NL], const float (&w)[kMaxInternal][kMaxNodes]) {
    if constexpr (MODEL == 0) {
#pragma unroll
        for (int v = 0; v < NI + NL; ++v) dlab[v] = dq[v];
#pragma unroll
        for (int l = 0; l < NL; ++l) dlab[NI + l] = Dv[l] + dlab[NI + l];
        push_down<NI, NI + NL, MASK>(dlab, w);
    } else {
        float run = 0.f;
        dlab[NI] = Dv[0];
#pragma unroll
        for (int i = 1; i < NL; ++i) {
            run = run + dq[i - 1];
            dlab[NI + i] = run + Dv[i];
        }
    }
}

// Unnormalised masses M of the flow-carrying nodes from the end-label masses ut.
//   MODEL 0: M_L = u~_L; bottom-up pushes
//   MODEL 1: M_N = u~_N; M_i = u~_i + M_{i+1} (suffix)
template <int MODEL, int NI, int NL, uint64_t MASK = kDenseMask>
__device__ __forceinline__ void node_masses(const float (&ut)[NL], float (&M)[Model<MODEL, NI, NL>::NF],
                                            const float (&w)[kMaxInternal][kMaxNodes]) {
    if constexpr (MODEL == 0) {
#pragma unroll
        for (int l = 0; l < NL; ++l) M[NI + l] = ut[l];
        push_up<NI, NI + NL, MASK>(M, w);
    } else {
        M[NI - 1] = ut[NL - 1];
#pragma unroll
        for (int f = NI - 2; f >= 0; --f) M[f] = ut[f + 1] + M[f + 1];
    }
}

// Flow step + capacity projection of one node at one voxel (P:148 / P:298; Eq. 8 / Eq. 16; R5, R14):
//   q^ = q - c tau nabla M;  q' = q^ if |q^| <= S else q^ S/|q^|  (CAP 0, l2)  |  clamp(q^, -S, S) (CAP 1).
// cx, cy, cz: c tau per axis, 0 where nabla_k M is 0 (last index along k) -- the staged kernel folds the
// boundary into the coefficient (q - 0 * g == q for the finite g it passes there).
// SCALED = false (StagedArgs.fastproj): the plain formula, for launches where no square can under- or overflow --
// SHIFT_MIN (masses u~ <= 1, so |q^| stays near S) with scalar capacities all >= 2^-60; there every decision and,
// since the rescale is by an exact power of two (and MUFU.RSQ of a 4^k-scaled argument is the 2^-k-scaled
// result), every value equals the scaled form's.
template <int CAP, bool SCALED = true>
__device__ __forceinline__ void flow_step3(float cx, float cy, float cz, float gx, float gy, float gz, float sv,
                                           float &hx, float &hy, float &hz) {
    hx = fmaf(-cx, gx, hx);
    hy = fmaf(-cy, gy, hy);
    hz = fmaf(-cz, gz, hz);
    if (CAP == 0 && !SCALED) {
        const float n2 = fmaf(hx, hx, fmaf(hy, hy, hz * hz));
        const float f = n2 > sv * sv ? sv * rsqrt_approx(n2) : 1.f;
        hx *= f; hy *= f; hz *= f;
    } else if (CAP == 0) {
        // Norm on a power-of-two rescaled copy (exact scaling), so tiny flows next to tiny capacities
        // (S(x) down to 1e-38 in the configs' edge-weighted S) neither under-flow their squares nor
        // need a slow path; for normal ranges the result is bitwise that of the unscaled formula.
        // (branch-free: m = 0 gives n2 = 0, which never exceeds ss^2, so f = 1 and q^ = 0 is kept)
        const float m = fmaxf(fabsf(hx), fmaxf(fabsf(hy), fabsf(hz)));
        const float sc = __int_as_float(0x7f000000 - (__float_as_int(m) & 0x7f800000));  // ~1/m, a power of 2
        const float sx = hx * sc, sy = hy * sc, sz = hz * sc;
        const float n2 = fmaf(sx, sx, fmaf(sy, sy, sz * sz));
        const float ss = sv * sc;
        const float f = n2 > ss * ss ? ss * rsqrt_approx(n2) : 1.f;  // S / |q^| when projecting
        hx *= f; hy *= f; hz *= f;
    } else {
        hx = fminf(fmaxf(hx, -sv), sv);
        hy = fminf(fmaxf(hy, -sv), sv);
        hz = fminf(fmaxf(hz, -sv), sv);
    }
}

template <int CAP>
__device__ __forceinline__ void flow_step(float ctau, float gx, float gy, float gz, float sv, float &hx, float &hy,
                                          float &hz) {
    flow_step3<CAP>(ctau, ctau, ctau, gx, gy, gz, sv, hx, hy, hz);
}

}  // namespace pf
