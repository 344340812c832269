// pf_math.cuh -- the per-voxel arithmetic of one pseudo-flow iteration, shared by both data-movement
// variants of the fused kernel (pf_kernels.cuh global-load, pf_staged.cuh TMA-staged) so that the two
// are bitwise identical.  Paper references: PAPER.md P:144-153 (Alg. 1), P:279-305 (Alg. 2).
#pragma once
#include <cfloat>
#include <cstdint>
#include <cstring>

namespace pf {

constexpr float kLog2e = 1.4426950408889634f;

// 2^x on the SFU (MUFU.EX2, max rel. error ~2^-22); subnormal results flush to 0, consistent with the
// u floor below.
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

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
__device__ __forceinline__ void st_stream(float *p, float v) {
    asm volatile("st.global.cs.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

// Label update of one voxel (P:147-150 / P:290-293, Eq. 7 / Eq. 15; reading R1):
//   m = min_L d_L (SHIFT_MIN) or 0;  u~_L = u_L exp(-(d_L - m)/c);  a = sum u~;  u'_L = u~_L / a,
// with u' below the fp32 normal range flushed to 0 (reading R18: u is stored in fp32).
// d[NI..NI+NL) holds the end-label excesses on entry; ut receives u~ (the unnormalised masses).
// Returns a; writes u' to unew.
//
// Summation order: a = (q0 + q1) + (q2 + q3), q_i the sequential sum of the i-th quarter of the labels
// (quarters = halves of halves).  With many labels (NL >= kHalfSplitNL) the two halves are shifted
// separately and rescaled (the "online softmax" identity exp(-(d-m)/c) = exp(-(d-m_h)/c) exp(-(m_h-m)/c)):
//   m_h = min over half h, u~^h_L = u_L exp(-(d_L - m_h)/c), a_h = quarter + quarter,
//   f_h = exp(-(m_h - m)/c), a = a_1 f_1 + a_0 f_0 (one fma), u~_L = u~^h_L f_h,
// which is the arithmetic of the label-split kernels (two warps or two CTAs per voxel row exchange only
// (m_h, a_h), once), so every variant rounds identically.
constexpr int kHalfSplitNL = 10;

__device__ __forceinline__ float halves_sum(float a0, float f0, float a1, float f1) { return fmaf(a1, f1, a0 * f0); }

template <int NI, int NL>
__device__ __forceinline__ float label_update(const float (&d)[NI + NL], const float (&uold)[NL], float (&ut)[NL],
                                              float (&unew)[NL], int shift, float k2 /* log2(e)/c */) {
    constexpr int H = NL / 2, Q1 = H / 2, Q3 = H + (NL - H) / 2;
    float sum;
    if constexpr (NL >= kHalfSplitNL) {
        float m0 = 0.f, m1 = 0.f;
        if (shift == 0) {
            m0 = d[NI];
#pragma unroll
            for (int l = 1; l < H; ++l) m0 = fminf(m0, d[NI + l]);
            m1 = d[NI + H];
#pragma unroll
            for (int l = H + 1; l < NL; ++l) m1 = fminf(m1, d[NI + l]);
        }
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
        for (int l = 0; l < NL; ++l) {
            ut[l] = uold[l] * ex2_approx(((l < H ? m0 : m1) - d[NI + l]) * k2);
            if (l < Q1) s0 += ut[l];
            else if (l < H) s1 += ut[l];
            else if (l < Q3) s2 += ut[l];
            else s3 += ut[l];
        }
        float f0 = 1.f, f1 = 1.f;
        if (shift == 0) {
            const float m = fminf(m0, m1);
            f0 = ex2_approx((m - m0) * k2);
            f1 = ex2_approx((m - m1) * k2);
        }
        sum = halves_sum(s0 + s1, f0, s2 + s3, f1);
#pragma unroll
        for (int l = 0; l < NL; ++l) ut[l] *= (l < H ? f0 : f1);
    } else {
        float m = 0.f;
        if (shift == 0) {
            m = d[NI];
#pragma unroll
            for (int l = 1; l < NL; ++l) m = fminf(m, d[NI + l]);
        }
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
        for (int l = 0; l < NL; ++l) {
            ut[l] = uold[l] * ex2_approx((m - d[NI + l]) * k2);
            if (l < Q1) s0 += ut[l];
            else if (l < H) s1 += ut[l];
            else if (l < Q3) s2 += ut[l];
            else s3 += ut[l];
        }
        sum = (s0 + s1) + (s2 + s3);
    }
    const float inv = __frcp_rn(sum);
#pragma unroll
    for (int l = 0; l < NL; ++l) {
        const float nu = ut[l] * inv;
        unew[l] = nu < FLT_MIN ? 0.f : nu;
    }
    return sum;
}

// Top-down excess pushes along O \ {S}: d_j += w_ij d_i for internal i (positions < NI).
template <int NI, int NV>
__device__ __forceinline__ void push_down(float (&d)[NV], const float (&w)[kMaxInternal][kMaxNodes]) {
#pragma unroll
    for (int i = 0; i < NI; ++i)
#pragma unroll
        for (int j = i + 1; j < NV; ++j) d[j] = fmaf(w[i][j], d[i], d[j]);
}

// Bottom-up masses along O^-1 \ {S}: M_i = sum_j w_ij M_j for internal i.
template <int NI, int NV>
__device__ __forceinline__ void push_up(float (&M)[NV], const float (&w)[kMaxInternal][kMaxNodes]) {
#pragma unroll
    for (int i = NI - 1; i >= 0; --i) {
        float acc = 0.f;
#pragma unroll
        for (int j = i + 1; j < NV; ++j) acc = fmaf(w[i][j], M[j], acc);
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
template <int MODEL, int NI, int NL>
__device__ __forceinline__ void label_excess(const float (&dq)[Model<MODEL, NI, NL>::NF], const float (&Dv)[NL],
                                             float (&dlab)[NI + NL], const float (&w)[kMaxInternal][kMaxNodes]) {
    if constexpr (MODEL == 0) {
#pragma unroll
        for (int v = 0; v < NI + NL; ++v) dlab[v] = dq[v];
#pragma unroll
        for (int l = 0; l < NL; ++l) dlab[NI + l] = Dv[l] + dlab[NI + l];
        push_down<NI, NI + NL>(dlab, w);
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
template <int MODEL, int NI, int NL>
__device__ __forceinline__ void node_masses(const float (&ut)[NL], float (&M)[Model<MODEL, NI, NL>::NF],
                                            const float (&w)[kMaxInternal][kMaxNodes]) {
    if constexpr (MODEL == 0) {
#pragma unroll
        for (int l = 0; l < NL; ++l) M[NI + l] = ut[l];
        push_up<NI, NI + NL>(M, w);
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
template <int CAP>
__device__ __forceinline__ void flow_step3(float cx, float cy, float cz, float gx, float gy, float gz, float sv,
                                           float &hx, float &hy, float &hz) {
    hx = fmaf(-cx, gx, hx);
    hy = fmaf(-cy, gy, hy);
    hz = fmaf(-cz, gz, hz);
    if (CAP == 0) {
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
