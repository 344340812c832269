// pf_aux.cu -- auxiliary sm_100a kernels: state init (row a0), thresholded labeling
// (row a9), primal / dual energies (row a8 diagnostics), capacity validation.
#include <cfloat>
#include <cstdint>

#include "pf_aux.cuh"

namespace pf {

__global__ void fill_kernel(float *p, int64_t n, float v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

// The stored label state at element idx: ufmt 0 = u itself in fp32 (explicit-flow ALM arm), 1 = lambda = log2 u
// in fp32 (pseudo-flow, reading R18), 2 = lambda in binary16 (pf_config.u_half).  raw: lambda itself, else u.
__device__ __forceinline__ float state_at(const void *u, int64_t idx, int ufmt) {
    return ufmt == 2 ? __half2float(reinterpret_cast<const __half *>(u)[idx]) : reinterpret_cast<const float *>(u)[idx];
}
__device__ __forceinline__ float u_at(const void *u, int64_t idx, int ufmt) {
    const float v = state_at(u, idx, ufmt);
    return ufmt ? u_of_log2(v) : v;
}

__global__ void fill_half_kernel(__half *p, int64_t n, float v) {
    const __half h = __float2half_rn(v);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = h;
}

// argmax over end labels, lowest label id wins ties ("thresholded"); compared on the same
// u values pf_get_labeling exports.
__global__ void argmax_kernel(const void *__restrict__ u, uint8_t *__restrict__ out, int NL, int nx, int ny,
                              int pitch, int64_t nz, int ufmt) {
    const int64_t V = (int64_t)nx * ny * nz, P = (int64_t)pitch * ny;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t z = i / ((int64_t)nx * ny);
        const int r = (int)(i - z * (int64_t)nx * ny);
        const int y = r / nx, x = r - y * nx;
        const int64_t b = z * NL * P + (int64_t)y * pitch + x;
        float best = u_at(u, b, ufmt);
        int arg = 0;
        for (int l = 1; l < NL; ++l) {
            const float v = u_at(u, b + l * P, ufmt);
            if (v > best) { best = v; arg = l; }
        }
        out[i] = (uint8_t)arg;
    }
}

// Labeling of any node: u_v(x) = sum_B W_(v,B) u_B(x) over the end labels B (path weights P:199-209),
// written densely as [z][y][x] (x fastest).
__global__ void node_labeling_kernel(const void *__restrict__ u, float *__restrict__ out, NodeWeights w, int NL,
                                     int nx, int ny, int pitch, int64_t nz, int ufmt) {
    const int64_t V = (int64_t)nx * ny * nz, P = (int64_t)pitch * ny;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t z = i / ((int64_t)nx * ny);
        const int r = (int)(i - z * (int64_t)nx * ny);
        const int y = r / nx, x = r - y * nx;
        const int64_t b = z * NL * P + (int64_t)y * pitch + x;
        float acc = 0.f;
        for (int l = 0; l < NL; ++l)
            if (w.W[l] != 0.f) acc = fmaf(w.W[l], u_at(u, b + l * P, ufmt), acc);
        out[i] = acc;
    }
}

__global__ void min_kernel(const float *__restrict__ p, int64_t n, unsigned int *out_bits_neg) {
    // records whether any value is negative or NaN (out = 1)
    bool bad = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float v = p[i];
        if (!(v >= 0.f) || !(v <= FLT_MAX)) bad = true;
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(out_bits_neg, 1u);
}

// ---------------------------------------------------------------------------
// Energies.  One thread per owned voxel; fp64 per-block partials reduced in a
// fixed order by energy_finish_kernel (deterministic).
// ---------------------------------------------------------------------------
struct NodeVals {
    float v[kMaxNodes];
};

__device__ __forceinline__ void labels_at(const EnergyArgs &a, int64_t ub, int64_t P, float *out) {
    // u_v for every position: end labels read, internal by bottom-up sums (Eq. 9);
    // Ishikawa chain: u_{N_i} = sum_{j >= i} u_{L_j}
    const int NV = a.NV, NI = a.NI;
    for (int l = 0; l < a.NL; ++l) out[NI + l] = u_at(a.u, ub + l * P, a.ufmt);
    if (a.model == 1) {
        double acc = 0.0;
        for (int f = NI - 1; f >= 0; --f) {
            acc += (double)out[NI + f + 1];
            out[f] = (float)acc;
        }
        return;
    }
    for (int i = NI - 1; i >= 0; --i) {
        double acc = 0.0;
        for (int j = i + 1; j < NV; ++j) acc += (double)(a.gw ? a.gw->w[i][j] : a.g.w[i][j]) * out[j];
        out[i] = (float)acc;
    }
}

// Export of the label state: internal [z][l][y][pitch] -> dense [l][z][y][x] fp32: the labeling u
// (pf_get_labeling) or, raw = 1, the stored lambda itself (pf_get_state).
__global__ void export_u_kernel(const void *__restrict__ u, float *__restrict__ out, int NL, int nx, int ny,
                                int pitch, int64_t nz, int ufmt, int raw) {
    const int64_t V = (int64_t)nx * ny * nz, P = (int64_t)pitch * ny;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t z = i / ((int64_t)nx * ny);
        const int r = (int)(i - z * (int64_t)nx * ny);
        const int y = r / nx, x = r - y * nx;
        const int64_t b = z * NL * P + (int64_t)y * pitch + x;
        for (int l = 0; l < NL; ++l) out[l * V + i] = raw ? state_at(u, b + l * P, ufmt) : u_at(u, b + l * P, ufmt);
    }
}

// Import of a label state (pf_set_state): dense [l][z][y][x] fp32 on the device -> internal storage.  linear = 1:
// the labeling u itself, lambda = log2 u (correctly rounded log2f; u = 0 gives -inf, a label that is exactly
// dead); else lambda.  Stored as fp32 or (ufmt 2) rounded to nearest binary16.
__global__ void import_u_kernel(const float *__restrict__ in, void *__restrict__ u, int NL, int nx, int ny, int pitch,
                                int64_t nz, int ufmt, int linear) {
    const int64_t V = (int64_t)nx * ny * nz, P = (int64_t)pitch * ny;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t z = i / ((int64_t)nx * ny);
        const int r = (int)(i - z * (int64_t)nx * ny);
        const int y = r / nx, x = r - y * nx;
        const int64_t b = z * NL * P + (int64_t)y * pitch + x;
        for (int l = 0; l < NL; ++l) {
            const float v = linear ? log2f(in[l * V + i]) : in[l * V + i];
            if (ufmt == 2) reinterpret_cast<__half *>(u)[b + l * P] = __float2half_rn(v);
            else reinterpret_cast<float *>(u)[b + l * P] = v;
        }
    }
}

__global__ void f32_to_bf16_kernel(const float *__restrict__ src, uint16_t *__restrict__ dst, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = f32_to_bf16_rn(src[i]);
}

__global__ void energy_kernel(const EnergyArgs a, double *partial) {
    const int64_t P = (int64_t)a.pitch * a.ny;
    const int64_t V = (int64_t)a.nx * a.ny * a.nzl;
    const int NV = a.NV, NI = a.NI, NL = a.NL, NF = a.NF;
    const int64_t ups = (int64_t)NL * P, qps = (int64_t)3 * NF * P;
    double e_acc = 0.0, f_acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t z = i / ((int64_t)a.nx * a.ny);
        const int r = (int)(i - z * (int64_t)a.nx * a.ny);
        const int y = r / a.nx, x = r - y * a.nx;
        const int64_t pix = (int64_t)y * a.pitch + x;
        const int64_t zg = a.zg0 + z;
        // ---- primal: sum_L D_L u_L + sum_v S_v |nabla u_v|
        float uc[2 * kMaxNodes], un[2 * kMaxNodes];
        labels_at(a, z * ups + pix, P, uc);
        for (int l = 0; l < NL; ++l) e_acc += (double)load_D(a.D, z * ups + l * P + pix, a.d_bf16) * (double)uc[NI + l];
        double g2[2 * kMaxNodes], g1[2 * kMaxNodes];
        for (int v = 0; v < NV; ++v) { g2[v] = 0.0; g1[v] = 0.0; }
        if (x < a.nx - 1) {
            labels_at(a, z * ups + pix + 1, P, un);
            for (int v = 0; v < NV; ++v) { double g = (double)un[v] - uc[v]; g2[v] += g * g; g1[v] += fabs(g); }
        }
        if (y < a.ny - 1) {
            labels_at(a, z * ups + pix + a.pitch, P, un);
            for (int v = 0; v < NV; ++v) { double g = (double)un[v] - uc[v]; g2[v] += g * g; g1[v] += fabs(g); }
        }
        if (a.ndim == 3 && zg < a.nzg - 1) {
            labels_at(a, (z + 1) * ups + pix, P, un);
            for (int v = 0; v < NV; ++v) { double g = (double)un[v] - uc[v]; g2[v] += g * g; g1[v] += fabs(g); }
        }
        for (int v = 0; v < NF; ++v) {  // nodes without a flow have zero capacity
            float sv;
            const float sn = a.gw ? a.gw->s[v] : a.g.s[v];
            if (a.s_kind == 0) sv = sn;
            else if (a.s_kind == 1) sv = a.S[z * P + pix] * sn;
            else sv = a.S[(z * NF + v) * P + pix];
            e_acc += (double)sv * (a.cap == 0 ? sqrt(g2[v]) : g1[v]);
        }
        // ---- dual: min over end labels of d_L
        double d[2 * kMaxNodes];
        const float *qb = a.q + z * qps + pix;
        for (int v = 0; v < NV; ++v) {
            double dv = 0.0;
            if (v < NF) {
                dv = (double)qb[v * P] - (x > 0 ? (double)qb[v * P - 1] : 0.0);
                dv += (double)qb[(NF + v) * P] - (y > 0 ? (double)qb[(NF + v) * P - a.pitch] : 0.0);
                if (a.ndim == 3)
                    dv += (double)qb[(2 * NF + v) * P] - (zg > 0 ? (double)qb[(2 * NF + v) * P - qps] : 0.0);
            }
            d[v] = dv;
        }
        for (int l = 0; l < NL; ++l) d[NI + l] += (double)load_D(a.D, z * ups + l * P + pix, a.d_bf16);
        if (a.model == 1) {  // prefix: d_{L_i} += sum_{j <= i} div q_j
            double run = 0.0;
            for (int i = 1; i < NL; ++i) {
                run += d[i - 1];
                d[NI + i] += run;
            }
        } else {
            for (int ii = 0; ii < NI; ++ii)
                for (int j = ii + 1; j < NV; ++j) d[j] += (double)(a.gw ? a.gw->w[ii][j] : a.g.w[ii][j]) * d[ii];
        }
        double mn = d[NI];
        for (int l = 1; l < NL; ++l) mn = fmin(mn, d[NI + l]);
        f_acc += mn;
    }
    __shared__ double se[256], sf[256];
    se[threadIdx.x] = e_acc;
    sf[threadIdx.x] = f_acc;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) { se[threadIdx.x] += se[threadIdx.x + s]; sf[threadIdx.x] += sf[threadIdx.x + s]; }
        __syncthreads();
    }
    if (threadIdx.x == 0) { partial[2 * blockIdx.x] = se[0]; partial[2 * blockIdx.x + 1] = sf[0]; }
}

__global__ void energy_finish_kernel(const double *partial, int n, double *out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double e = 0.0, f = 0.0;
        for (int i = 0; i < n; ++i) { e += partial[2 * i]; f += partial[2 * i + 1]; }
        out[0] = e;
        out[1] = f;
    }
}

cudaError_t launch_fill(float *p, int64_t n, float v, cudaStream_t st) {
    fill_kernel<<<1184, 256, 0, st>>>(p, n, v);
    return cudaGetLastError();
}

cudaError_t launch_argmax(const void *u, uint8_t *out, int NL, int nx, int ny, int pitch, int64_t nz, int ufmt,
                          cudaStream_t st) {
    argmax_kernel<<<1184, 256, 0, st>>>(u, out, NL, nx, ny, pitch, nz, ufmt);
    return cudaGetLastError();
}

cudaError_t launch_export_u(const void *u, float *out, int NL, int nx, int ny, int pitch, int64_t nz, int ufmt, int raw,
                            cudaStream_t st) {
    export_u_kernel<<<1184, 256, 0, st>>>(u, out, NL, nx, ny, pitch, nz, ufmt, raw);
    return cudaGetLastError();
}

cudaError_t launch_import_u(const float *in, void *u, int NL, int nx, int ny, int pitch, int64_t nz, int ufmt,
                            int linear, cudaStream_t st) {
    import_u_kernel<<<1184, 256, 0, st>>>(in, u, NL, nx, ny, pitch, nz, ufmt, linear);
    return cudaGetLastError();
}

cudaError_t launch_fill_half(void *p, int64_t n, float v, cudaStream_t st) {
    fill_half_kernel<<<1184, 256, 0, st>>>(reinterpret_cast<__half *>(p), n, v);
    return cudaGetLastError();
}

cudaError_t launch_f32_to_bf16(const float *src, uint16_t *dst, int64_t n, cudaStream_t st) {
    f32_to_bf16_kernel<<<1184, 256, 0, st>>>(src, dst, n);
    return cudaGetLastError();
}

cudaError_t launch_node_labeling(const void *u, float *out, const NodeWeights &w, int NL, int nx, int ny, int pitch,
                                 int64_t nz, int ufmt, cudaStream_t st) {
    node_labeling_kernel<<<1184, 256, 0, st>>>(u, out, w, NL, nx, ny, pitch, nz, ufmt);
    return cudaGetLastError();
}

cudaError_t launch_check_nonneg(const float *p, int64_t n, unsigned int *flag, cudaStream_t st) {
    min_kernel<<<592, 256, 0, st>>>(p, n, flag);
    return cudaGetLastError();
}

cudaError_t launch_energy(const EnergyArgs &a, double *partial, int nblocks, double *out, cudaStream_t st) {
    energy_kernel<<<nblocks, 256, 0, st>>>(a, partial);
    energy_finish_kernel<<<1, 32, 0, st>>>(partial, nblocks, out);
    return cudaGetLastError();
}

}  // namespace pf
